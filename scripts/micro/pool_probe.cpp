// Cost of one parallel region of the host pool (csrc/linalg.cpp Pool via parallelFor): an
// empty region over all threads, timed back to back (dev probe for the QP schedule).
#include <chrono>
#include <cstdio>

#include "morap.hpp"

int main() {
  using clk = std::chrono::steady_clock;
  for (int parts : {2, 4, 8, 16}) {
    for (int i = 0; i < 1000; ++i) morap::parallelFor(parts, [](int) {});
    const auto t0 = clk::now();
    const int N = 20000;
    for (int i = 0; i < N; ++i) morap::parallelFor(parts, [](int) {});
    std::printf("parts %2d: %.2f us per region\n", parts,
                std::chrono::duration<double, std::micro>(clk::now() - t0).count() / N);
  }
}
