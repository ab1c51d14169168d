// Blocked/threaded solveDense (csrc/linalg.cpp) vs the unblocked elimination it restates
// (common.hpp's Gaussian elimination): the same bits on random sparse KKT-like systems with
// exact ties, signed zeros and tiny pivots, or the same SingularSystem error.
#include <cstdio>
#include <cstring>
#include <random>

#include "morap.hpp"

using namespace morap;

int main() {
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-2.0, 2.0);
  int bad = 0, cases = 0, singular = 0;
  for (int n : {20, 61, 127, 128, 129, 150, 203, 260, 333}) {
    for (int rep = 0; rep < 6; ++rep) {
      const double density = rep < 2 ? 0.05 : rep < 4 ? 0.3 : 1.0;
      Mat A(n, n, 0.0);
      Vec b(n);
      for (int r = 0; r < n; ++r) {
        b[r] = U(rng);
        for (int c = 0; c < n; ++c) {
          const double u = std::uniform_real_distribution<double>(0, 1)(rng);
          if (u < density) A(r, c) = rep % 2 ? std::round(U(rng) * 4) / 4 : U(rng);  // quarter grid: ties
          else if (u < density + 0.05) A(r, c) = -0.0;
        }
        A(r, r) += rep == 5 ? 1e-13 : 0.5;  // rep 5: near-singular columns
      }
      if (rep == 3) A(n / 2, 0) = A(n / 3, 0) = 9.0;  // tie for the first pivot
      if (rep == 4 && n % 2) for (int r = 0; r < n; ++r) A(r, n - 3) = r % 3 ? 0.0 : -0.0;  // singular
      Vec x[2];
      int err[2] = {0, 0};
      for (int mode = 0; mode < 2; ++mode) {
        denseSolveMode() = mode;
        try {
          x[mode] = solveDense(A, b);
        } catch (const Error& e) {
          err[mode] = 1 + static_cast<int>(e.code());
        }
      }
      // recorded elimination, then a re-solve for another rhs: the bits of a fresh solve
      if (!err[0]) {
        Mat Ar = A;
        Vec br = b;
        DenseLU lu;
        const Vec xr = solveDenseRecorded(Ar.a.data(), n, n, br, lu);
        Vec b2(n);
        for (int r = 0; r < n; ++r) b2[r] = U(rng);
        const Vec x2 = solveLU(lu, b2), f2 = solveDense(A, b2);
        if (std::memcmp(xr.data(), x[0].data(), sizeof(double) * n) != 0 ||
            std::memcmp(x2.data(), f2.data(), sizeof(double) * n) != 0) {
          ++bad;
          std::printf("n=%d rep=%d: recorded elimination / re-solve differs\n", n, rep);
        }
      }
      ++cases;
      singular += err[0] != 0;
      const bool same = err[0] == err[1] &&
                        (err[0] || std::memcmp(x[0].data(), x[1].data(), sizeof(double) * n) == 0);
      if (!same) {
        ++bad;
        std::printf("n=%d rep=%d differs (err %d/%d)\n", n, rep, err[0], err[1]);
      }
    }
  }
  std::printf("%d cases, %d singular, %d differ\n", cases, singular, bad);
  return bad ? 1 : 0;
}
