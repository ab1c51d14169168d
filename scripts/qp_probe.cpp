// Times projectToLowerApprox (geometry.hpp:225's active-set QP, csrc/geometry.cpp) on the
// supporting points of a recorded query (tests/golden/replay/*.npz, converted by
// scripts/qp_probe.py) with the unblocked and the blocked/threaded dense solve, and checks
// that both return the same bits. Host-only: no GPU involved.
//   qp_probe <points.bin> k1 k2 ...
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "morap.hpp"

using namespace morap;

#ifdef MORAP_QP_PROFILE
namespace morap {
extern double g_qpProf[8];
}
#endif

static unsigned long long fingerprint(const ProjectionResult& p) {
  unsigned long long h = 1469598103934665603ull;
  auto mix = [&](double x) {
    unsigned long long b;
    std::memcpy(&b, &x, 8);
    h = (h ^ b) * 1099511628211ull;
  };
  for (double x : p.x) mix(x);
  for (double x : p.lambda) mix(x);
  mix(p.distance);
  return h;
}

int main(int argc, char** argv) {
  FILE* f = std::fopen(argv[1], "rb");
  long long hdr[2];
  if (!f || std::fread(hdr, 8, 2, f) != 2) return 2;
  const int T = static_cast<int>(hdr[0]), d = static_cast<int>(hdr[1]);
  Vec t(d);
  std::vector<Vec> r(T, Vec(d));
  bool ok = std::fread(t.data(), 8, d, f) == static_cast<size_t>(d);
  for (auto& v : r) ok = ok && std::fread(v.data(), 8, d, f) == static_cast<size_t>(d);
  if (!ok) return 2;
  int bad = 0;
  for (int a = 2; a < argc; ++a) {
    const int k = std::atoi(argv[a]);
    LowerApprox phi;
    phi.points.assign(r.begin(), r.begin() + k);
    double sec[2];
    unsigned long long h[2];
    for (int mode = 1; mode >= 0; --mode) {
      denseSolveMode() = mode;
#ifdef MORAP_QP_PROFILE
      std::fill_n(g_qpProf, 8, 0.0);  // the profile is the blocked run's
#endif
      const auto t0 = std::chrono::steady_clock::now();
      const ProjectionResult p = projectToLowerApprox(t, phi, NormMatrix::identity(d));
      sec[mode] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      h[mode] = fingerprint(p);
    }
    bad += h[0] != h[1];
#ifdef MORAP_QP_PROFILE
    std::printf("  blocked solve: panels %.3f (inside the next region)  list %.3f  pivot rows %.3f  lookahead + "
                "overlapped region %.3f  re-solves %.3f  KKT assembly %.3f  rest of the QP %.3f s\n",
                g_qpProf[0], g_qpProf[1], g_qpProf[2], g_qpProf[3], g_qpProf[4], g_qpProf[5],
                sec[0] - (g_qpProf[1] + g_qpProf[2] + g_qpProf[3] + g_qpProf[4] + g_qpProf[5]));
    std::printf("  per projection: eliminations %.1f G row updates (sum dim^3/3), re-solves %.0f\n",
                g_qpProf[6] / 1e3, g_qpProf[7]);
    std::fill_n(g_qpProf, 8, 0.0);
#endif
    std::printf("D=%d points=%d unblocked %.3f s  blocked %.3f s  (x%.2f)  bits %s\n", d, k, sec[1], sec[0],
                sec[1] / sec[0], h[0] == h[1] ? "equal" : "DIFFER");
  }
  return bad ? 1 : 0;
}
