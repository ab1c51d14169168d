// Time buildProduct on one C4 product (10x10 grid, 100 racks): dev probe for the host build.
#include <chrono>
#include <cstdio>

#include "morap.hpp"

using namespace morap;

// (levels) BFS depth of a product: how many level-synchronous steps a device BFS takes
int levels_of(const ProductMdp& p) {
  const Mdp& m = p.mdp;
  std::vector<int> lvl(m.numStates, -1);
  std::vector<int> q{m.initial};
  lvl[m.initial] = 0;
  int depth = 0;
  for (size_t h = 0; h < q.size(); ++h) {
    int x = q[h];
    for (int r = m.rowOffset[x]; r < m.rowOffset[x + 1]; ++r)
      for (int k = m.trnOffset[r]; k < m.trnOffset[r + 1]; ++k)
        if (lvl[m.succ[k]] < 0) { lvl[m.succ[k]] = lvl[x] + 1; depth = std::max(depth, lvl[x] + 1); q.push_back(m.succ[k]); }
  }
  return depth;
}

int main(int argc, char** argv) {
  WarehouseConfig c;
  c.width = c.height = 10;
  c.agents = 100;
  c.slip = 0.05;
  c.feed = {0, 0};
  c.seed = 42;
  for (int k = 0; k < 100; ++k) c.racks.push_back({9 - k % 10, 9 - k / 10});
  auto [m, cost] = generateAgent(c, 0);
  Dfa d = taskAutomaton(c, argc > 1 ? atoi(argv[1]) : 0);
  printf("agent S=%d R=%d nnz=%zu  dfa Q=%d L=%d\n", m.numStates, m.numActions(), m.succ.size(), d.numLocations,
         d.numLetters());
  for (int rep = 0; rep < 5; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    ProductMdp p = buildProduct(m, cost, d, 0, 0);
    auto t1 = std::chrono::steady_clock::now();
    bool rf = checkRewardFinite(p);
    auto t2 = std::chrono::steady_clock::now();
    printf("S=%d R=%d nnz=%zu build %.2f ms (checkRewardFinite alone %.2f ms) rf=%d\n", p.mdp.numStates,
           p.mdp.numActions(), p.mdp.succ.size(), std::chrono::duration<double, std::milli>(t1 - t0).count(),
           std::chrono::duration<double, std::milli>(t2 - t1).count(), (int)rf);
    if (rep == 0) printf("BFS depth %d\n", levels_of(p));
  }
}
