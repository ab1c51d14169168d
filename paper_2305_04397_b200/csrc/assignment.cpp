// Agent-to-task assignment (reference: assignment.hpp:54-136,138-150).
//
// Maximum-value assignment by the O(n^3) shortest-augmenting-path Hungarian method on
// the cost -c with row/column potentials, followed by the reference's deterministic tie
// rule: among all optimal assignments (= perfect matchings inside the tight-edge graph,
// |a - u - v| <= 1e-9 (1 + max|c|)) return the lexicographically smallest
// (f(0), f(1), ...). The potential updates use the same operation order as the reference
// so the tight graph -- and hence the chosen assignment -- is identical.
#include <algorithm>
#include <cmath>
#include <limits>

#include "morap.hpp"

namespace morap {

namespace {

// Kuhn augmenting paths restricted to the still-free tasks/agents.
class TightMatcher {
 public:
  TightMatcher(const std::vector<std::vector<char>>& tight, const std::vector<char>& freeTask,
               const std::vector<char>& freeAgent)
      : tight_(tight), freeTask_(freeTask), freeAgent_(freeAgent), owner_(tight.size(), -1), mark_(tight.size()) {}

  bool perfect() {
    const int n = static_cast<int>(tight_.size());
    for (int j = 0; j < n; ++j) {
      if (!freeTask_[j]) continue;
      std::fill(mark_.begin(), mark_.end(), 0);
      if (!grow(j)) return false;
    }
    return true;
  }

 private:
  bool grow(int task) {
    const int n = static_cast<int>(tight_.size());
    for (int i = 0; i < n; ++i) {
      if (!freeAgent_[i] || !tight_[task][i] || mark_[i]) continue;
      mark_[i] = 1;
      if (owner_[i] < 0 || grow(owner_[i])) {
        owner_[i] = task;
        return true;
      }
    }
    return false;
  }
  const std::vector<std::vector<char>>& tight_;
  const std::vector<char>& freeTask_;
  const std::vector<char>& freeAgent_;
  std::vector<int> owner_;
  std::vector<char> mark_;
};

}  // namespace

Assignment maxAssignment(const Mat& c) {
  if (c.rows != c.cols) fail(Errc::NonSquare, "assignment needs a square value matrix");
  const int n = c.rows;
  if (n == 0) return {};
  double big = 0.0;
  for (double v : c.a) {
    if (!std::isfinite(v)) fail(Errc::InvalidModel, "assignment value must be finite");
    big = std::max(big, std::fabs(v));
  }
  // 1-based potentials; column 0 is the virtual start of every augmenting search
  const double INF = std::numeric_limits<double>::infinity();
  auto cost = [&](int agent, int task) { return -c(agent - 1, task - 1); };
  std::vector<double> u(static_cast<size_t>(n) + 1, 0.0), v(static_cast<size_t>(n) + 1, 0.0), slack(static_cast<size_t>(n) + 1);
  std::vector<int> rowOfCol(static_cast<size_t>(n) + 1, 0), from(static_cast<size_t>(n) + 1, 0);
  for (int agent = 1; agent <= n; ++agent) {
    rowOfCol[0] = agent;
    int col = 0;
    std::fill(slack.begin(), slack.end(), INF);
    std::vector<char> done(static_cast<size_t>(n) + 1, 0);
    while (true) {
      done[col] = 1;
      const int r = rowOfCol[col];
      double step = INF;
      int nextCol = -1;
      for (int j = 1; j <= n; ++j) {
        if (done[j]) continue;
        const double reduced = cost(r, j) - u[r] - v[j];
        if (reduced < slack[j]) {
          slack[j] = reduced;
          from[j] = col;
        }
        if (slack[j] < step) {
          step = slack[j];
          nextCol = j;
        }
      }
      for (int j = 0; j <= n; ++j) {
        if (done[j]) {
          u[rowOfCol[j]] += step;
          v[j] -= step;
        } else {
          slack[j] -= step;
        }
      }
      col = nextCol;
      if (rowOfCol[col] == 0) break;
    }
    while (col) {  // flip the augmenting path
      const int prev = from[col];
      rowOfCol[col] = rowOfCol[prev];
      col = prev;
    }
  }

  const double tau = 1e-9 * (1.0 + big);
  std::vector<std::vector<char>> tight(static_cast<size_t>(n), std::vector<char>(static_cast<size_t>(n), 0));
  for (int j = 1; j <= n; ++j)
    for (int i = 1; i <= n; ++i) tight[j - 1][i - 1] = std::fabs(cost(i, j) - u[i] - v[j]) <= tau;

  Assignment out;
  out.agentOf.assign(static_cast<size_t>(n), -1);
  std::vector<char> freeTask(static_cast<size_t>(n), 1), freeAgent(static_cast<size_t>(n), 1);
  for (int j = 0; j < n; ++j) {
    freeTask[j] = 0;
    for (int i = 0; i < n && out.agentOf[j] < 0; ++i) {
      if (!freeAgent[i] || !tight[j][i]) continue;
      freeAgent[i] = 0;
      if (TightMatcher(tight, freeTask, freeAgent).perfect()) out.agentOf[j] = i;
      else freeAgent[i] = 1;
    }
    if (out.agentOf[j] < 0) fail(Errc::SolverFailure, "tight graph lost its perfect matching");
  }
  for (int j = 0; j < n; ++j) out.value += c(out.agentOf[j], j);
  return out;
}

bool validateBistochastic(const Mat& x, double entryTol, double sumTol) {
  if (x.rows != x.cols) return false;
  for (double e : x.a)
    if (!std::isfinite(e) || e < -entryTol) return false;
  const int n = x.rows;
  for (int i = 0; i < n; ++i) {
    double rs = 0.0, cs = 0.0;
    for (int j = 0; j < n; ++j) {
      rs += std::max(0.0, x(i, j));
      cs += std::max(0.0, x(j, i));
    }
    if (std::fabs(rs - 1.0) > sumTol || std::fabs(cs - 1.0) > sumTol) return false;
  }
  return true;
}

}  // namespace morap
