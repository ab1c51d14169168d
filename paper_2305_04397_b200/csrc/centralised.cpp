// Centralised formulation (reference: centralised.hpp) on the GPU.
//
// buildCentralised explores (agent block i, task j, product state p, assigned mask) breadth
// first from (0, 0, initial of product (0,0), {}) and numbers states in discovery order, so
// its CSR is the reference's array for array (tests/test_centralised.py). The rows of a
// state: an agent that holds the current task moves with its product's rows (costs to
// objective i, successes to objective n + j) until the task ends, then b3 hands the next
// task to the lowest free agent (or "!halt" after the last task); an agent that does not
// hold it gets b1 (take it) and, if one exists, b2 (pass it to the next free agent).
// The supporting point is one weighted optimize job on the whole model plus one fused
// multi-RHS evaluation of its policy under all 2n objectives -- the same device kernels as
// the decentralised path, on a single large model instead of n^2 small ones.
#include <chrono>
#include <cstring>
#include <unordered_map>

#include "morap.hpp"
#include "morap_cuda.h"

namespace morap {

namespace {

void ck(morap_ctx* ctx, int status, const char* what) {
  if (status == MORAP_OK) return;
  const std::string msg = std::string(what) + ": " + morap_cuda_last_error(ctx);
  if (status >= 1 && status <= 21) throw Error(static_cast<Errc>(status - 1), msg);
  throw Error(Errc::SolverFailure, msg);
}

[[noreturn]] void jobFailed(int status, const char* what) {
  const Errc e = status >= 1 && status <= 21 ? static_cast<Errc>(status - 1) : Errc::SolverFailure;
  const char* why = status == MORAP_NON_CONVERGENCE     ? "value iteration did not converge within the sweep cap"
                    : status == MORAP_NOT_REWARD_FINITE ? "some scheduler avoids the objective with positive probability"
                                                        : "job failed";
  throw Error(e, std::string(what) + ": " + why);
}

double seconds(std::chrono::steady_clock::time_point a) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
}

// (i, j, mask, p) packed: 5 + 5 + 16 bits above a 38-bit product state
uint64_t tupleKey(int i, int j, int p, uint32_t mask) {
  return (static_cast<uint64_t>(i) << 59) | (static_cast<uint64_t>(j) << 54) | (static_cast<uint64_t>(mask) << 38) |
         static_cast<uint64_t>(p);
}

}  // namespace

CentralisedMdp buildCentralised(const MorapInstance& inst, long stateGuard) {
  const int n = inst.n;
  if (n > 16) fail(Errc::SizeGuard, "centralised construction supports at most 16 agents");
  if (stateGuard < 1) fail(Errc::InvalidConfig, "state guard must be positive");
  CentralisedMdp c;
  c.n = n;
  c.realTasks = inst.realTasks;
  auto product = [&](int i, int j) -> const ProductMdp& {
    const ProductMdp& p = *inst.products[static_cast<size_t>(i)][static_cast<size_t>(j)];
    requireFull(p, "centralised construction");
    return p;
  };

  std::unordered_map<uint64_t, int> id;
  auto visit = [&](int i, int j, int p, uint32_t mask) {
    auto [it, fresh] = id.emplace(tupleKey(i, j, p, mask), static_cast<int>(c.agentIdx.size()));
    if (fresh) {
      if (it->second >= stateGuard)
        fail(Errc::SizeGuard, "centralised reachable states exceed the guard of " + std::to_string(stateGuard));
      c.agentIdx.push_back(i);
      c.taskIdx.push_back(j);
      c.productState.push_back(p);
      c.assigned.push_back(mask);
    }
    return it->second;
  };
  visit(0, 0, product(0, 0).mdp.initial, 0u);

  Mdp& m = c.mdp;
  m.trnOffset.push_back(0);
  std::vector<int> rowAgent, rowTask;  // owning block of each agent-move row (-1: control row)
  std::vector<double> rowCost, rowSuccess;
  auto controlRow = [&](const char* name, int to) {
    m.succ.push_back(to);
    m.prob.push_back(1.0);
    m.trnOffset.push_back(static_cast<int>(m.succ.size()));
    m.actionName.emplace_back(name);
    rowAgent.push_back(-1);
    rowTask.push_back(-1);
    rowCost.push_back(0.0);
    rowSuccess.push_back(0.0);
  };
  // states are processed in discovery order (a FIFO over ids is exactly that)
  for (size_t s = 0; s < c.agentIdx.size(); ++s) {
    const int i = c.agentIdx[s], j = c.taskIdx[s], p = c.productState[s];
    const uint32_t mask = c.assigned[s];
    const ProductMdp& prod = product(i, j);
    const bool ended = prod.done[static_cast<size_t>(p)] != 0;
    const bool last = j == n - 1;
    const bool holds = (mask >> i) & 1u;
    m.rowOffset.push_back(m.numActions());
    c.taskEnded.push_back(ended ? 1 : 0);
    c.done.push_back(ended && last ? 1 : 0);
    if (holds && ended && last) {
      controlRow("!halt", static_cast<int>(s));
    } else if (holds && ended) {
      int next = 0;
      while ((mask >> next) & 1u) ++next;  // a free agent always exists (one b1 per started task)
      controlRow("b3", visit(next, j + 1, product(next, j + 1).mdp.initial, mask));
    } else if (holds) {
      const Mdp& a = prod.mdp;
      for (int r = a.actionsBegin(p); r < a.actionsEnd(p); ++r) {
        for (int k = a.trnBegin(r); k < a.trnEnd(r); ++k) {
          const int to = visit(i, j, a.succ[k], mask);
          m.succ.push_back(to);
          m.prob.push_back(a.prob[k]);
        }
        m.trnOffset.push_back(static_cast<int>(m.succ.size()));
        m.actionName.push_back(a.actionName[r]);
        rowAgent.push_back(i);
        rowTask.push_back(j);
        rowCost.push_back(prod.cost[static_cast<size_t>(r)]);
        rowSuccess.push_back(prod.success[static_cast<size_t>(r)]);
      }
    } else {
      controlRow("b1", visit(i, j, p, mask | (1u << i)));
      for (int k = i + 1; k < n; ++k)
        if (!((mask >> k) & 1u)) {
          controlRow("b2", visit(k, j, product(k, j).mdp.initial, mask));
          break;
        }
    }
  }
  m.numStates = static_cast<int>(c.agentIdx.size());
  m.rowOffset.push_back(m.numActions());
  m.initial = 0;
  m.labels.assign(static_cast<size_t>(m.numStates), {});
  validateMdp(m);
  const int R = m.numActions();
  c.rewards.assign(static_cast<size_t>(2 * n), RewardStructure(static_cast<size_t>(R), 0.0));
  for (int r = 0; r < R; ++r) {
    if (rowAgent[r] >= 0) c.rewards[static_cast<size_t>(rowAgent[r])][static_cast<size_t>(r)] = rowCost[r];
    if (rowTask[r] >= 0) c.rewards[static_cast<size_t>(n + rowTask[r])][static_cast<size_t>(r)] = rowSuccess[r];
  }
  c.rewardFinite = checkRewardFinite(m, c.done);
  return c;
}

namespace {

int deviceModel(const CentralisedMdp& c, GpuBackend& gpu) {
  const int K = static_cast<int>(c.rewards.size());
  std::vector<const double*> objs;
  if (K <= MORAP_MAX_OBJECTIVES)  // weights applied on the device; else rho_w from the host
    for (const auto& r : c.rewards) objs.push_back(r.data());
  std::vector<uint8_t> done(c.done.begin(), c.done.end());
  morap_csr_view v{};
  v.num_states = c.mdp.numStates;
  v.num_rows = c.mdp.numActions();
  v.nnz = static_cast<int32_t>(c.mdp.succ.size());
  v.initial = c.mdp.initial;
  v.reward_finite = c.rewardFinite ? 1 : 0;
  v.num_objectives = static_cast<int32_t>(objs.size());
  v.row_offset = c.mdp.rowOffset.data();
  v.trn_offset = c.mdp.trnOffset.data();
  v.succ = c.mdp.succ.data();
  v.prob = c.mdp.prob.data();
  v.done = done.data();
  v.rewards = objs.data();
  return gpu.modelIdFor(c.uid, v);
}

Vec expandCentralised(const CentralisedMdp& c, const Vec& user) {
  if (static_cast<int>(user.size()) != c.n + c.realTasks)
    fail(Errc::DimensionMismatch, "expected " + std::to_string(c.n + c.realTasks) +
                                      " thresholds (costs first, then task probabilities)");
  Vec t(static_cast<size_t>(2 * c.n), 0.0);
  for (int i = 0; i < c.n; ++i) t[static_cast<size_t>(i)] = user[static_cast<size_t>(i)];
  for (int j = 0; j < c.realTasks; ++j) t[static_cast<size_t>(c.n + j)] = user[static_cast<size_t>(c.n + j)];
  return t;
}

}  // namespace

SupportingPoint centralisedSupportingPoint(const CentralisedMdp& c, const Vec& w, GpuBackend& gpu, double valueEps,
                                           QueryStats* stats) {
  const int K = static_cast<int>(c.rewards.size());
  if (static_cast<int>(w.size()) != K) fail(Errc::DimensionMismatch, "weight vector must have one entry per objective");
  const int32_t id = deviceModel(c, gpu);
  morap_ctx* ctx = gpu.ctx();
  const int S = c.mdp.numStates;
  const auto t0 = std::chrono::steady_clock::now();
  double value = 0, resid = 0;
  int32_t sweeps = 0, status = 0;
  if (K <= MORAP_MAX_OBJECTIVES) {
    ck(ctx, morap_cuda_optimize(ctx, 1, &id, w.data(), K, valueEps, 100000, &value, &sweeps, &resid, &status),
       "centralised optimize");
  } else {
    std::vector<const RewardStructure*> parts;
    for (const auto& r : c.rewards) parts.push_back(&r);
    const RewardStructure rho = weightedReward(parts, w);
    const double* rp = rho.data();
    ck(ctx, morap_cuda_optimize_rho(ctx, 1, &id, &rp, valueEps, 100000, &value, &sweeps, &resid, &status),
       "centralised optimize");
  }
  if (status != MORAP_OK) jobFailed(status, "centralised weighted optimization failed");
  SupportingPoint out;
  out.schedulers.resize(1);
  out.schedulers[0].rows.resize(static_cast<size_t>(S));
  ck(ctx, morap_cuda_fetch_policy(ctx, 0, out.schedulers[0].rows.data()), "fetch policy");
  if (stats) {
    stats->optimizeJobs += 1;
    stats->optimizeBackups += static_cast<double>(sweeps) * static_cast<double>(c.mdp.succ.size());
    stats->optimizeSeconds += seconds(t0);
  }
  // the optimal scheduler under every objective (centralised.hpp:208-210), one fused batch
  const auto t1 = std::chrono::steady_clock::now();
  out.r.assign(static_cast<size_t>(K), 0.0);
  std::vector<int32_t> esw(static_cast<size_t>(K)), est(static_cast<size_t>(K));
  std::vector<double> eres(static_cast<size_t>(K));
  if (K <= MORAP_MAX_RHS && K <= MORAP_MAX_OBJECTIVES) {
    std::vector<int32_t> objective(static_cast<size_t>(K));
    for (int k = 0; k < K; ++k) objective[k] = k;
    const int32_t job = 0;
    ck(ctx, morap_cuda_evaluate_optimized(ctx, 1, &job, K, objective.data(), valueEps, 100000, out.r.data(),
                                          esw.data(), eres.data(), est.data()),
       "centralised evaluate");
  } else {
    std::vector<int32_t> ids(static_cast<size_t>(K), id);
    std::vector<const int32_t*> pol(static_cast<size_t>(K), out.schedulers[0].rows.data());
    std::vector<const double*> rho(static_cast<size_t>(K));
    for (int k = 0; k < K; ++k) rho[k] = c.rewards[static_cast<size_t>(k)].data();
    ck(ctx, morap_cuda_evaluate(ctx, K, ids.data(), pol.data(), rho.data(), valueEps, 100000, out.r.data(),
                                esw.data(), eres.data(), est.data()),
       "centralised evaluate");
  }
  for (int k = 0; k < K; ++k)
    if (est[k] != MORAP_OK) jobFailed(est[k], "centralised evaluation failed");
  if (stats) {
    stats->evaluateJobs += K;
    for (int k = 0; k < K; ++k) stats->evaluateStateBackups += static_cast<double>(esw[k]) * S;
    stats->evaluateSeconds += seconds(t1);
  }
  return out;
}

ParetoResult centralisedParetoPoint(const CentralisedMdp& c, const Vec& thresholds, const NormMatrix& norm,
                                    double eps, GpuBackend& gpu, int iterationCap, QueryStats* stats) {
  return runParetoCore(expandCentralised(c, thresholds), norm, eps, iterationCap, false, nullptr,
                       [&](const Vec& w) { return centralisedSupportingPoint(c, w, gpu, 1e-6, stats); });
}

}  // namespace morap
