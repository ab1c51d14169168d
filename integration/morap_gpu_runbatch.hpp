// morap_gpu_runbatch.hpp -- the B200 backend as a plug-in for the reference's job engine.
//
// Drop-in for
//     std::map<long, JobResult> runBatch(std::vector<Job>, const PoolConfig&)
//         (/root/reference/proj/include/morap/engine.hpp:370-425)
// with the same contract: one JobResult per job id, failures contained per job
// (JobResult{ok = false, error, errc}, engine.hpp:140-150), duplicate ids / a bad pool
// configuration rejected with Errc::InvalidConfig, results independent of how the batch is
// split. Every Bellman solve runs in libmorap_cuda.so (include/morap_cuda.h) and returns
// the reference's bits: values, sweeps, residuals and argmax policies.
//
// A maintainer wires it in at the two runBatch call sites of supportingPoint
// (solver.hpp:133,172), e.g. by building solver.hpp with
//     #include "morap/engine.hpp"
//     #include "morap_gpu_runbatch.hpp"
//     #define runBatch gpu_runBatch
//     #include "morap/solver.hpp"
// (INTEGRATION.md shows this and the equivalent one-line hook in runBatch itself;
// oracle/ref_gpu_routed.cpp runs the reference's own paretoPoint that way).
//
// Products are uploaded once per ProductMdp (the engine keeps the shared_ptr alive, as the
// reference's instance does, instance.hpp:26). Optimize jobs carry explicit reward vectors
// (Job::reward) -> morap_cuda_optimize_rho; evaluate jobs carry deterministic schedulers ->
// morap_cuda_evaluate. A randomized scheduler is refused per job (the solver never builds
// one). Jobs of a batch are grouped by (kind, eps, sweepCap).
#ifndef MORAP_GPU_RUNBATCH_HPP
#define MORAP_GPU_RUNBATCH_HPP

#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "morap_cuda.h"

namespace morap {

class GpuEngine {
 public:
  static GpuEngine& instance(int device = 0) {
    static GpuEngine eng(device);
    return eng;
  }
  ~GpuEngine() {
    if (ctx_) morap_cuda_destroy(ctx_);
  }

  // Device id of a product (uploaded on first use).
  int32_t model(const std::shared_ptr<const ProductMdp>& m) {
    auto it = ids_.find(m.get());
    if (it != ids_.end()) return it->second;
    const Mdp& g = m->mdp;
    done_.emplace_back(m->done.begin(), m->done.end());
    const double* rw[2] = {m->cost.data(), m->success.data()};
    morap_csr_view v{};
    v.num_states = g.numStates;
    v.num_rows = g.numActions();
    v.nnz = static_cast<int32_t>(g.succ.size());
    v.initial = g.initial;
    v.reward_finite = m->rewardFinite ? 1 : 0;
    v.num_objectives = 2;
    v.row_offset = g.rowOffset.data();
    v.trn_offset = g.trnOffset.data();
    v.succ = g.succ.data();
    v.prob = g.prob.data();
    v.done = done_.back().data();
    v.rewards = rw;
    int32_t id = -1;
    check(morap_cuda_upload(ctx_, 1, &v, &id), "upload");
    keep_.push_back(m);
    ids_.emplace(m.get(), id);
    return id;
  }

  std::map<long, JobResult> run(std::vector<Job>& jobs) {
    std::map<long, JobResult> out;
    // group by (kind, eps, sweepCap): each group is one device batch
    std::map<std::tuple<int, double, int>, std::vector<size_t>> groups;
    for (size_t k = 0; k < jobs.size(); ++k) {
      const Job& j = jobs[k];
      if (!j.model) {
        out[j.id] = failed(Errc::InvalidModel, "job carries no model");
        continue;
      }
      groups[{j.kind == JobKind::Optimize ? 0 : 1, j.eps, j.sweepCap}].push_back(k);
    }
    for (auto& [key, idx] : groups) {
      const bool opt = std::get<0>(key) == 0;
      const double eps = std::get<1>(key);
      const int cap = std::get<2>(key);
      std::vector<int32_t> ids, pos;
      std::vector<const double*> rho;
      std::vector<std::vector<int32_t>> rows;
      std::vector<const int32_t*> rowPtr;
      for (size_t k : idx) {
        Job& j = jobs[k];
        if (static_cast<int>(j.reward.size()) != j.model->mdp.numActions()) {  // numerics.hpp checkReward
          out[j.id] = failed(Errc::DimensionMismatch, "reward structure does not match action rows");
          continue;
        }
        if (!opt) {
          std::vector<int32_t> r;
          if (!deterministic(j.scheduler, j.model->mdp.numStates, r)) {
            out[j.id] = failed(Errc::SolverFailure, "the GPU backend evaluates deterministic schedulers only");
            continue;
          }
          rows.push_back(std::move(r));
        }
        ids.push_back(model(j.model));
        rho.push_back(j.reward.data());
        pos.push_back(static_cast<int32_t>(k));
      }
      const int n = static_cast<int>(ids.size());
      if (n == 0) continue;
      std::vector<double> val(n), res(n);
      std::vector<int32_t> sw(n), st(n);
      if (opt) {
        check(morap_cuda_optimize_rho(ctx_, n, ids.data(), rho.data(), eps, cap, val.data(), sw.data(), res.data(),
                                      st.data()),
              "optimize");
      } else {
        for (auto& r : rows) rowPtr.push_back(r.data());
        check(morap_cuda_evaluate(ctx_, n, ids.data(), rowPtr.data(), rho.data(), eps, cap, val.data(), sw.data(),
                                  res.data(), st.data()),
              "evaluate");
      }
      for (int q = 0; q < n; ++q) {
        const Job& j = jobs[pos[q]];
        if (st[q] != MORAP_OK) {
          out[j.id] = failed(static_cast<Errc>(st[q] - 1), st[q] == MORAP_NOT_REWARD_FINITE
                                                               ? "model is not reward-finite"
                                                               : "value iteration did not converge within the cap");
          continue;
        }
        JobResult r;
        r.ok = true;
        r.value = val[q];
        r.stats.sweeps = sw[q];
        r.stats.residual = res[q];
        r.values.resize(static_cast<size_t>(j.model->mdp.numStates));
        if (opt) {
          check(morap_cuda_fetch_values(ctx_, q, r.values.data()), "fetch values");
          std::vector<int32_t> pol(static_cast<size_t>(j.model->mdp.numStates));
          check(morap_cuda_fetch_policy(ctx_, q, pol.data()), "fetch policy");
          r.policy = makeDeterministic(std::vector<int>(pol.begin(), pol.end()));
        } else {
          check(morap_cuda_fetch_eval_values(ctx_, q, 0, r.values.data()), "fetch values");
        }
        out[j.id] = std::move(r);
      }
    }
    return out;
  }

 private:
  explicit GpuEngine(int device) { check(morap_cuda_create(device, &ctx_), "create"); }

  void check(int rc, const char* what) {
    if (rc != MORAP_OK) {
      const Errc code = rc >= 1 && rc <= 21 ? static_cast<Errc>(rc - 1) : Errc::SolverFailure;
      fail(code, std::string("GPU backend ") + what + ": " + morap_cuda_last_error(ctx_));
    }
  }
  static JobResult failed(Errc c, const std::string& msg) {
    JobResult r;
    r.ok = false;
    r.errc = c;
    r.error = msg;
    return r;
  }
  static bool deterministic(const Scheduler& mu, int S, std::vector<int32_t>& rows) {
    if (static_cast<int>(mu.choice.size()) != S) return false;
    rows.resize(static_cast<size_t>(S));
    for (int s = 0; s < S; ++s) {
      const auto& c = mu.choice[s];
      if (c.size() != 1 || c[0].second != 1.0) return false;
      rows[s] = c[0].first;
    }
    return true;
  }

  morap_ctx* ctx_ = nullptr;
  std::unordered_map<const ProductMdp*, int32_t> ids_;
  std::vector<std::shared_ptr<const ProductMdp>> keep_;
  std::vector<std::vector<uint8_t>> done_;
};

// runBatch's signature and contract (engine.hpp:370-382), on the GPU.
inline std::map<long, JobResult> gpu_runBatch(std::vector<Job> jobs, const PoolConfig& cfg) {
  if (cfg.workers < 1 || cfg.queues < 1 || cfg.capacity < 1) fail(Errc::InvalidConfig, "invalid pool configuration");
  if (jobs.empty()) return {};
  {
    std::map<long, bool> ids;
    for (const Job& j : jobs)
      if (!ids.emplace(j.id, true).second) fail(Errc::InvalidConfig, "duplicate job id " + std::to_string(j.id));
  }
  return GpuEngine::instance().run(jobs);
}

}  // namespace morap

#endif  // MORAP_GPU_RUNBATCH_HPP
