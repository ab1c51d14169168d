// Sharded supporting points: the Pareto query over several GPUs.
//
// The n x n agent-task products are independent, so they are partitioned over shards (one
// GPU each; owner per pair). Per Algorithm-1 iteration (supportingPoint, solver.hpp:103-184):
//   1. every shard optimizes the deduplicated (product, weight bits) jobs of the pairs it
//      owns (one device batch, solver.hpp:110-131);
//   2. the n^2 initial-state values are combined -- each entry from its owner, exact bits;
//   3. the host Hungarian step (maxAssignment) runs on the combined matrix;
//   4. the owner of each assigned pair evaluates its policy under all K objectives (fused
//      multi-RHS batch) and the K*n values are combined.
// No per-sweep communication. Two drivers share these steps:
//   * one process per GPU (torch.distributed): runParetoCore runs on every rank with an
//     exchange callback (an allgather -- NCCL over NVLink on GPUs, gloo in the CPU tests);
//     every rank takes the same decisions from the same combined data;
//   * one process driving several GPUs (the reference's model: one engine feeding several
//     backend queues, engine.hpp:66-72,370-425): one host thread per device runs the shard
//     steps concurrently, the host combines in memory.
// Failures are contained like runBatch (engine.hpp:140-150): a shard whose job failed
// publishes the status in its mask, so every rank / the driver raises the same error.
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <thread>

#include "morap.hpp"
#include "morap_cuda.h"

namespace morap {

namespace {

uint64_t bits(double v) {
  uint64_t b;
  std::memcpy(&b, &v, sizeof b);
  return b;
}

void ck(morap_ctx* ctx, int status, const char* what) {
  if (status == MORAP_OK) return;
  const std::string msg = std::string(what) + ": " + morap_cuda_last_error(ctx);
  if (status >= 1 && status <= 21) throw Error(static_cast<Errc>(status - 1), msg);
  throw Error(Errc::SolverFailure, msg);
}

[[noreturn]] void failStatus(int status, const char* what) {
  const Errc e = status >= 1 && status <= 21 ? static_cast<Errc>(status - 1) : Errc::SolverFailure;
  throw Error(e, std::string(what) + (status == MORAP_NON_CONVERGENCE
                                          ? ": value iteration did not converge within the sweep cap"
                                          : status == MORAP_NOT_REWARD_FINITE
                                                ? ": some scheduler avoids the objective with positive probability"
                                                : ": job failed"));
}

double seconds(std::chrono::steady_clock::time_point a) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
}

// entry k of the combined array: the value of the one shard whose mask is set
void combine(int world, int count, const double* recv, double* out, const char* what) {
  for (int k = 0; k < count; ++k) {
    int owner = -1;
    for (int r = 0; r < world; ++r) {
      const double m = recv[static_cast<size_t>(r) * 2 * count + count + k];
      if (m == 0.0) continue;
      if (m >= 2.0) failStatus(static_cast<int>(m) - 2, what);
      if (owner >= 0) fail(Errc::SolverFailure, std::string(what) + ": an entry has two owners");
      owner = r;
    }
    if (owner < 0) fail(Errc::SolverFailure, std::string(what) + ": an entry has no owner");
    out[k] = recv[static_cast<size_t>(owner) * 2 * count + k];
  }
}

}  // namespace

std::vector<int> lptOwners(const MorapInstance& inst, int world) {
  if (world < 1) fail(Errc::InvalidConfig, "shard count must be positive");
  const int n = inst.n;
  std::vector<int> owner(static_cast<size_t>(n) * n, 0);
  std::map<uint64_t, int> ownerOf;  // distinct product -> shard
  std::vector<std::pair<double, uint64_t>> sized;
  std::vector<uint64_t> order;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const ProductMdp& p = *inst.products[i][j];
      if (ownerOf.emplace(p.uid, -1).second) {
        sized.push_back({static_cast<double>(productNnz(p)), p.uid});
        order.push_back(p.uid);
      }
    }
  // longest processing time first: largest product to the least loaded shard (ties: first
  // occurrence, lowest shard) -- deterministic, the same on every rank
  std::vector<size_t> idx(sized.size());
  for (size_t k = 0; k < idx.size(); ++k) idx[k] = k;
  std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return sized[a].first > sized[b].first; });
  std::vector<double> load(static_cast<size_t>(world), 0.0);
  for (size_t k : idx) {
    const int r = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
    load[static_cast<size_t>(r)] += sized[k].first;
    ownerOf[sized[k].second] = r;
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) owner[static_cast<size_t>(i) * n + j] = ownerOf[inst.products[i][j]->uid];
  return owner;
}

Shard::Shard(const MorapInstance& inst, GpuBackend& gpu, std::vector<int> owner, int rank)
    : inst_(inst), gpu_(gpu), owner_(std::move(owner)), rank_(rank) {
  const size_t pairs = static_cast<size_t>(inst.n) * inst.n;
  if (owner_.size() != pairs) fail(Errc::DimensionMismatch, "one owner per agent-task pair");
}

void Shard::upload() {
  std::vector<const ProductMdp*> mine;
  const int n = inst_.n;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (owner_[static_cast<size_t>(i) * n + j] == rank_) mine.push_back(inst_.products[i][j].get());
  gpu_.uploadCached(mine, gpu_.lean() && inst_.objectives <= 4);
}

void Shard::optimize(const Vec& w, double* values, double* mask, QueryStats* stats) {
  const int n = inst_.n, K = inst_.objectives;
  auto coord = [&](int k, int i, int j) { return k < K - 1 ? k * n + i : (K - 1) * n + j; };
  const auto t0 = std::chrono::steady_clock::now();
  morap_ctx* ctx = gpu_.ctx();
  std::map<std::vector<uint64_t>, int> jobOf;
  jobIJ_.assign(static_cast<size_t>(n) * n, -1);
  std::vector<int32_t> models;
  std::vector<double> weights;
  std::vector<double> nnzOf;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const size_t q = static_cast<size_t>(i) * n + j;
      if (owner_[q] != rank_) continue;
      const ProductMdp* p = inst_.products[i][j].get();
      std::vector<uint64_t> key{p->uid};
      for (int k = 0; k < K; ++k) key.push_back(bits(w[coord(k, i, j)]));
      auto [it, fresh] = jobOf.emplace(std::move(key), static_cast<int>(models.size()));
      if (fresh) {
        models.push_back(gpu_.modelId(p));
        for (int k = 0; k < K; ++k) weights.push_back(w[coord(k, i, j)]);
        nnzOf.push_back(static_cast<double>(productNnz(*p)));
      }
      jobIJ_[q] = it->second;
    }
  const int nj = static_cast<int>(models.size());
  std::vector<double> value(static_cast<size_t>(nj)), resid(static_cast<size_t>(nj));
  std::vector<int32_t> sweeps(static_cast<size_t>(nj)), status(static_cast<size_t>(nj));
  if (nj > 0)
    ck(ctx, morap_cuda_optimize(ctx, nj, models.data(), weights.data(), K, 1e-6, 100000, value.data(), sweeps.data(),
                                resid.data(), status.data()),
       "optimize batch");
  for (size_t q = 0; q < jobIJ_.size(); ++q) {
    values[q] = 0.0;
    mask[q] = 0.0;
    if (jobIJ_[q] < 0) continue;
    const int st = status[static_cast<size_t>(jobIJ_[q])];
    values[q] = st == MORAP_OK ? value[static_cast<size_t>(jobIJ_[q])] : 0.0;
    mask[q] = st == MORAP_OK ? 1.0 : 2.0 + st;
  }
  if (stats) {
    stats->optimizeJobs += nj;
    for (int q = 0; q < nj; ++q) stats->optimizeBackups += static_cast<double>(sweeps[q]) * nnzOf[q];
    stats->optimizeSeconds += seconds(t0);
  }
}

void Shard::evaluate(const Assignment& a, double* r, double* mask, std::vector<Scheduler>& schedulers,
                     QueryStats* stats) {
  const int n = inst_.n, K = inst_.objectives;
  auto coord = [&](int k, int i, int j) { return k < K - 1 ? k * n + i : (K - 1) * n + j; };
  const auto t0 = std::chrono::steady_clock::now();
  morap_ctx* ctx = gpu_.ctx();
  std::vector<int32_t> evalJobs, cols;
  for (int j = 0; j < n; ++j) {
    const size_t q = static_cast<size_t>(a.agentOf[j]) * n + j;
    if (owner_[q] == rank_) {
      evalJobs.push_back(jobIJ_[q]);
      cols.push_back(j);
    }
  }
  for (int k = 0; k < K * n; ++k) r[k] = mask[k] = 0.0;
  const int m = static_cast<int>(evalJobs.size());
  if (m == 0) return;
  std::vector<int32_t> objectives(static_cast<size_t>(K));
  for (int k = 0; k < K; ++k) objectives[k] = k;
  std::vector<double> ev(static_cast<size_t>(m) * K), eres(static_cast<size_t>(m) * K);
  std::vector<int32_t> esw(static_cast<size_t>(m) * K), est(static_cast<size_t>(m) * K);
  ck(ctx, morap_cuda_evaluate_optimized(ctx, m, evalJobs.data(), K, objectives.data(), 1e-6, 100000, ev.data(),
                                        esw.data(), eres.data(), est.data()),
     "evaluate batch");
  for (int q = 0; q < m; ++q) {
    const int j = cols[q], i = a.agentOf[j];
    for (int k = 0; k < K; ++k) {
      const int32_t st = est[static_cast<size_t>(q) * K + k];
      r[coord(k, i, j)] = st == MORAP_OK ? ev[static_cast<size_t>(q) * K + k] : 0.0;
      mask[coord(k, i, j)] = st == MORAP_OK ? 1.0 : 2.0 + st;
    }
  }
  // the schedulers of the pairs evaluated here (IterationRecord::schedulers); the other
  // shards' pairs stay empty on this shard
  std::vector<const int32_t*> rows(static_cast<size_t>(m));
  ck(ctx, morap_cuda_policy_views(ctx, m, evalJobs.data(), rows.data()), "fetch policies");
  for (int q = 0; q < m; ++q) {
    const int j = cols[q];
    schedulers[j].rows.assign(rows[q], rows[q] + inst_.products[a.agentOf[j]][j]->mdp.numStates);
  }
  if (stats) {
    stats->evaluateJobs += static_cast<long>(m) * K;
    for (int q = 0; q < m; ++q)
      for (int k = 0; k < K; ++k)
        stats->evaluateStateBackups += static_cast<double>(esw[static_cast<size_t>(q) * K + k]) *
                                       inst_.products[a.agentOf[cols[q]]][cols[q]]->mdp.numStates;
    stats->evaluateSeconds += seconds(t0);
  }
}

// ---- one process per GPU: this rank's shard + an allgather ------------------------------
SupportingPoint shardedSupportingPoint(Shard& shard, int world, const Exchange& exchange, const Vec& w,
                                       QueryStats* stats) {
  const MorapInstance& inst = shard.instance();
  const int n = inst.n, K = inst.objectives;
  if (static_cast<int>(w.size()) != K * n) fail(Errc::DimensionMismatch, "weight vector must have one entry per objective");
  const int pairs = n * n;
  std::vector<double> send(2 * static_cast<size_t>(pairs)), recv(static_cast<size_t>(world) * 2 * pairs);
  shard.optimize(w, send.data(), send.data() + pairs, stats);
  exchange(send.data(), 2 * pairs, recv.data());
  Mat c(n, n);
  combine(world, pairs, recv.data(), c.a.data(), "weighted optimization failed");
  const auto t1 = std::chrono::steady_clock::now();
  SupportingPoint out;
  out.assignment = maxAssignment(c);
  if (stats) stats->hostSeconds += seconds(t1);
  out.schedulers.resize(static_cast<size_t>(n));
  const int kn = K * n;
  send.assign(2 * static_cast<size_t>(kn), 0.0);
  recv.assign(static_cast<size_t>(world) * 2 * kn, 0.0);
  shard.evaluate(out.assignment, send.data(), send.data() + kn, out.schedulers, stats);
  exchange(send.data(), 2 * kn, recv.data());
  out.r.assign(static_cast<size_t>(kn), 0.0);
  combine(world, kn, recv.data(), out.r.data(), "evaluation failed");
  return out;
}

ParetoResult paretoPointSharded(Shard& shard, int world, const Exchange& exchange, const Vec& thresholds,
                                const NormMatrix& norm, double eps, int iterationCap, QueryStats* stats) {
  return runParetoCore(expandThresholds(shard.instance(), thresholds), norm, eps, iterationCap, false, nullptr,
                       [&](const Vec& w) { return shardedSupportingPoint(shard, world, exchange, w, stats); });
}

// ---- one process, several GPUs: one host thread per device ------------------------------
SupportingPoint multiSupportingPoint(const std::vector<Shard*>& shards, const Vec& w, QueryStats* stats) {
  if (shards.empty()) fail(Errc::InvalidConfig, "no shards");
  const MorapInstance& inst = shards[0]->instance();
  const int n = inst.n, K = inst.objectives, world = static_cast<int>(shards.size());
  if (static_cast<int>(w.size()) != K * n) fail(Errc::DimensionMismatch, "weight vector must have one entry per objective");
  const int pairs = n * n, kn = K * n;
  std::vector<double> recv(static_cast<size_t>(world) * 2 * pairs);
  std::vector<QueryStats> part(static_cast<size_t>(world));
  std::vector<std::exception_ptr> err(static_cast<size_t>(world));
  auto fan = [&](auto&& step) {  // step(shard index) on one thread per device
    std::vector<std::thread> pool;
    for (int r = 1; r < world; ++r)
      pool.emplace_back([&, r] {
        try {
          step(r);
        } catch (...) {
          err[r] = std::current_exception();
        }
      });
    try {
      step(0);
    } catch (...) {
      err[0] = std::current_exception();
    }
    for (auto& t : pool) t.join();
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
  };
  fan([&](int r) {
    double* s = recv.data() + static_cast<size_t>(r) * 2 * pairs;
    shards[r]->optimize(w, s, s + pairs, stats ? &part[r] : nullptr);
  });
  Mat c(n, n);
  combine(world, pairs, recv.data(), c.a.data(), "weighted optimization failed");
  const auto t1 = std::chrono::steady_clock::now();
  SupportingPoint out;
  out.assignment = maxAssignment(c);
  const double host = seconds(t1);
  std::vector<std::vector<Scheduler>> sched(static_cast<size_t>(world), std::vector<Scheduler>(static_cast<size_t>(n)));
  recv.assign(static_cast<size_t>(world) * 2 * kn, 0.0);
  fan([&](int r) {
    double* s = recv.data() + static_cast<size_t>(r) * 2 * kn;
    shards[r]->evaluate(out.assignment, s, s + kn, sched[r], stats ? &part[r] : nullptr);
  });
  out.r.assign(static_cast<size_t>(kn), 0.0);
  combine(world, kn, recv.data(), out.r.data(), "evaluation failed");
  out.schedulers.resize(static_cast<size_t>(n));
  for (int r = 0; r < world; ++r)
    for (int j = 0; j < n; ++j)
      if (!sched[r][j].rows.empty()) out.schedulers[j] = std::move(sched[r][j]);
  if (stats) {  // work summed over the devices, time as the slowest device
    double opt = 0, ev = 0;
    for (const QueryStats& q : part) {
      stats->optimizeJobs += q.optimizeJobs;
      stats->optimizeBackups += q.optimizeBackups;
      stats->evaluateJobs += q.evaluateJobs;
      stats->evaluateStateBackups += q.evaluateStateBackups;
      opt = std::max(opt, q.optimizeSeconds);
      ev = std::max(ev, q.evaluateSeconds);
    }
    stats->optimizeSeconds += opt;
    stats->evaluateSeconds += ev;
    stats->hostSeconds += host;
  }
  return out;
}

ParetoResult paretoPointMulti(const std::vector<Shard*>& shards, const Vec& thresholds, const NormMatrix& norm,
                              double eps, int iterationCap, QueryStats* stats) {
  if (shards.empty()) fail(Errc::InvalidConfig, "no shards");
  return runParetoCore(expandThresholds(shards[0]->instance(), thresholds), norm, eps, iterationCap, false, nullptr,
                       [&](const Vec& w) { return multiSupportingPoint(shards, w, stats); });
}

}  // namespace morap
