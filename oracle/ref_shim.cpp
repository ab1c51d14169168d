// TEST INFRASTRUCTURE ONLY -- the reference checker, never the product path.
//
// Thin extern "C" shim over the UNMODIFIED reference headers in
// /root/reference/proj/include (header-only C++20). Built by oracle/Makefile
// into oracle/_ref/libmorap_ref.so. Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline leg and --impl reference) may load it.
//
// Every entry calls the reference's own functions:
//   generateInstance        warehouse.hpp:176
//   buildInstance           instance.hpp:42
//   optimalSchedulerOn      numerics.hpp:74
//   evaluateSchedulerOn     numerics.hpp:130
//   weightedReward          numerics.hpp:224
//   runBatch                engine.hpp:370
//   supportingPoint         solver.hpp:103
//   paretoPoint/verifyOnly  solver.hpp:281/289
//   synthesize              solver.hpp:299
//   maxAssignment           assignment.hpp:54
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>

#include "morap/assignment.hpp"
#include "morap/centralised.hpp"
#include "morap/engine.hpp"
#include "morap/geometry.hpp"
#include "morap/instance.hpp"
#include "morap/numerics.hpp"
#include "morap/solver.hpp"
#include "morap/warehouse.hpp"

using namespace morap;

namespace {

thread_local std::string g_err;

int code_of(const Error& e) { return static_cast<int>(e.code()) + 1; }

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return code_of(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1000;
  }
}

struct Handle {
  MorapInstance inst;
  std::unique_ptr<CentralisedMdp> cent;  // built on first use (ref_centralised_*)
};

const CentralisedMdp& centralised_of(void* p, long guard) {
  Handle* h = static_cast<Handle*>(p);
  if (!h->cent) h->cent = std::make_unique<CentralisedMdp>(buildCentralised(h->inst, guard));
  return *h->cent;
}

// Scheduler fingerprint (test-only): FNV-style over 32-bit rows, same as capi.cpp rowsHash.
uint64_t fnv_rows(const Scheduler& mu) {
  uint64_t h = 1469598103934665603ull;
  for (const auto& c : mu.choice) {
    const uint32_t r = static_cast<uint32_t>(c.empty() ? -1 : c[0].first);
    h = (h ^ r) * 1099511628211ull;
  }
  return h;
}

Mdp csr_to_mdp(int S, int R, int nnz, int initial, const int* rowOffset, const int* trnOffset,
               const int* succ, const double* prob) {
  Mdp m;
  m.numStates = S;
  m.initial = initial;
  m.rowOffset.assign(rowOffset, rowOffset + S + 1);
  m.trnOffset.assign(trnOffset, trnOffset + R + 1);
  m.succ.assign(succ, succ + nnz);
  m.prob.assign(prob, prob + nnz);
  m.labels.assign(S, {});
  m.actionName.assign(R, "");
  return m;
}

// Report of one Pareto run: resultToJson plus converged, thresholds, lambdaStar, the
// per-iteration tUp/tDown/scheduler hashes and the synthesis marginals.
Json pareto_report(const ParetoResult& res) {
  Json j;
  std::unique_ptr<SynthesisResult> syn;
  try {
    if (res.converged) syn = std::make_unique<SynthesisResult>(synthesize(res));
  } catch (const Error& e) {
    j["synthesisError"] = static_cast<int>(e.code()) + 1;
  }
  j = resultToJson(res, syn.get());
  j["converged"] = res.converged;
  j["thresholds"] = res.thresholds;
  j["lambdaStar"] = res.lambdaStar;
  Json recs = Json::array();
  for (const auto& rec : res.iterations) {
    Json it;
    it["tUp"] = rec.tUp;
    it["tDown"] = rec.tDown;
    Json hs = Json::array();
    for (const auto& mu : rec.schedulers) hs.push_back(std::to_string(fnv_rows(mu)));
    it["schedulerHash"] = hs;
    recs.push_back(std::move(it));
  }
  j["records"] = recs;
  if (syn) {
    Json mg = Json::array();
    for (int a = 0; a < syn->marginal.rows; ++a) {
      Json row = Json::array();
      for (int b = 0; b < syn->marginal.cols; ++b) row.push_back(syn->marginal(a, b));
      mg.push_back(row);
    }
    j["marginal"] = mg;
  }
  return j;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Instance from the reference's instance-file JSON ({"agents": [...], "tasks": [...]})
// following cli.hpp:93-117 (inline agents and LTL strings only).
void* ref_instance_from_json(const char* text) {
  Handle* h = nullptr;
  int rc = guarded([&] {
    Json j = Json::parse(text);
    std::vector<Mdp> agents;
    std::vector<RewardStructure> costs;
    for (const auto& a : j.at("agents")) {
      auto [m, c] = mdpFromJson(a);
      agents.push_back(std::move(m));
      costs.push_back(std::move(c));
    }
    std::vector<Dfa> tasks;
    for (const auto& t : j.at("tasks")) tasks.push_back(insertPreSinks(formulaToDfa(parseCoSafe(t.get<std::string>()))));
    h = new Handle{buildInstance(std::move(agents), std::move(costs), std::move(tasks))};
  });
  return rc == 0 ? h : nullptr;
}

void* ref_instance_warehouse(const char* config_json) {
  Handle* h = nullptr;
  int rc = guarded([&] {
    WarehouseConfig cfg = warehouseConfigFromJson(Json::parse(config_json));
    h = new Handle{generateInstance(cfg)};
  });
  return rc == 0 ? h : nullptr;
}

void ref_instance_free(void* p) { delete static_cast<Handle*>(p); }

int ref_instance_n(void* p) { return static_cast<Handle*>(p)->inst.n; }
int ref_instance_real_tasks(void* p) { return static_cast<Handle*>(p)->inst.realTasks; }
int ref_instance_distinct(void* p) { return static_cast<Handle*>(p)->inst.distinctProducts; }

// dims = {S, R, nnz, initial, rewardFinite}
int ref_product_dims(void* p, int i, int j, int64_t* dims, uint64_t* hash) {
  return guarded([&] {
    const ProductMdp& pr = *static_cast<Handle*>(p)->inst.products.at(i).at(j);
    dims[0] = pr.mdp.numStates;
    dims[1] = pr.mdp.numActions();
    dims[2] = static_cast<int64_t>(pr.mdp.succ.size());
    dims[3] = pr.mdp.initial;
    dims[4] = pr.rewardFinite ? 1 : 0;
    *hash = pr.structuralHash;
  });
}

// Identity of the shared product object (dedup check, instance.hpp:70-89).
int64_t ref_product_slot(void* p, int i, int j) {
  const auto& inst = static_cast<Handle*>(p)->inst;
  const ProductMdp* target = inst.products.at(i).at(j).get();
  int64_t slot = 0;
  for (int a = 0; a < inst.n; ++a)
    for (int b = 0; b < inst.n; ++b) {
      if (inst.products[a][b].get() == target) return slot;
      ++slot;
    }
  return -1;
}

int ref_product_export(void* p, int i, int j, int* rowOffset, int* trnOffset, int* succ, double* prob,
                       double* cost, double* success, unsigned char* done, unsigned char* accept) {
  return guarded([&] {
    const ProductMdp& pr = *static_cast<Handle*>(p)->inst.products.at(i).at(j);
    const Mdp& m = pr.mdp;
    std::memcpy(rowOffset, m.rowOffset.data(), m.rowOffset.size() * sizeof(int));
    std::memcpy(trnOffset, m.trnOffset.data(), m.trnOffset.size() * sizeof(int));
    std::memcpy(succ, m.succ.data(), m.succ.size() * sizeof(int));
    std::memcpy(prob, m.prob.data(), m.prob.size() * sizeof(double));
    std::memcpy(cost, pr.cost.data(), pr.cost.size() * sizeof(double));
    std::memcpy(success, pr.success.data(), pr.success.size() * sizeof(double));
    for (int s = 0; s < m.numStates; ++s) {
      done[s] = pr.done[s] ? 1 : 0;
      accept[s] = pr.accept[s] ? 1 : 0;
    }
  });
}

// optimalScheduler on product (i,j) with rho = weightedReward({cost, success}, {wc, ws})
// exactly as supportingPoint builds it (solver.hpp:118-128).
int ref_optimize(void* p, int i, int j, double wc, double ws, double eps, int cap, double* values,
                 int* policy, int* sweeps, double* residual, double* value) {
  return guarded([&] {
    const ProductMdp& pr = *static_cast<Handle*>(p)->inst.products.at(i).at(j);
    RewardStructure rho = weightedReward({&pr.cost, &pr.success}, {wc, ws});
    OptimizeResult r = optimalScheduler(pr, rho, eps, cap);
    std::memcpy(values, r.values.data(), r.values.size() * sizeof(double));
    for (size_t s = 0; s < r.policy.choice.size(); ++s) policy[s] = r.policy.choice[s][0].first;
    *sweeps = r.stats.sweeps;
    *residual = r.stats.residual;
    *value = r.value;
  });
}

// evaluateScheduler on product (i,j) with a deterministic policy; which: 0 cost, 1 success.
int ref_evaluate(void* p, int i, int j, const int* policy, int which, double eps, int cap, double* values,
                 int* sweeps, double* residual, double* value) {
  return guarded([&] {
    const ProductMdp& pr = *static_cast<Handle*>(p)->inst.products.at(i).at(j);
    std::vector<int> rows(policy, policy + pr.mdp.numStates);
    EvaluateResult r = evaluateScheduler(pr, makeDeterministic(rows), which == 0 ? pr.cost : pr.success, eps, cap);
    std::memcpy(values, r.values.data(), r.values.size() * sizeof(double));
    *sweeps = r.stats.sweeps;
    *residual = r.stats.residual;
    *value = r.value;
  });
}

// Raw-CSR entry points (random models, tests/golden generation).
int ref_optimize_csr(int S, int R, int nnz, int initial, const int* rowOffset, const int* trnOffset,
                     const int* succ, const double* prob, const unsigned char* done, int rewardFinite,
                     const double* rho, double eps, int cap, double* values, int* policy, int* sweeps,
                     double* residual) {
  return guarded([&] {
    Mdp m = csr_to_mdp(S, R, nnz, initial, rowOffset, trnOffset, succ, prob);
    std::vector<char> d(done, done + S);
    RewardStructure r(rho, rho + R);
    OptimizeResult o = optimalSchedulerOn(m, d, rewardFinite != 0, r, eps, cap);
    std::memcpy(values, o.values.data(), S * sizeof(double));
    for (int s = 0; s < S; ++s) policy[s] = o.policy.choice[s][0].first;
    *sweeps = o.stats.sweeps;
    *residual = o.stats.residual;
  });
}

int ref_evaluate_csr(int S, int R, int nnz, int initial, const int* rowOffset, const int* trnOffset,
                     const int* succ, const double* prob, const unsigned char* done, const int* policy,
                     const double* rho, double eps, int cap, double* values, int* sweeps, double* residual) {
  return guarded([&] {
    Mdp m = csr_to_mdp(S, R, nnz, initial, rowOffset, trnOffset, succ, prob);
    std::vector<char> d(done, done + S);
    RewardStructure r(rho, rho + R);
    std::vector<int> rows(policy, policy + S);
    EvaluateResult o = evaluateSchedulerOn(m, d, makeDeterministic(rows), r, eps, cap);
    std::memcpy(values, o.values.data(), S * sizeof(double));
    *sweeps = o.stats.sweeps;
    *residual = o.stats.residual;
  });
}

int ref_reward_finite_csr(int S, int R, int nnz, const int* rowOffset, const int* trnOffset, const int* succ,
                          const double* prob, const unsigned char* done) {
  Mdp m = csr_to_mdp(S, R, nnz, 0, rowOffset, trnOffset, succ, prob);
  std::vector<char> d(done, done + S);
  return checkRewardFinite(m, d) ? 1 : 0;
}

int ref_max_assignment(int n, const double* c, int* agentOf) {
  return guarded([&] {
    Mat m(n, n);
    for (int k = 0; k < n * n; ++k) m.a[k] = c[k];
    Assignment a = maxAssignment(m);
    for (int j = 0; j < n; ++j) agentOf[j] = a.agentOf[j];
  });
}

// Optimize phase of supportingPoint (solver.hpp:108-133) through the reference engine,
// timed: returns wall seconds and the nnz backups performed (sum sweeps * nnz).
int ref_optimize_phase(void* p, const double* w, int workers, double* seconds, double* backups) {
  return guarded([&] {
    const MorapInstance& inst = static_cast<Handle*>(p)->inst;
    const int n = inst.n;
    using Key = std::tuple<uintptr_t, uint64_t, uint64_t>;
    std::map<Key, long> seen;
    std::vector<Job> jobs;
    std::vector<long> nnzOf;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const auto& m = inst.products[i][j];
        Key k{reinterpret_cast<uintptr_t>(m.get()), solverdetail::doubleBits(w[i]), solverdetail::doubleBits(w[n + j])};
        if (seen.count(k)) continue;
        Job job;
        job.id = static_cast<long>(jobs.size());
        job.kind = JobKind::Optimize;
        job.model = m;
        job.reward = weightedReward({&m->cost, &m->success}, {w[i], w[n + j]});
        seen.emplace(k, job.id);
        nnzOf.push_back(static_cast<long>(m->mdp.succ.size()));
        jobs.push_back(std::move(job));
      }
    PoolConfig pool = configurePool(workers > 0 ? workers : defaultWorkerCount());
    auto t0 = std::chrono::steady_clock::now();
    auto res = runBatch(std::move(jobs), pool);
    auto t1 = std::chrono::steady_clock::now();
    double total = 0.0;
    for (auto& [id, r] : res) {
      if (!r.ok) solverdetail::rethrowJobFailure(r, "optimize");
      total += static_cast<double>(r.stats.sweeps) * static_cast<double>(nnzOf[id]);
    }
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    *backups = total;
  });
}

// Work of a recorded Pareto query, counted on the reference engine (untimed): for every
// iteration, the supportingPoint jobs (solver.hpp:110-171) at that iteration's w and
// assignment through runBatch; optimize backups = sweeps x nnz, evaluate state backups =
// sweeps x states (the units bench.py's `value` counts). w: iters x 2n, agentOf: iters x n.
int ref_query_backups(void* p, const double* wAll, const int* agentOfAll, int iters, int workers, double* optBackups,
                      double* evalBackups) {
  return guarded([&] {
    const MorapInstance& inst = static_cast<Handle*>(p)->inst;
    const int n = inst.n;
    PoolConfig pool = configurePool(workers > 0 ? workers : defaultWorkerCount());
    double ob = 0.0, eb = 0.0;
    for (int it = 0; it < iters; ++it) {
      const double* w = wAll + static_cast<size_t>(it) * 2 * n;
      using Key = std::tuple<uintptr_t, uint64_t, uint64_t>;
      std::map<Key, long> jobOf;
      std::vector<Job> jobs;
      std::vector<double> nnzOf;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          const auto& m = inst.products[i][j];
          Key k{reinterpret_cast<uintptr_t>(m.get()), solverdetail::doubleBits(w[i]),
                solverdetail::doubleBits(w[n + j])};
          if (jobOf.count(k)) continue;
          Job job;
          job.id = static_cast<long>(jobs.size());
          job.kind = JobKind::Optimize;
          job.model = m;
          job.reward = weightedReward({&m->cost, &m->success}, {w[i], w[n + j]});
          jobOf.emplace(k, job.id);
          nnzOf.push_back(static_cast<double>(m->mdp.succ.size()));
          jobs.push_back(std::move(job));
        }
      auto opt = runBatch(std::move(jobs), pool);
      for (auto& [id, r] : opt) {
        if (!r.ok) solverdetail::rethrowJobFailure(r, "optimize");
        ob += static_cast<double>(r.stats.sweeps) * nnzOf[id];
      }
      std::vector<Job> ev;
      std::vector<double> statesOf;
      for (int j = 0; j < n; ++j) {
        const int i = agentOfAll[static_cast<size_t>(it) * n + j];
        const auto& m = inst.products[i][j];
        Key k{reinterpret_cast<uintptr_t>(m.get()), solverdetail::doubleBits(w[i]), solverdetail::doubleBits(w[n + j])};
        for (int which = 0; which < 2; ++which) {
          Job job;
          job.id = 2 * j + which;
          job.kind = JobKind::Evaluate;
          job.model = m;
          job.scheduler = opt.at(jobOf.at(k)).policy;
          job.reward = which ? m->success : m->cost;
          ev.push_back(std::move(job));
        }
        statesOf.push_back(static_cast<double>(m->mdp.numStates));
      }
      auto er = runBatch(std::move(ev), pool);
      for (auto& [id, r] : er) {
        if (!r.ok) solverdetail::rethrowJobFailure(r, "evaluate");
        eb += static_cast<double>(r.stats.sweeps) * statesOf[id / 2];
      }
    }
    *optBackups = ob;
    *evalBackups = eb;
  });
}

// Full supportingPoint (solver.hpp:103) on the reference engine.
int ref_supporting_point(void* p, const double* w, int workers, double* r_out, int* agentOf, double* seconds) {
  return guarded([&] {
    const MorapInstance& inst = static_cast<Handle*>(p)->inst;
    Vec wv(w, w + 2 * inst.n);
    PoolConfig pool = configurePool(workers > 0 ? workers : defaultWorkerCount());
    auto t0 = std::chrono::steady_clock::now();
    SupportingPoint sp = supportingPoint(inst, wv, pool);
    auto t1 = std::chrono::steady_clock::now();
    for (int k = 0; k < 2 * inst.n; ++k) r_out[k] = sp.r[k];
    for (int j = 0; j < inst.n; ++j) agentOf[j] = sp.assignment.agentOf[j];
    *seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

// paretoPoint / verifyOnly (solver.hpp:281-294) with the identity norm (or `norm`, row-major
// 2n x 2n, when non-null). Writes a JSON report: resultToJson plus converged, thresholds,
// lambdaStar, per-iteration tUp/tDown/scheduler hashes and the synthesis marginals.
int ref_pareto(void* p, const double* thresholds, int nt, const double* norm, double eps, int workers,
               int iterCap, int verify, char* out, int outlen, double* seconds) {
  return guarded([&] {
    const MorapInstance& inst = static_cast<Handle*>(p)->inst;
    const int d = 2 * inst.n;
    Mat nm(d, d, 0.0);
    if (norm)
      for (int k = 0; k < d * d; ++k) nm.a[k] = norm[k];
    else
      for (int k = 0; k < d; ++k) nm(k, k) = 1.0;
    NormMatrix M(nm);
    Vec t(thresholds, thresholds + nt);
    PoolConfig pool = configurePool(workers > 0 ? workers : defaultWorkerCount());
    Json j;
    auto t0 = std::chrono::steady_clock::now();
    if (verify) {
      bool verdict = verifyOnly(inst, t, M, eps, pool, iterCap);
      j["verdict"] = verdict;
    } else {
      ParetoResult res = paretoPoint(inst, t, M, eps, pool, iterCap);
      auto t1 = std::chrono::steady_clock::now();
      *seconds = std::chrono::duration<double>(t1 - t0).count();
      j = pareto_report(res);
    }
    if (verify) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::string s = j.dump();
    if (static_cast<int>(s.size()) + 1 > outlen) fail(Errc::Io, "output buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

// runParetoCore (solver.hpp:192-266) over an external supporting-point source: the same
// callback signature as morap_pareto_core (include/morap.h), so the restated sandwich loop
// and geometry QPs can be compared with the reference's at any dimension (identity norm
// when `norm` is null).
typedef int (*ref_query_fn)(void* user, const double* w, int d, double* r_out, int32_t* agent_of_out, int n);
int ref_pareto_core(const double* thresholds, int d, int n, const double* norm, double eps, int iterCap, int verify,
                    ref_query_fn query, void* user, char* out, int outlen) {
  return guarded([&] {
    Mat nm(d, d, 0.0);
    if (norm)
      for (int k = 0; k < d * d; ++k) nm.a[k] = norm[k];
    else
      for (int k = 0; k < d; ++k) nm(k, k) = 1.0;
    bool verdict = false;
    auto q = [&](const Vec& w) {
      SupportingPoint sp;
      sp.r.assign(d, 0.0);
      sp.assignment.agentOf.assign(n, 0);
      std::vector<int32_t> a(n, 0);
      if (query(user, w.data(), d, sp.r.data(), a.data(), n) != 0) fail(Errc::SolverFailure, "query callback failed");
      for (int j = 0; j < n; ++j) sp.assignment.agentOf[j] = a[j];
      sp.schedulers.resize(n);
      return sp;
    };
    ParetoResult res = solverdetail::runParetoCore(Vec(thresholds, thresholds + d), NormMatrix(nm), eps, iterCap,
                                                   verify != 0, verify ? &verdict : nullptr, q);
    Json j = pareto_report(res);
    if (verify) j["verdict"] = verdict;
    std::string s = j.dump();
    if (static_cast<int>(s.size()) + 1 > outlen) fail(Errc::Io, "output buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

int ref_hardware_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

// buildCentralised (centralised.hpp:54): dims[6] = {S, R, nnz, initial, rewardFinite, 2n}
int ref_centralised_dims(void* p, long guard, int64_t* dims) {
  return guarded([&] {
    const CentralisedMdp& c = centralised_of(p, guard);
    const int64_t v[6] = {c.mdp.numStates, c.mdp.numActions(), static_cast<int64_t>(c.mdp.succ.size()),
                          c.mdp.initial, c.rewardFinite ? 1 : 0, static_cast<int64_t>(c.rewards.size())};
    std::memcpy(dims, v, sizeof v);
  });
}

int ref_centralised_export(void* p, long guard, int* rowOffset, int* trnOffset, int* succ, double* prob,
                           unsigned char* done, double* rewards /* 2n x R, row-major */) {
  return guarded([&] {
    const CentralisedMdp& c = centralised_of(p, guard);
    std::memcpy(rowOffset, c.mdp.rowOffset.data(), sizeof(int) * c.mdp.rowOffset.size());
    std::memcpy(trnOffset, c.mdp.trnOffset.data(), sizeof(int) * c.mdp.trnOffset.size());
    std::memcpy(succ, c.mdp.succ.data(), sizeof(int) * c.mdp.succ.size());
    std::memcpy(prob, c.mdp.prob.data(), sizeof(double) * c.mdp.prob.size());
    for (size_t s = 0; s < c.done.size(); ++s) done[s] = c.done[s] ? 1 : 0;
    const size_t R = static_cast<size_t>(c.mdp.numActions());
    for (size_t k = 0; k < c.rewards.size(); ++k) std::memcpy(rewards + k * R, c.rewards[k].data(), sizeof(double) * R);
  });
}

// centralisedParetoPoint (centralised.hpp:216) with the identity norm; same JSON report as ref_pareto
int ref_centralised_pareto(void* p, long guard, const double* thresholds, int nt, double eps, int iterCap, char* out,
                           int outlen, double* seconds) {
  return guarded([&] {
    const CentralisedMdp& c = centralised_of(p, guard);
    const int d = static_cast<int>(c.rewards.size());
    Mat nm(d, d, 0.0);
    for (int k = 0; k < d; ++k) nm(k, k) = 1.0;
    auto t0 = std::chrono::steady_clock::now();
    ParetoResult res = centralisedParetoPoint(c, Vec(thresholds, thresholds + nt), NormMatrix(nm), eps, iterCap);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::string s = pareto_report(res).dump();
    if (static_cast<int>(s.size()) + 1 > outlen) fail(Errc::Io, "output buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

}  // extern "C"
