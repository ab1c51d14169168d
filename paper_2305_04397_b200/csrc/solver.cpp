// Pareto-point query with GPU supporting points (reference: solver.hpp).
//
// supportingPoint is Algorithm 2: one weighted optimize job per distinct
// (product, per-objective weights) -- deduplicated on the weight BITS exactly like
// solver.hpp:110-131 -- all in one device batch; the n x n matrix of initial-state values
// goes to the host Hungarian step; the n assigned pairs are then re-evaluated under all K
// objectives in one fused multi-RHS device batch, using the optimize jobs' policies that
// never left the GPU. runParetoCore is Algorithm 1 (the sandwich loop) on the host.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <fstream>
#include <tuple>

#include "morap.hpp"
#include "morap_cuda.h"

namespace morap {

namespace {

uint64_t bitsOf(double v) {
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

}  // namespace

SupportingPoint supportingPoint(const MorapInstance& inst, const Vec& w, GpuBackend& gpu, QueryStats* stats) {
  const int n = inst.n, K = inst.objectives;
  if (static_cast<int>(w.size()) != K * n) fail(Errc::DimensionMismatch, "weight vector must have one entry per objective");
  double l1 = 0.0;
  for (double v : w) {
    if (!std::isfinite(v)) fail(Errc::InvalidConfig, "weight vector entries must be finite");
    l1 += std::fabs(v);
  }
  if (std::fabs(l1 - 1.0) > 1e-6) fail(Errc::InvalidConfig, "weight vector must have unit 1-norm");
  gpu.uploadInstance(inst);
  morap_ctx* ctx = gpu.ctx();
  auto coord = [&](int k, int i, int j) { return k < K - 1 ? k * n + i : (K - 1) * n + j; };

  // ---- optimize batch: one job per distinct (model, weight bits) -------------------------
  auto t0 = std::chrono::steady_clock::now();
  std::map<std::vector<uint64_t>, int> jobOf;
  std::vector<int> jobIJ(static_cast<size_t>(n) * n);
  std::vector<int32_t> models;
  std::vector<double> weights;
  std::vector<long> nnzOf;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const ProductMdp* p = inst.products[i][j].get();
      std::vector<uint64_t> key{reinterpret_cast<uintptr_t>(p)};
      for (int k = 0; k < K; ++k) key.push_back(bitsOf(w[coord(k, i, j)]));
      auto [it, fresh] = jobOf.emplace(std::move(key), static_cast<int>(models.size()));
      if (fresh) {
        models.push_back(gpu.modelId(p));
        for (int k = 0; k < K; ++k) weights.push_back(w[coord(k, i, j)]);
        nnzOf.push_back(static_cast<long>(productNnz(*p)));
      }
      jobIJ[static_cast<size_t>(i) * n + j] = it->second;
    }
  const int nj = static_cast<int>(models.size());
  std::vector<double> value(nj), resid(nj);
  std::vector<int32_t> sweeps(nj), status(nj);
  ck(ctx, morap_cuda_optimize(ctx, nj, models.data(), weights.data(), K, 1e-6, 100000, value.data(), sweeps.data(),
                              resid.data(), status.data()),
     "optimize batch");
  Mat c(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const int q = jobIJ[static_cast<size_t>(i) * n + j];
      if (status[q] != MORAP_OK) jobFailed(status[q], "weighted optimization failed");
      c(i, j) = value[q];
    }
  if (stats) {
    stats->optimizeJobs += nj;
    for (int q = 0; q < nj; ++q) stats->optimizeBackups += static_cast<double>(sweeps[q]) * nnzOf[q];
    stats->optimizeSeconds += seconds(t0);
  }

  // ---- host assignment -------------------------------------------------------------------
  auto t1 = std::chrono::steady_clock::now();
  SupportingPoint out;
  out.assignment = maxAssignment(c);
  if (stats) stats->hostSeconds += seconds(t1);

  // ---- fused evaluation of the n assigned pairs under all K objectives -------------------
  auto t2 = std::chrono::steady_clock::now();
  std::vector<int32_t> evalJobs(static_cast<size_t>(n)), objectives(static_cast<size_t>(K));
  for (int j = 0; j < n; ++j) evalJobs[j] = jobIJ[static_cast<size_t>(out.assignment.agentOf[j]) * n + j];
  for (int k = 0; k < K; ++k) objectives[k] = k;
  std::vector<double> ev(static_cast<size_t>(n) * K), eres(static_cast<size_t>(n) * K);
  std::vector<int32_t> esw(static_cast<size_t>(n) * K), est(static_cast<size_t>(n) * K);
  ck(ctx, morap_cuda_evaluate_optimized(ctx, n, evalJobs.data(), K, objectives.data(), 1e-6, 100000, ev.data(),
                                        esw.data(), eres.data(), est.data()),
     "evaluate batch");
  const auto t2b = std::chrono::steady_clock::now();
  if (stats) stats->evaluateSweepSeconds += seconds(t2);
  out.r.assign(static_cast<size_t>(K) * n, 0.0);
  out.schedulers.resize(static_cast<size_t>(n));
  for (int j = 0; j < n; ++j) {
    const int i = out.assignment.agentOf[j];
    for (int k = 0; k < K; ++k) {
      const int32_t st = est[static_cast<size_t>(j) * K + k];
      if (st != MORAP_OK) jobFailed(st, k == K - 1 ? "success evaluation failed" : "cost evaluation failed");
    }
    for (int k = 0; k < K; ++k) out.r[coord(k, i, j)] = ev[static_cast<size_t>(j) * K + k];
  }
  // the n schedulers of the assigned pairs (IterationRecord::schedulers, solver.hpp:38-45),
  // copied out of the pinned staging area on the host threads
  const auto t3 = std::chrono::steady_clock::now();
  std::vector<const int32_t*> rowsIn(static_cast<size_t>(n));
  ck(ctx, morap_cuda_policy_views(ctx, n, evalJobs.data(), rowsIn.data()), "fetch policies");
  const auto t3b = std::chrono::steady_clock::now();
  // (allocated here, on the calling thread: its heap keeps the pages of earlier queries'
  // schedulers, so the copies do not fault; pool threads would each allocate in their own
  // malloc arena)
  for (int j = 0; j < n; ++j)
    out.schedulers[j].rows.resize(static_cast<size_t>(inst.products[out.assignment.agentOf[j]][j]->mdp.numStates));
  parallelFor(n, [&](int j) {
    std::memcpy(out.schedulers[j].rows.data(), rowsIn[j], sizeof(int32_t) * out.schedulers[j].rows.size());
  });
  if (std::getenv("MORAP_TRACE"))
    std::fprintf(stderr, "[morap] supportingPoint: optimize %.3f ms (%d jobs), assign %.3f ms, evaluate %.3f ms "
                         "(device batch %.3f ms), policies %.3f ms (wait %.3f ms)\n",
                 1e3 * std::chrono::duration<double>(t1 - t0).count(), nj,
                 1e3 * std::chrono::duration<double>(t2 - t1).count(),
                 1e3 * std::chrono::duration<double>(t3 - t2).count(),
                 1e3 * std::chrono::duration<double>(t2b - t2).count(), 1e3 * seconds(t3),
                 1e3 * std::chrono::duration<double>(t3b - t3).count());
  if (stats) {
    stats->evaluateJobs += static_cast<long>(n) * K;
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < K; ++k)
        stats->evaluateStateBackups +=
            static_cast<double>(esw[static_cast<size_t>(j) * K + k]) *
            inst.products[out.assignment.agentOf[j]][j]->mdp.numStates;
    stats->evaluateSeconds += seconds(t2);
  }
  return out;
}

ParetoResult runParetoCore(Vec t, const NormMatrix& norm, double eps, int iterationCap, bool verifyMode, bool* verdict,
                           const QueryFn& query) {
  if (!(eps >= 0.0)) fail(Errc::InvalidConfig, "eps must be nonnegative");
  if (iterationCap < 1) fail(Errc::InvalidConfig, "iteration cap must be positive");
  if (norm.dim() != static_cast<int>(t.size())) fail(Errc::DimensionMismatch, "norm matrix must match the objective count");
  ParetoResult res;
  res.eps = eps;
  res.thresholds = std::move(t);
  const Vec& thr = res.thresholds;
  res.tDown = thr;
  Vec w(thr.size(), 0.0);
  w[0] = 1.0;
  auto minus = [](const Vec& a, const Vec& b) {
    Vec d(a);
    for (size_t k = 0; k < d.size(); ++k) d[k] -= b[k];
    return d;
  };
  const bool trace = std::getenv("MORAP_TRACE") != nullptr;
  for (int iter = 0; iter < iterationCap; ++iter) {
    if (!res.phi.points.empty()) {
      const auto tq = std::chrono::steady_clock::now();
      ProjectionResult low = projectToLowerApprox(thr, res.phi, norm);
      if (trace)
        std::fprintf(stderr, "[morap] iteration %d: lower projection %.3f ms, gap %.6g\n", iter, 1e3 * seconds(tq),
                     normDistance(norm, minus(res.tDown, low.x)));
      res.tUp = low.x;
      res.lambdaStar = low.lambda;
      if (normDistance(norm, minus(res.tDown, res.tUp)) <= eps) {
        res.converged = true;
        break;
      }
      try {
        w = weightVector(thr, res.tUp, norm);
      } catch (const Error& e) {
        if (e.code() != Errc::DegenerateDirection) throw;
        res.converged = true;  // t sits on its own projection: the gap is numerically zero
        break;
      }
    }
    SupportingPoint sp = query(w);
    res.phi.points.push_back(sp.r);
    res.lambda.cuts.push_back({w, sp.r});
    IterationRecord rec;
    rec.w = w;
    rec.r = sp.r;
    rec.assignment = sp.assignment;
    rec.schedulers = std::move(sp.schedulers);
    rec.tUp = res.tUp;
    if (dot(w, sp.r) < dot(w, res.tDown)) {
      if (verifyMode) {
        *verdict = false;
        rec.tDown = res.tDown;
        res.iterations.push_back(std::move(rec));
        return res;
      }
      const auto tq = std::chrono::steady_clock::now();
      res.tDown = projectToUpperApprox(thr, res.lambda, norm);
      if (trace) std::fprintf(stderr, "[morap] iteration %d: upper projection %.3f ms\n", iter, 1e3 * seconds(tq));
    }
    rec.tDown = res.tDown;
    res.iterations.push_back(std::move(rec));
  }
  if (!res.converged) {
    if (verifyMode) fail(Errc::NonConvergence, "verification hit the iteration cap without a verdict");
    res.feasible = false;
    return res;
  }
  res.feasible = normDistance(norm, minus(res.tDown, thr)) <= eps;
  if (verifyMode) *verdict = res.feasible;
  return res;
}

ParetoResult paretoPoint(const MorapInstance& inst, const Vec& thresholds, const NormMatrix& norm, double eps,
                         GpuBackend& gpu, int iterationCap, QueryStats* stats) {
  return runParetoCore(expandThresholds(inst, thresholds), norm, eps, iterationCap, false, nullptr,
                       [&](const Vec& w) { return supportingPoint(inst, w, gpu, stats); });
}

bool verifyOnly(const MorapInstance& inst, const Vec& thresholds, const NormMatrix& norm, double eps, GpuBackend& gpu,
                int iterationCap) {
  bool verdict = false;
  runParetoCore(expandThresholds(inst, thresholds), norm, eps, iterationCap, true, &verdict,
                [&](const Vec& w) { return supportingPoint(inst, w, gpu, nullptr); });
  return verdict;
}

SynthesisResult synthesize(const ParetoResult& res) {
  if (!res.converged) fail(Errc::NoCertificate, "synthesis requires a converged result");
  if (res.iterations.empty() || res.tUp.empty() || res.lambdaStar.empty())
    fail(Errc::NoCertificate, "synthesis requires at least one lower projection");
  const size_t ell = res.iterations.size();
  if (res.lambdaStar.size() != ell || res.phi.points.size() != ell)
    fail(Errc::NoCertificate, "certificate does not cover all iterations");
  auto clampNormalise = [](Vec v) {
    double s = 0.0;
    for (double& x : v) s += (x = x < 0.0 ? 0.0 : x);
    if (s <= 0.0) fail(Errc::NoCertificate, "degenerate convex weights");
    for (double& x : v) x /= s;
    return v;
  };
  auto dominates = [&](const Vec& v, double slack) {
    Vec mix(res.tUp.size(), 0.0);
    for (size_t k = 0; k < ell; ++k)
      for (size_t d = 0; d < mix.size(); ++d) mix[d] += v[k] * res.phi.points[k][d];
    for (size_t d = 0; d < mix.size(); ++d)
      if (mix[d] < res.tUp[d] - slack) return false;
    return true;
  };
  Vec v = clampNormalise(res.lambdaStar);
  if (!dominates(v, 1e-9)) {
    const ProjectionResult again =
        projectToLowerApprox(res.tUp, res.phi, NormMatrix::identity(static_cast<int>(res.tUp.size())));
    v = clampNormalise(again.lambda);
    if (!dominates(v, 1e-6)) fail(Errc::NoCertificate, "no convex combination dominates tUp");
  }
  const int n = static_cast<int>(res.iterations.front().assignment.agentOf.size());
  SynthesisResult out;
  out.marginal = Mat(n, n);
  for (size_t k = 0; k < ell; ++k) {
    if (v[k] <= 0.0) continue;
    SynthesisTerm term{v[k], res.iterations[k].assignment, res.iterations[k].schedulers};
    for (int j = 0; j < n; ++j) out.marginal(term.assignment.agentOf[j], j) += v[k];
    out.terms.push_back(std::move(term));
  }
  if (!validateBistochastic(out.marginal, 1e-9, 1e-6)) fail(Errc::NoCertificate, "mixture marginals are not bistochastic");
  return out;
}

Json resultToJson(const ParetoResult& result, const SynthesisResult* synthesis) {
  Json j;
  j["feasible"] = result.feasible;
  j["tUp"] = result.tUp;
  j["tDown"] = result.tDown;
  Json its = Json::array();
  for (const IterationRecord& rec : result.iterations)
    its.push_back({{"w", rec.w}, {"r", rec.r}, {"assignment", rec.assignment.agentOf}});
  j["iterations"] = its;
  Json syn = Json::array();
  if (synthesis)
    for (const SynthesisTerm& t : synthesis->terms) syn.push_back({{"p", t.p}, {"assignment", t.assignment.agentOf}});
  j["synthesis"] = syn;
  return j;
}

MorapInstance instanceFromJson(const Json& j, const std::string& baseDir, const InstanceBuilder* build) {
  if (!j.is_object() || !j.contains("agents") || !j.contains("tasks"))
    fail(Errc::InvalidConfig, "instance file needs agents and tasks");
  auto readFile = [&](const std::string& rel) {
    std::ifstream in(baseDir + "/" + rel);
    if (!in) fail(Errc::Io, "cannot open " + baseDir + "/" + rel);
    try {
      return Json::parse(in);
    } catch (const Json::exception& e) {
      fail(Errc::Io, rel + ": " + e.what());
    }
  };
  std::vector<Mdp> agents;
  std::vector<RewardStructure> costs;
  for (const Json& a : j.at("agents")) {
    auto [m, c] = mdpFromJson(a.is_string() ? readFile(a.get<std::string>()) : a);
    agents.push_back(std::move(m));
    costs.push_back(std::move(c));
  }
  std::vector<Dfa> tasks;
  for (const Json& t : j.at("tasks")) {
    if (t.is_object()) {
      tasks.push_back(dfaFromJson(t));
      continue;
    }
    if (!t.is_string()) fail(Errc::InvalidConfig, "task entries must be strings or DFA objects");
    const std::string s = t.get<std::string>();
    if (s.size() > 5 && s.compare(s.size() - 5, 5, ".json") == 0) tasks.push_back(dfaFromJson(readFile(s)));
    else tasks.push_back(insertPreSinks(formulaToDfa(parseCoSafe(s))));
  }
  if (build) return (*build)(std::move(agents), std::move(costs), std::move(tasks));
  return buildInstance(std::move(agents), std::move(costs), std::move(tasks));
}

}  // namespace morap
