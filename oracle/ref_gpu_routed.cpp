// TEST INFRASTRUCTURE ONLY -- proves the drop-in: the reference's OWN
// supportingPoint / paretoPoint (solver.hpp:103-294, compiled unmodified from
// /root/reference/proj/include) with its two runBatch calls (solver.hpp:133,172) routed to
// libmorap_cuda.so through the plug-in integration/morap_gpu_runbatch.hpp. Built by
// oracle/Makefile into oracle/_ref/ref_gpu_routed (the reference is not on the GPU box;
// the binary is). tests/test_integration_gpu.py compares its reports with the goldens the
// unmodified CPU reference wrote.
//
//   ref_gpu_routed pareto fig2 <instance.json> <t1,t2,...> <eps>
//   ref_gpu_routed pareto warehouse '<config json>' <t1,...> <eps>
//   ref_gpu_routed jobs '<config json>'     runBatch (CPU engine) vs gpu_runBatch, bitwise
#include "morap/engine.hpp"
#include "../integration/morap_gpu_runbatch.hpp"
#define runBatch gpu_runBatch  // the seam: supportingPoint's batches go to the GPU
#include "morap/solver.hpp"
#undef runBatch
#include "morap/instance.hpp"
#include "morap/logic.hpp"
#include "morap/warehouse.hpp"

#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>

using namespace morap;

namespace {

uint64_t fnvRows(const Scheduler& mu) {  // scheduler fingerprint, as oracle/ref_shim.cpp
  uint64_t h = 1469598103934665603ull;
  for (const auto& c : mu.choice) h = (h ^ static_cast<uint32_t>(c.empty() ? -1 : c[0].first)) * 1099511628211ull;
  return h;
}

Json report(const ParetoResult& res) {  // the same report as oracle/ref_shim.cpp pareto_report
  std::unique_ptr<SynthesisResult> syn;
  Json j;
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
    Json hs = Json::array();
    for (const auto& mu : rec.schedulers) hs.push_back(std::to_string(fnvRows(mu)));
    recs.push_back({{"tUp", rec.tUp}, {"tDown", rec.tDown}, {"schedulerHash", hs}});
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

MorapInstance fromFile(const char* path) {  // inline agents + LTL tasks (cli.hpp:93-117 subset)
  std::ifstream f(path);
  std::stringstream ss;
  ss << f.rdbuf();
  Json j = Json::parse(ss.str());
  std::vector<Mdp> agents;
  std::vector<RewardStructure> costs;
  for (const auto& a : j.at("agents")) {
    auto [m, c] = mdpFromJson(a);
    agents.push_back(std::move(m));
    costs.push_back(std::move(c));
  }
  std::vector<Dfa> tasks;
  for (const auto& t : j.at("tasks")) tasks.push_back(insertPreSinks(formulaToDfa(parseCoSafe(t.get<std::string>()))));
  return buildInstance(std::move(agents), std::move(costs), std::move(tasks));
}

bool sameBits(const Vec& a, const Vec& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

int jobsCheck(const MorapInstance& inst) {
  // optimize jobs over every product at several weights, then evaluate jobs on their
  // policies -- the reference engine on all host threads vs the GPU plug-in
  const double ws[][2] = {{1.0, 0.0}, {0.0, 1.0}, {0.3, 0.7}, {0.125, 0.375}};
  auto make = [&](std::vector<Job>& jobs) {
    long id = 0;
    for (int i = 0; i < inst.n; ++i)
      for (int j = 0; j < inst.n; ++j)
        for (const auto& w : ws) {
          Job job;
          job.id = id++;
          job.kind = JobKind::Optimize;
          job.model = inst.products[i][j];
          job.reward = weightedReward({&job.model->cost, &job.model->success}, {w[0], w[1]});
          jobs.push_back(std::move(job));
        }
  };
  std::vector<Job> a, b;
  make(a);
  make(b);
  const PoolConfig pool = configurePool(defaultWorkerCount());
  auto cpu = runBatch(std::move(a), pool);
  auto gpu = gpu_runBatch(std::move(b), pool);
  int bad = 0;
  std::vector<Job> ea, eb;
  for (auto& [id, r] : cpu) {
    const JobResult& g = gpu.at(id);
    if (r.ok != g.ok || r.value != g.value || r.stats.sweeps != g.stats.sweeps ||
        r.stats.residual != g.stats.residual || !sameBits(r.values, g.values) ||
        fnvRows(r.policy) != fnvRows(g.policy))
      ++bad;
    const int i = static_cast<int>(id / 4) / inst.n, j = static_cast<int>(id / 4) % inst.n;
    for (int which = 0; which < 2; ++which)
      for (auto* v : {&ea, &eb}) {
        Job e;
        e.id = 2 * id + which;
        e.kind = JobKind::Evaluate;
        e.model = inst.products[i][j];
        e.scheduler = r.policy;
        e.reward = which ? e.model->success : e.model->cost;
        v->push_back(std::move(e));
      }
  }
  auto ec = runBatch(std::move(ea), pool);
  auto eg = gpu_runBatch(std::move(eb), pool);
  for (auto& [id, r] : ec) {
    const JobResult& g = eg.at(id);
    if (r.ok != g.ok || r.value != g.value || r.stats.sweeps != g.stats.sweeps ||
        r.stats.residual != g.stats.residual || !sameBits(r.values, g.values))
      ++bad;
  }
  std::printf("{\"optimize_jobs\": %zu, \"evaluate_jobs\": %zu, \"mismatches\": %d}\n", cpu.size(), ec.size(), bad);
  return bad ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc >= 3 && std::string(argv[1]) == "jobs") {
      return jobsCheck(generateInstance(warehouseConfigFromJson(Json::parse(argv[2]))));
    }
    if (argc >= 6 && std::string(argv[1]) == "pareto") {
      MorapInstance inst = std::string(argv[2]) == "fig2" ? fromFile(argv[3])
                                                          : generateInstance(warehouseConfigFromJson(Json::parse(argv[3])));
      Vec t;
      for (std::stringstream ts(argv[4]); ts.good();) {
        std::string tok;
        std::getline(ts, tok, ',');
        if (!tok.empty()) t.push_back(std::stod(tok));
      }
      const double eps = std::stod(argv[5]);
      const PoolConfig pool = configurePool(1);
      // paretoPoint (solver.hpp:281) verbatim; its supportingPoint batches run on the GPU
      ParetoResult res = paretoPoint(inst, t, NormMatrix::identity(2 * inst.n), eps, pool);
      std::cout << report(res).dump() << "\n";
      return 0;
    }
    std::fprintf(stderr, "usage: ref_gpu_routed pareto fig2|warehouse <file|config> <t,...> <eps> | jobs <config>\n");
    return 2;
  } catch (const Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
