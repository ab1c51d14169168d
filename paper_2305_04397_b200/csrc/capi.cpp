// extern "C" face of the host library (include/morap.h).
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <chrono>
#include <cstdio>
#include <thread>

#include "morap.h"
#include "morap.hpp"

struct morap_instance {
  morap::MorapInstance inst;
  std::map<const morap::ProductMdp*, int64_t> firstSlot;  // lazily filled (product_dims)
  std::map<uint64_t, int> owner;                           // sharded builds: product uid -> rank
};

struct morap_solver {
  std::unique_ptr<morap::GpuBackend> gpu;
  bool fingerprints = true;  // per-iteration scheduler hashes in the pareto report
};

struct morap_centralised {
  morap::CentralisedMdp c;
};

struct morap_multi {
  std::vector<std::unique_ptr<morap::GpuBackend>> gpus;
  std::vector<std::unique_ptr<morap::Shard>> shards;
  const morap::MorapInstance* inst = nullptr;
};

namespace {

thread_local std::string g_error;

template <class F>
int guard(F&& body) {
  try {
    body();
    return MORAP_OK;
  } catch (const morap::Error& e) {
    g_error = e.what();
    return morap::statusOf(e.code());
  } catch (const std::exception& e) {
    g_error = e.what();
    return morap::statusOf(morap::Errc::SolverFailure);
  }
}

uint64_t rowsHash(const morap::Scheduler& mu) {  // FNV-style over the int32 rows (test fingerprint)
  uint64_t h = 1469598103934665603ull;
  for (int32_t r : mu.rows) h = (h ^ static_cast<uint32_t>(r)) * 1099511628211ull;
  return h;
}

void putJson(const morap::Json& j, char* out, int cap) {
  const std::string s = j.dump();
  if (!out || static_cast<int>(s.size()) + 1 > cap) morap::fail(morap::Errc::Io, "output buffer too small");
  std::memcpy(out, s.c_str(), s.size() + 1);
}

morap::Json reportJson(const morap::ParetoResult& res, bool fingerprints = true) {
  std::unique_ptr<morap::SynthesisResult> syn;
  int synErr = 0;
  if (res.converged) {
    try {
      syn = std::make_unique<morap::SynthesisResult>(morap::synthesize(res));
    } catch (const morap::Error& e) {
      synErr = morap::statusOf(e.code());
    }
  }
  morap::Json j = morap::resultToJson(res, syn.get());
  j["converged"] = res.converged;
  j["thresholds"] = res.thresholds;
  j["lambdaStar"] = res.lambdaStar;
  // scheduler fingerprints (test evidence, not part of paretoPoint): every (record,
  // scheduler) pair on the host worker pool
  std::vector<std::vector<uint64_t>> hashes(res.iterations.size());
  if (fingerprints) {
    std::vector<std::pair<int, int>> items;
    for (size_t k = 0; k < res.iterations.size(); ++k) {
      hashes[k].resize(res.iterations[k].schedulers.size());
      for (size_t q = 0; q < res.iterations[k].schedulers.size(); ++q)
        items.push_back({static_cast<int>(k), static_cast<int>(q)});
    }
    morap::parallelFor(static_cast<int>(items.size()), [&](int i) {
      const auto [k, q] = items[i];
      hashes[k][q] = rowsHash(res.iterations[k].schedulers[q]);
    });
  }
  morap::Json recs = morap::Json::array();
  for (size_t k = 0; k < res.iterations.size(); ++k) {
    const auto& rec = res.iterations[k];
    morap::Json hs = morap::Json::array();
    for (uint64_t h : hashes[k]) hs.push_back(std::to_string(h));
    if (fingerprints) recs.push_back({{"tUp", rec.tUp}, {"tDown", rec.tDown}, {"schedulerHash", hs}});
    else recs.push_back({{"tUp", rec.tUp}, {"tDown", rec.tDown}});
  }
  j["records"] = recs;
  if (syn) {
    morap::Json mg = morap::Json::array();
    for (int a = 0; a < syn->marginal.rows; ++a) {
      morap::Json row = morap::Json::array();
      for (int b = 0; b < syn->marginal.cols; ++b) row.push_back(syn->marginal(a, b));
      mg.push_back(row);
    }
    j["marginal"] = mg;
  }
  if (synErr) j["synthesisError"] = synErr;
  return j;
}

void putStats(const morap::QueryStats& q, double* out) {
  if (!out) return;
  out[0] = static_cast<double>(q.optimizeJobs);
  out[1] = q.optimizeBackups;
  out[2] = static_cast<double>(q.evaluateJobs);
  out[3] = q.evaluateStateBackups;
  out[4] = q.optimizeSeconds;
  out[5] = q.evaluateSeconds;
  out[6] = q.hostSeconds;
  out[7] = q.evaluateSweepSeconds;
}

morap::NormMatrix normOf(const double* norm, int d) {
  morap::Mat m(d, d, 0.0);
  if (norm) std::memcpy(m.a.data(), norm, sizeof(double) * d * d);
  else
    for (int k = 0; k < d; ++k) m(k, k) = 1.0;
  return morap::NormMatrix(std::move(m));
}

}  // namespace

extern "C" {

const char* morap_last_error(void) { return g_error.c_str(); }

int morap_instance_warehouse(const char* config_json, int threads, morap_instance** out) {
  return guard([&] {
    if (!out || !config_json) morap::fail(morap::Errc::InvalidConfig, "null argument");
    morap::WarehouseConfig cfg = morap::warehouseConfigFromJson(morap::Json::parse(config_json));
    *out = new morap_instance{morap::generateInstance(cfg, threads), {}, {}};
  });
}

namespace {
int fromJson(const char* text, const char* base_dir, morap_instance** out, double* norm_out, int norm_cap,
             int* has_norm, const morap::InstanceBuilder* build) {
  return guard([&] {
    if (!out || !text) morap::fail(morap::Errc::InvalidConfig, "null argument");
    morap::Json j;
    try {
      j = morap::Json::parse(text);
    } catch (const morap::Json::exception& e) {
      morap::fail(morap::Errc::Io, e.what());
    }
    const std::string base = base_dir ? base_dir : ".";
    auto inst = std::make_unique<morap_instance>(morap_instance{morap::instanceFromJson(j, base, build), {}, {}});
    if (has_norm) *has_norm = 0;
    if (j.contains("norm") && norm_out) {
      morap::Json nj = j.at("norm");
      if (nj.is_string()) {
        std::ifstream in(base + "/" + nj.get<std::string>());
        if (!in) morap::fail(morap::Errc::Io, "cannot open norm file");
        nj = morap::Json::parse(in);
      }
      if (!nj.is_array() || nj.empty()) morap::fail(morap::Errc::InvalidConfig, "norm matrix must be a nonempty array of rows");
      const int d = static_cast<int>(nj.size());
      if (d * d > norm_cap) morap::fail(morap::Errc::DimensionMismatch, "norm buffer too small");
      morap::Mat m(d, d);
      for (int r = 0; r < d; ++r) {
        if (!nj[r].is_array() || static_cast<int>(nj[r].size()) != d)
          morap::fail(morap::Errc::InvalidConfig, "norm matrix rows must all have the matrix dimension");
        for (int c = 0; c < d; ++c) m(r, c) = nj[r][c].get<double>();
      }
      morap::NormMatrix check(m);  // validates symmetry / definiteness
      std::memcpy(norm_out, m.a.data(), sizeof(double) * d * d);
      if (has_norm) *has_norm = d;
    }
    *out = inst.release();
  });
}
}  // namespace

int morap_instance_from_json(const char* text, const char* base_dir, morap_instance** out, double* norm_out,
                             int norm_cap, int* has_norm) {
  return fromJson(text, base_dir, out, norm_out, norm_cap, has_norm, nullptr);
}

int morap_instance_from_json_device(const char* text, const char* base_dir, morap_solver* s, morap_instance** out,
                                    double* norm_out, int norm_cap, int* has_norm) {
  if (!s) return guard([&] { morap::fail(morap::Errc::InvalidConfig, "null solver"); });
  morap::GpuBackend& gpu = *s->gpu;
  const morap::InstanceBuilder build = [&](std::vector<morap::Mdp> agents, std::vector<morap::RewardStructure> costs,
                                           std::vector<morap::Dfa> tasks) {
    return morap::buildInstanceOnDevice(gpu, std::move(agents), std::move(costs), std::move(tasks));
  };
  return fromJson(text, base_dir, out, norm_out, norm_cap, has_norm, &build);
}

void morap_instance_free(morap_instance* inst) { delete inst; }

int morap_instance_info(const morap_instance* p, int64_t* out) {
  return guard([&] {
    const auto& I = p->inst;
    int64_t S = 0, R = 0, Z = 0, Zd = 0;
    std::set<const morap::ProductMdp*> seen;
    for (const auto& row : I.products)
      for (const auto& q : row) {
        S += q->mdp.numStates;
        R += morap::productRows(*q);
        Z += morap::productNnz(*q);
        if (seen.insert(q.get()).second) Zd += morap::productNnz(*q);
      }
    const int64_t v[8] = {I.n, I.realTasks, I.distinctProducts, I.objectives, S, R, Z, Zd};
    std::memcpy(out, v, sizeof v);
  });
}

int morap_instance_product_dims(const morap_instance* p, int i, int j, int64_t* dims, uint64_t* hash) {
  return guard([&] {
    const auto& I = p->inst;
    if (i < 0 || j < 0 || i >= I.n || j >= I.n) morap::fail(morap::Errc::InvalidConfig, "product index out of range");
    const morap::ProductMdp& q = *I.products[i][j];
    auto& firstSlot = const_cast<morap_instance*>(p)->firstSlot;
    if (firstSlot.empty())
      for (int a = I.n - 1; a >= 0; --a)
        for (int b = I.n - 1; b >= 0; --b) firstSlot[I.products[a][b].get()] = static_cast<int64_t>(a) * I.n + b;
    const int64_t v[6] = {q.mdp.numStates, morap::productRows(q), morap::productNnz(q), q.mdp.initial,
                          q.rewardFinite ? 1 : 0, firstSlot.at(&q)};
    std::memcpy(dims, v, sizeof v);
    if (hash) *hash = q.structuralHash;
  });
}

int morap_instance_product_export(const morap_instance* p, int i, int j, int32_t* ro, int32_t* to, int32_t* succ,
                                  double* prob, double* cost, double* success, uint8_t* done, uint8_t* accept) {
  return guard([&] {
    const auto& I = p->inst;
    if (i < 0 || j < 0 || i >= I.n || j >= I.n) morap::fail(morap::Errc::InvalidConfig, "product index out of range");
    const morap::ProductMdp& q = *I.products[i][j];
    morap::requireFull(q, "product export");
    auto cp = [](auto* dst, const auto& v) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(ro, q.mdp.rowOffset);
    cp(to, q.mdp.trnOffset);
    cp(succ, q.mdp.succ);
    cp(prob, q.mdp.prob);
    cp(cost, q.cost);
    cp(success, q.success);
    for (int s = 0; s < q.mdp.numStates; ++s) {
      if (done) done[s] = q.done[s] ? 1 : 0;
      if (accept) accept[s] = q.accept[s] ? 1 : 0;
    }
  });
}

int morap_instance_product_objective(const morap_instance* p, int i, int j, int k, double* out) {
  return guard([&] {
    const auto& I = p->inst;
    if (i < 0 || j < 0 || i >= I.n || j >= I.n || k < 0 || k >= I.objectives)
      morap::fail(morap::Errc::InvalidConfig, "objective index out of range");
    const morap::ProductMdp& q = *I.products[i][j];
    morap::requireFull(q, "product objective");
    const morap::RewardStructure& v = k == 0 ? q.cost : k == I.objectives - 1 ? q.success : q.extra.at(k - 1);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}

int morap_instance_add_objectives(morap_instance* p, int K, uint64_t seed) {
  return guard([&] {
    morap::addSyntheticObjectives(p->inst, K, seed);
    p->firstSlot.clear();
  });
}

int morap_solver_create(int device, morap_solver** out) {
  return guard([&] {
    if (!out) morap::fail(morap::Errc::InvalidConfig, "null argument");
    auto s = std::make_unique<morap_solver>();
    s->gpu = std::make_unique<morap::GpuBackend>(device);
    *out = s.release();
  });
}

void morap_solver_free(morap_solver* s) { delete s; }

morap_ctx* morap_solver_cuda(morap_solver* s) { return s && s->gpu ? s->gpu->ctx() : nullptr; }

int morap_solver_upload(morap_solver* s, const morap_instance* inst) {
  return guard([&] { s->gpu->uploadInstance(inst->inst); });
}

int morap_solver_release(morap_solver* s) {
  return guard([&] { s->gpu->release(); });
}

int morap_instance_warehouse_shard(const char* config_json, int threads, int rank, int world, int chunk,
                                   morap_instance** out) {
  return guard([&] {
    if (!out || !config_json) morap::fail(morap::Errc::InvalidConfig, "null argument");
    if (world < 1 || rank < 0 || rank >= world || chunk < 1) morap::fail(morap::Errc::InvalidConfig, "bad shard");
    morap::WarehouseConfig cfg = morap::warehouseConfigFromJson(morap::Json::parse(config_json));
    std::map<uint64_t, int> owner;
    std::vector<double> load(static_cast<size_t>(world), 0.0);
    // distinct products arrive in (i, j) order of first occurrence: each goes to the least
    // loaded rank (by nnz, lowest rank on ties) -- the same decision on every rank
    const morap::ProductSink sink = [&](const std::vector<morap::ProductMdp*>& fresh) {
      std::vector<morap::ProductMdp*> drop;
      for (morap::ProductMdp* p : fresh) {
        const int r = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
        load[static_cast<size_t>(r)] += static_cast<double>(morap::productNnz(*p));
        owner[p->uid] = r;
        if (r != rank) drop.push_back(p);
      }
      for (morap::ProductMdp* p : drop) morap::slimProduct(*p);
    };
    const std::function<void()> retry = [&] {
      owner.clear();
      std::fill(load.begin(), load.end(), 0.0);
    };
    morap::MorapInstance inst = morap::generateInstance(cfg, threads, static_cast<size_t>(chunk), &sink, &retry);
    *out = new morap_instance{std::move(inst), {}, std::move(owner)};
  });
}

int morap_instance_product_owner(const morap_instance* p, int i, int j) {
  if (!p || i < 0 || j < 0 || i >= p->inst.n || j >= p->inst.n) return -1;
  auto it = p->owner.find(p->inst.products[i][j]->uid);
  return it == p->owner.end() ? -1 : it->second;
}

int morap_solver_set_lean(morap_solver* s, int on) {
  return guard([&] { s->gpu->setLean(on != 0); });
}

int morap_solver_set_fingerprints(morap_solver* s, int on) {
  return guard([&] {
    if (!s) morap::fail(morap::Errc::InvalidConfig, "null solver");
    s->fingerprints = on != 0;
  });
}

int morap_instance_warehouse_streamed(const char* config_json, int threads, morap_solver* s, int chunk,
                                      morap_instance** out) {
  return guard([&] {
    if (!out || !config_json || !s) morap::fail(morap::Errc::InvalidConfig, "null argument");
    if (chunk < 1) morap::fail(morap::Errc::InvalidConfig, "chunk must be positive");
    morap::WarehouseConfig cfg = morap::warehouseConfigFromJson(morap::Json::parse(config_json));
    morap::GpuBackend& gpu = *s->gpu;
    const bool trace = std::getenv("MORAP_TRACE") != nullptr;
    const morap::ProductSink sink = [&](const std::vector<morap::ProductMdp*>& fresh) {
      const auto t0 = std::chrono::steady_clock::now();
      gpu.uploadProducts(std::vector<const morap::ProductMdp*>(fresh.begin(), fresh.end()), gpu.lean());
      if (trace)
        std::fprintf(stderr, "[morap] streamed chunk: upload %.1f ms\n",
                     1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      std::vector<std::thread> pool;
      const size_t T = std::max(1u, std::thread::hardware_concurrency());
      for (size_t t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
          for (size_t k = t; k < fresh.size(); k += T) morap::slimProduct(*fresh[k]);
        });
      for (auto& th : pool) th.join();
    };
    const std::function<void()> retry = [&] { gpu.release(); };
    *out = new morap_instance{morap::generateInstance(cfg, threads, static_cast<size_t>(chunk), &sink, &retry), {}, {}};
  });
}

int morap_instance_warehouse_device(const char* config_json, morap_solver* s, morap_instance** out) {
  return guard([&] {
    if (!out || !config_json || !s) morap::fail(morap::Errc::InvalidConfig, "null argument");
    morap::WarehouseConfig cfg = morap::warehouseConfigFromJson(morap::Json::parse(config_json));
    morap::GpuBackend& gpu = *s->gpu;
    const morap::InstanceBuilder build = [&](std::vector<morap::Mdp> agents, std::vector<morap::RewardStructure> costs,
                                             std::vector<morap::Dfa> tasks) {
      return morap::buildInstanceOnDevice(gpu, std::move(agents), std::move(costs), std::move(tasks));
    };
    const std::function<void()> retry = [&] { gpu.release(); };
    *out = new morap_instance{morap::generateInstanceWith(cfg, build, &retry), {}, {}};
  });
}

int morap_instance_warehouse_device_shard(const char* config_json, morap_solver* s, int rank, int world,
                                          morap_instance** out) {
  return guard([&] {
    if (!out || !config_json || !s) morap::fail(morap::Errc::InvalidConfig, "null argument");
    if (world < 1 || rank < 0 || rank >= world) morap::fail(morap::Errc::InvalidConfig, "bad shard");
    morap::WarehouseConfig cfg = morap::warehouseConfigFromJson(morap::Json::parse(config_json));
    morap::GpuBackend& gpu = *s->gpu;
    std::map<uint64_t, int> owner;
    // every rank measures every pair (a fraction of a second at C4) and so takes the same
    // owners as morap_instance_warehouse_shard: distinct products in first-occurrence order,
    // each to the least loaded rank by nnz; it then builds only its own
    const morap::InstanceBuilder build = [&](std::vector<morap::Mdp> agents, std::vector<morap::RewardStructure> costs,
                                             std::vector<morap::Dfa> tasks) {
      auto plan = morap::planDeviceBuild(gpu, std::move(agents), std::move(costs), std::move(tasks));
      std::vector<double> load(static_cast<size_t>(world), 0.0);
      std::vector<size_t> mine;
      owner.clear();
      for (size_t k = 0; k < plan->distinct.size(); ++k) {
        const morap::ProductMdp* p = plan->distinct[k];
        const int r = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
        load[static_cast<size_t>(r)] += static_cast<double>(morap::productNnz(*p));
        owner[p->uid] = r;
        if (r == rank) mine.push_back(k);
      }
      plan->write(gpu, mine);
      return std::move(plan->inst);
    };
    morap::MorapInstance inst = morap::generateInstanceWith(cfg, build);
    *out = new morap_instance{std::move(inst), {}, std::move(owner)};
  });
}

int morap_multi_warehouse_device(morap_multi* m, const char* config_json, morap_instance** out) {
  return guard([&] {
    if (!m || !out || !config_json) morap::fail(morap::Errc::InvalidConfig, "null argument");
    morap::WarehouseConfig cfg = morap::warehouseConfigFromJson(morap::Json::parse(config_json));
    const int world = static_cast<int>(m->gpus.size());
    for (auto& g : m->gpus) g->release();
    m->shards.clear();
    m->inst = nullptr;
    std::unique_ptr<morap::DeviceBuild> plan;
    const morap::InstanceBuilder build = [&](std::vector<morap::Mdp> agents, std::vector<morap::RewardStructure> costs,
                                             std::vector<morap::Dfa> tasks) {
      plan = morap::planDeviceBuild(*m->gpus[0], std::move(agents), std::move(costs), std::move(tasks));
      return morap::MorapInstance{};
    };
    morap::generateInstanceWith(cfg, build);
    auto mi = std::make_unique<morap_instance>(morap_instance{std::move(plan->inst), {}, {}});
    const morap::MorapInstance& inst = mi->inst;
    // the owners morap_multi_upload would take (LPT by nnz); each device builds its own
    const std::vector<int> owner = morap::lptOwners(inst, world);
    std::map<const morap::ProductMdp*, int> ownerOf;
    for (int i = 0; i < inst.n; ++i)
      for (int j = 0; j < inst.n; ++j) ownerOf[inst.products[i][j].get()] = owner[static_cast<size_t>(i) * inst.n + j];
    std::vector<std::vector<size_t>> mine(static_cast<size_t>(world));
    for (size_t k = 0; k < plan->distinct.size(); ++k) mine[ownerOf.at(plan->distinct[k])].push_back(k);
    std::vector<std::thread> pool;  // one build thread per device
    std::vector<std::exception_ptr> err(static_cast<size_t>(world));
    for (int r = 0; r < world; ++r)
      pool.emplace_back([&, r] {
        try {
          plan->write(*m->gpus[r], mine[r]);
        } catch (...) {
          err[r] = std::current_exception();
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
    for (int r = 0; r < world; ++r) {
      m->shards.push_back(std::make_unique<morap::Shard>(inst, *m->gpus[r], owner, r));
      m->shards.back()->upload();  // registers nothing new: every owned product is resident
    }
    m->inst = &mi->inst;
    *out = mi.release();
  });
}

int morap_multi_create(const int* devices, int ndevices, morap_multi** out) {
  return guard([&] {
    if (!out || !devices || ndevices < 1) morap::fail(morap::Errc::InvalidConfig, "need at least one device");
    auto m = std::make_unique<morap_multi>();
    for (int d = 0; d < ndevices; ++d) m->gpus.push_back(std::make_unique<morap::GpuBackend>(devices[d]));
    *out = m.release();
  });
}

void morap_multi_free(morap_multi* m) { delete m; }

int morap_multi_upload(morap_multi* m, const morap_instance* p) {
  return guard([&] {
    if (!m || !p) morap::fail(morap::Errc::InvalidConfig, "null argument");
    const int world = static_cast<int>(m->gpus.size());
    std::vector<int> owner = morap::lptOwners(p->inst, world);
    m->shards.clear();
    for (auto& g : m->gpus) g->release();
    for (int r = 0; r < world; ++r) m->shards.push_back(std::make_unique<morap::Shard>(p->inst, *m->gpus[r], owner, r));
    std::vector<std::thread> pool;  // one upload thread per device
    std::vector<std::exception_ptr> err(static_cast<size_t>(world));
    for (int r = 0; r < world; ++r)
      pool.emplace_back([&, r] {
        try {
          m->shards[r]->upload();
        } catch (...) {
          err[r] = std::current_exception();
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
    m->inst = &p->inst;
  });
}

int morap_multi_owner(const morap_multi* m, int i, int j) {
  if (!m || m->shards.empty() || !m->inst || i < 0 || j < 0 || i >= m->inst->n || j >= m->inst->n) return -1;
  return m->shards[0]->owners()[static_cast<size_t>(i) * m->inst->n + j];
}

int morap_multi_pareto(morap_multi* m, const morap_instance* p, const double* thresholds, int nt, const double* norm,
                       double eps, int iteration_cap, char* json_out, int json_cap, double* stats_out) {
  return guard([&] {
    if (!m || !p) morap::fail(morap::Errc::InvalidConfig, "null argument");
    if (m->inst != &p->inst) morap_multi_upload(m, p) == 0 ? void() : morap::fail(morap::Errc::SolverFailure, g_error);
    const int d = p->inst.objectives * p->inst.n;
    morap::NormMatrix M = normOf(norm, d);
    morap::Vec t(thresholds, thresholds + nt);
    morap::QueryStats st;
    std::vector<morap::Shard*> shards;
    for (auto& s : m->shards) shards.push_back(s.get());
    morap::ParetoResult res = morap::paretoPointMulti(shards, t, M, eps, iteration_cap, &st);
    putJson(reportJson(res, false), json_out, json_cap);
    putStats(st, stats_out);
  });
}

int morap_shard_pareto(morap_solver* s, const morap_instance* p, int rank, int world, morap_allgather_fn allgather,
                       void* user, const double* thresholds, int nt, const double* norm, double eps, int iteration_cap,
                       char* json_out, int json_cap, double* stats_out) {
  return guard([&] {
    if (!s || !p || !allgather) morap::fail(morap::Errc::InvalidConfig, "null argument");
    if (world < 1 || rank < 0 || rank >= world) morap::fail(morap::Errc::InvalidConfig, "bad shard");
    const int n = p->inst.n;
    std::vector<int> owner;
    if (!p->owner.empty()) {  // built per rank (morap_instance_warehouse_shard): its owners
      owner.resize(static_cast<size_t>(n) * n);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          auto it = p->owner.find(p->inst.products[i][j]->uid);
          if (it == p->owner.end() || it->second >= world)
            morap::fail(morap::Errc::InvalidConfig, "instance was sharded for a different world size");
          owner[static_cast<size_t>(i) * n + j] = it->second;
        }
    } else {
      owner = morap::lptOwners(p->inst, world);
    }
    morap::Shard shard(p->inst, *s->gpu, owner, rank);
    shard.upload();
    const morap::Exchange ex = [&](const double* send, int count, double* recv) {
      const int rc = allgather(user, send, count, recv);
      if (rc != 0) morap::fail(morap::Errc::SolverFailure, "allgather failed (" + std::to_string(rc) + ")");
    };
    const int d = p->inst.objectives * n;
    morap::NormMatrix M = normOf(norm, d);
    morap::Vec t(thresholds, thresholds + nt);
    morap::QueryStats st;
    morap::ParetoResult res = morap::paretoPointSharded(shard, world, ex, t, M, eps, iteration_cap, &st);
    putJson(reportJson(res, false), json_out, json_cap);
    putStats(st, stats_out);
  });
}

int morap_supporting_point(morap_solver* s, const morap_instance* p, const double* w, int nw, double* r_out,
                           int32_t* agent_of, double* stats_out) {
  return guard([&] {
    morap::QueryStats st;
    morap::SupportingPoint sp = morap::supportingPoint(p->inst, morap::Vec(w, w + nw), *s->gpu, &st);
    std::memcpy(r_out, sp.r.data(), sizeof(double) * sp.r.size());
    for (size_t j = 0; j < sp.assignment.agentOf.size(); ++j) agent_of[j] = sp.assignment.agentOf[j];
    putStats(st, stats_out);
  });
}

int morap_pareto(morap_solver* s, const morap_instance* p, const double* thresholds, int nt, const double* norm,
                 double eps, int iteration_cap, int verify, char* json_out, int json_cap, double* stats_out) {
  return guard([&] {
    const int d = p->inst.objectives * p->inst.n;
    morap::NormMatrix M = normOf(norm, d);
    morap::Vec t(thresholds, thresholds + nt);
    morap::QueryStats st;
    if (verify) {
      const bool v = morap::verifyOnly(p->inst, t, M, eps, *s->gpu, iteration_cap);
      putJson(morap::Json{{"verdict", v}}, json_out, json_cap);
    } else {
      morap::ParetoResult res = morap::paretoPoint(p->inst, t, M, eps, *s->gpu, iteration_cap, &st);
      putJson(reportJson(res, s->fingerprints), json_out, json_cap);
    }
    putStats(st, stats_out);
  });
}

int morap_pareto_core(const double* thr, int d, int n, const double* norm, double eps, int iteration_cap, int verify,
                      morap_query_fn query, void* user, char* json_out, int json_cap) {
  return guard([&] {
    if (!query) morap::fail(morap::Errc::InvalidConfig, "null query callback");
    morap::NormMatrix M = normOf(norm, d);
    bool verdict = false;
    auto q = [&](const morap::Vec& w) {
      morap::SupportingPoint sp;
      sp.r.assign(static_cast<size_t>(d), 0.0);
      std::vector<int32_t> a(static_cast<size_t>(n), -1);
      const int rc = query(user, w.data(), d, sp.r.data(), a.data(), n);
      if (rc != 0) {
        const morap::Errc e = rc >= 1 && rc <= 21 ? static_cast<morap::Errc>(rc - 1) : morap::Errc::SolverFailure;
        morap::fail(e, "external supporting-point query failed");
      }
      sp.assignment.agentOf.assign(a.begin(), a.end());
      sp.schedulers.resize(static_cast<size_t>(n));
      return sp;
    };
    morap::ParetoResult res =
        morap::runParetoCore(morap::Vec(thr, thr + d), M, eps, iteration_cap, verify != 0, verify ? &verdict : nullptr, q);
    morap::Json j = reportJson(res);
    if (verify) j["verdict"] = verdict;
    putJson(j, json_out, json_cap);
  });
}

int morap_centralised_build(const morap_instance* inst, int64_t state_guard, morap_centralised** out) {
  return guard([&] {
    if (!inst || !out) morap::fail(morap::Errc::InvalidConfig, "null argument");
    *out = new morap_centralised{morap::buildCentralised(inst->inst, static_cast<long>(state_guard))};
  });
}

void morap_centralised_free(morap_centralised* c) { delete c; }

int morap_centralised_info(const morap_centralised* p, int64_t* out) {
  return guard([&] {
    const auto& c = p->c;
    const int64_t v[6] = {c.mdp.numStates, c.mdp.numActions(), static_cast<int64_t>(c.mdp.succ.size()),
                          c.mdp.initial, c.rewardFinite ? 1 : 0, static_cast<int64_t>(c.rewards.size())};
    std::memcpy(out, v, sizeof v);
  });
}

int morap_centralised_export(const morap_centralised* p, int32_t* ro, int32_t* to, int32_t* succ, double* prob,
                             uint8_t* done, double* const* rewards) {
  return guard([&] {
    const auto& c = p->c;
    auto cp = [](auto* dst, const auto& v) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(ro, c.mdp.rowOffset);
    cp(to, c.mdp.trnOffset);
    cp(succ, c.mdp.succ);
    cp(prob, c.mdp.prob);
    if (done)
      for (size_t s = 0; s < c.done.size(); ++s) done[s] = c.done[s] ? 1 : 0;
    if (rewards)
      for (size_t k = 0; k < c.rewards.size(); ++k) cp(rewards[k], c.rewards[k]);
  });
}

int morap_centralised_pareto(morap_solver* s, const morap_centralised* p, const double* thresholds, int nt,
                             const double* norm, double eps, int iteration_cap, char* json_out, int json_cap,
                             double* stats_out) {
  return guard([&] {
    const int d = static_cast<int>(p->c.rewards.size());
    morap::NormMatrix M = normOf(norm, d);
    morap::QueryStats st;
    morap::ParetoResult res = morap::centralisedParetoPoint(p->c, morap::Vec(thresholds, thresholds + nt), M, eps,
                                                            *s->gpu, iteration_cap, &st);
    putJson(reportJson(res), json_out, json_cap);
    putStats(st, stats_out);
  });
}

int morap_run_batch(morap_solver* s, const morap_instance* p, int njobs, const morap_job* jobs,
                    morap_job_result* results, double* const* values_out, int32_t* const* policy_out) {
  return guard([&] {
    if (!s || !p || njobs < 0 || (njobs > 0 && (!jobs || !results))) morap::fail(morap::Errc::InvalidConfig, "null argument");
    const auto& I = p->inst;
    std::vector<morap::Job> batch(static_cast<size_t>(njobs));
    for (int k = 0; k < njobs; ++k) {
      const morap_job& j = jobs[k];
      morap::Job& J = batch[static_cast<size_t>(k)];
      J.id = static_cast<long>(j.id);
      J.kind = j.kind == 1 ? morap::JobKind::Evaluate : morap::JobKind::Optimize;
      if (j.agent >= 0) {
        if (j.agent >= I.n || j.task < 0 || j.task >= I.n) morap::fail(morap::Errc::InvalidConfig, "product index out of range");
        J.model = I.products[static_cast<size_t>(j.agent)][static_cast<size_t>(j.task)];
      }
      if (j.reward && j.reward_len > 0) J.reward.assign(j.reward, j.reward + j.reward_len);
      if (j.scheduler && j.scheduler_len > 0) J.scheduler.rows.assign(j.scheduler, j.scheduler + j.scheduler_len);
      J.eps = j.eps;
      J.sweepCap = j.sweep_cap;
    }
    std::map<long, morap::JobResult> res = morap::runBatch(std::move(batch), *s->gpu);
    for (int k = 0; k < njobs; ++k) {
      const morap::JobResult& r = res.at(static_cast<long>(jobs[k].id));
      morap_job_result& o = results[k];
      o.id = jobs[k].id;
      o.status = r.ok ? 0 : (r.errc ? morap::statusOf(*r.errc) : morap::statusOf(morap::Errc::SolverFailure));
      o.sweeps = r.stats.sweeps;
      o.value = r.value;
      o.residual = r.stats.residual;
      if (r.ok && values_out && values_out[k]) std::memcpy(values_out[k], r.values.data(), sizeof(double) * r.values.size());
      if (r.ok && policy_out && policy_out[k])
        for (size_t q = 0; q < r.policy.rows.size(); ++q) policy_out[k][q] = r.policy.rows[q];
    }
  });
}

int morap_max_assignment(int n, const double* c, int32_t* agent_of) {
  return guard([&] {
    morap::Mat m(n, n);
    std::memcpy(m.a.data(), c, sizeof(double) * n * n);
    morap::Assignment a = morap::maxAssignment(m);
    for (int j = 0; j < n; ++j) agent_of[j] = a.agentOf[j];
  });
}

}  // extern "C"
