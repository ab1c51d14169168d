// Per-model solve and the job engine on the GPU (reference: numerics.hpp, engine.hpp).
//
// GpuBackend owns one morap_ctx (include/morap_cuda.h) and the product -> device-model
// map: products are uploaded once and stay resident for every Pareto iteration
// (the reference keeps shared_ptr<const ProductMdp> alive the same way). runBatch keeps
// the engine's contract -- one JobResult per job id, per-job failure containment with
// the library error code, results independent of how jobs are batched -- but executes
// each kind of job as a single device batch instead of a CPU worker pool.
#include <cstring>
#include <malloc.h>
#include <mutex>
#include <set>

#include "morap.hpp"
#include "morap_cuda.h"

namespace morap {

namespace {

void check(morap_ctx* ctx, int status, const char* what) {
  if (status == MORAP_OK) return;
  std::string msg = std::string(what) + ": " + (ctx ? morap_cuda_last_error(ctx) : "no context");
  if (status >= 1 && status <= 21) throw Error(static_cast<Errc>(status - 1), msg);
  throw Error(Errc::SolverFailure, msg);
}

// Device objective order: cost, extra cost-type objectives, success -- objective k < K-1
// is weighted by the agent's coordinate, the last one by the task's.
std::vector<const double*> objectivesOf(const ProductMdp& p) {
  std::vector<const double*> o{p.cost.data()};
  for (const auto& e : p.extra) o.push_back(e.data());
  o.push_back(p.success.data());
  return o;
}

morap_csr_view viewOf(const ProductMdp& p, const std::vector<const double*>& objs, std::vector<uint8_t>& doneBytes) {
  requireFull(p, "upload to another device");
  morap_csr_view v{};
  v.num_states = p.mdp.numStates;
  v.num_rows = p.mdp.numActions();
  v.nnz = static_cast<int32_t>(p.mdp.succ.size());
  v.initial = p.mdp.initial;
  v.reward_finite = p.rewardFinite ? 1 : 0;
  v.num_objectives = static_cast<int32_t>(objs.size());
  v.row_offset = p.mdp.rowOffset.data();
  v.trn_offset = p.mdp.trnOffset.data();
  v.succ = p.mdp.succ.data();
  v.prob = p.mdp.prob.data();
  doneBytes.assign(p.done.begin(), p.done.end());
  v.done = doneBytes.data();
  v.rewards = objs.data();
  return v;
}

}  // namespace

namespace {
// Every Pareto iteration keeps n fresh scheduler vectors (IterationRecord::schedulers,
// ~0.3 MB each on C2). With glibc's defaults those come from fresh mmaps and are
// page-faulted in on every iteration (~1 ms per C2 iteration); keeping large blocks on
// the heap lets later queries reuse the pages.
void keepLargeBlocksOnHeap() {
  static std::once_flag once;
  std::call_once(once, [] {
    mallopt(M_MMAP_THRESHOLD, 256 << 20);
    mallopt(M_TRIM_THRESHOLD, 1 << 30);
  });
}
}  // namespace

GpuBackend::GpuBackend(int device) : device_(device) {
  keepLargeBlocksOnHeap();
  const int rc = morap_cuda_create(device, &ctx_);
  if (rc != MORAP_OK) {
    ctx_ = nullptr;
    throw Error(Errc::InvalidConfig, "morap_cuda_create failed on device " + std::to_string(device) +
                                         " (an sm_100 GPU is required; there is no CPU fallback)");
  }
}

GpuBackend::~GpuBackend() {
  if (image_) morap_cuda_free_image(image_);
  if (ctx_) morap_cuda_destroy(ctx_);
}

void GpuBackend::release() {
  check(ctx_, morap_cuda_release_models(ctx_), "release models");
  ids_.clear();
  fullIds_.clear();
}

bool GpuBackend::isLean(int id) {
  int32_t info[6];
  check(ctx_, morap_cuda_model_info(ctx_, id, info), "model info");
  return info[5] != 0;
}

// Pareto-query uploads are lean when the objectives fit the policy-chain evaluation
// (K <= 4): compact products then travel without their fp64 arrays. Jobs with an explicit
// reward vector (runBatch, optimalScheduler, evaluateScheduler) need those arrays and get a
// full copy of such a product on first use.
int GpuBackend::modelId(const ProductMdp* p, bool full) {
  auto it = ids_.find(p->uid);
  if (full) {
    if (it != ids_.end() && !isLean(it->second)) return it->second;
    auto f = fullIds_.find(p->uid);
    if (f != fullIds_.end()) return f->second;
  } else if (it != ids_.end()) {
    return it->second;
  }
  std::vector<const double*> objs = objectivesOf(*p);
  std::vector<uint8_t> done;
  morap_csr_view v = viewOf(*p, objs, done);
  const bool lean = !full && leanDefault_ && objs.size() <= 4;
  check(ctx_, morap_cuda_set_lean(ctx_, lean ? 1 : 0), "set lean");
  int32_t id = -1;
  check(ctx_, morap_cuda_upload(ctx_, 1, &v, &id), "upload model");
  (full ? fullIds_ : ids_).emplace(p->uid, id);
  return id;
}

int GpuBackend::modelIdFor(uint64_t uid, const morap_csr_view& view) {
  auto it = ids_.find(uid);
  if (it != ids_.end()) return it->second;
  check(ctx_, morap_cuda_set_lean(ctx_, 0), "set lean");
  int32_t id = -1;
  check(ctx_, morap_cuda_upload(ctx_, 1, &view, &id), "upload model");
  ids_.emplace(uid, id);
  return id;
}

void GpuBackend::setLean(bool on) { leanDefault_ = on; }

// A whole instance goes through a cached device image (morap_cuda_build_image): the
// product builder's packed output for these products stays in pinned host memory, so
// re-uploading the same instance (after release(), or on a fresh context of the same
// device) is a single host-to-device copy.
void GpuBackend::uploadInstance(const MorapInstance& inst) {
  std::vector<const ProductMdp*> todo;
  for (const auto& row : inst.products)
    for (const auto& p : row) todo.push_back(p.get());
  uploadCached(todo, leanDefault_ && inst.objectives <= 4);
}

void GpuBackend::uploadCached(const std::vector<const ProductMdp*>& products, bool lean) {
  std::vector<const ProductMdp*> todo;
  std::set<uint64_t> queued;
  for (const ProductMdp* p : products)
    if (!ids_.count(p->uid) && queued.insert(p->uid).second) todo.push_back(p);
  if (todo.empty()) return;
  std::vector<uint64_t> key{lean ? 1ull : 0ull};
  for (const ProductMdp* p : todo) {
    if (p->slim) {  // streamed / slimmed products have no host arrays to image
      uploadProducts(todo, lean);
      return;
    }
    key.push_back(p->uid);
  }
  if (!image_ || imageKey_ != key) {
    if (image_) morap_cuda_free_image(image_);
    image_ = nullptr;
    std::vector<std::vector<const double*>> objs(todo.size());
    std::vector<std::vector<uint8_t>> done(todo.size());
    std::vector<morap_csr_view> views(todo.size());
    for (size_t k = 0; k < todo.size(); ++k) {
      objs[k] = objectivesOf(*todo[k]);
      views[k] = viewOf(*todo[k], objs[k], done[k]);
    }
    check(ctx_, morap_cuda_set_lean(ctx_, lean ? 1 : 0), "set lean");
    check(ctx_, morap_cuda_build_image(ctx_, static_cast<int>(todo.size()), views.data(), &image_), "build image");
    imageKey_ = std::move(key);
  }
  std::vector<int32_t> ids(todo.size());
  check(ctx_, morap_cuda_upload_image(ctx_, image_, ids.data()), "upload instance");
  for (size_t k = 0; k < todo.size(); ++k) ids_.emplace(todo[k]->uid, ids[k]);
}

void GpuBackend::uploadProducts(const std::vector<const ProductMdp*>& products, bool lean) {
  std::vector<const ProductMdp*> todo;
  std::set<uint64_t> queued;
  for (const ProductMdp* p : products)
    if (!ids_.count(p->uid) && queued.insert(p->uid).second) todo.push_back(p);
  if (todo.empty()) return;
  std::vector<std::vector<const double*>> objs(todo.size());
  std::vector<std::vector<uint8_t>> done(todo.size());
  std::vector<morap_csr_view> views(todo.size());
  for (size_t k = 0; k < todo.size(); ++k) {
    objs[k] = objectivesOf(*todo[k]);
    views[k] = viewOf(*todo[k], objs[k], done[k]);
  }
  check(ctx_, morap_cuda_set_lean(ctx_, lean ? 1 : 0), "set lean");
  std::vector<int32_t> ids(todo.size());
  check(ctx_, morap_cuda_upload(ctx_, static_cast<int>(todo.size()), views.data(), ids.data()), "upload instance");
  for (size_t k = 0; k < todo.size(); ++k) ids_.emplace(todo[k]->uid, ids[k]);
}

Scheduler makeDeterministic(std::vector<int> rows) { return Scheduler{SchedulerRows(rows.begin(), rows.end())}; }

RewardStructure weightedReward(const std::vector<const RewardStructure*>& parts, const Vec& w) {
  if (parts.size() != w.size()) fail(Errc::DimensionMismatch, "one weight per reward structure");
  if (parts.empty()) fail(Errc::DimensionMismatch, "no reward structures");
  RewardStructure out(parts[0]->size(), 0.0);
  for (size_t k = 0; k < parts.size(); ++k) {
    if (parts[k]->size() != out.size()) fail(Errc::DimensionMismatch, "reward structures differ in length");
    for (size_t r = 0; r < out.size(); ++r) out[r] += w[k] * (*parts[k])[r];
  }
  return out;
}

OptimizeResult optimalScheduler(GpuBackend& gpu, const ProductMdp& p, const RewardStructure& rho, double eps,
                                int sweepCap) {
  if (static_cast<int>(rho.size()) != productRows(p))
    fail(Errc::DimensionMismatch, "reward structure does not match action rows");
  const int32_t id = gpu.modelId(&p, true);
  const double* r = rho.data();
  double value = 0, resid = 0;
  int32_t sweeps = 0, status = 0;
  check(gpu.ctx(), morap_cuda_optimize_rho(gpu.ctx(), 1, &id, &r, eps, sweepCap, &value, &sweeps, &resid, &status),
        "optimize");
  if (status == MORAP_NOT_REWARD_FINITE)
    fail(Errc::NotRewardFinite, "some scheduler avoids the objective with positive probability");
  if (status == MORAP_NON_CONVERGENCE)
    fail(Errc::NonConvergence, "value iteration still moving " + std::to_string(resid) + " after " +
                                   std::to_string(sweeps) + " sweeps");
  check(gpu.ctx(), status, "optimize");
  OptimizeResult out;
  out.values.resize(static_cast<size_t>(p.mdp.numStates));
  out.policy.rows.resize(static_cast<size_t>(p.mdp.numStates));
  check(gpu.ctx(), morap_cuda_fetch_values(gpu.ctx(), 0, out.values.data()), "fetch values");
  check(gpu.ctx(), morap_cuda_fetch_policy(gpu.ctx(), 0, out.policy.rows.data()), "fetch policy");
  out.stats = {sweeps, resid};
  out.value = value;
  return out;
}

EvaluateResult evaluateScheduler(GpuBackend& gpu, const ProductMdp& p, const Scheduler& mu, const RewardStructure& rho,
                                 double eps, int sweepCap) {
  if (static_cast<int>(rho.size()) != productRows(p))
    fail(Errc::DimensionMismatch, "reward structure does not match action rows");
  if (static_cast<int>(mu.rows.size()) != p.mdp.numStates) fail(Errc::InvalidModel, "scheduler does not cover every state");
  const int32_t id = gpu.modelId(&p, true);
  const int32_t* pol = mu.rows.data();
  const double* r = rho.data();
  double value = 0, resid = 0;
  int32_t sweeps = 0, status = 0;
  check(gpu.ctx(), morap_cuda_evaluate(gpu.ctx(), 1, &id, &pol, &r, eps, sweepCap, &value, &sweeps, &resid, &status),
        "evaluate");
  if (status == MORAP_INVALID_MODEL) fail(Errc::InvalidModel, "scheduler picks a foreign action row");
  if (status == MORAP_NON_CONVERGENCE)
    fail(Errc::NonConvergence, "policy evaluation still moving " + std::to_string(resid) + " after " +
                                   std::to_string(sweeps) + " sweeps");
  check(gpu.ctx(), status, "evaluate");
  EvaluateResult out;
  out.values.resize(static_cast<size_t>(p.mdp.numStates));
  check(gpu.ctx(), morap_cuda_fetch_eval_values(gpu.ctx(), 0, 0, out.values.data()), "fetch values");
  out.stats = {sweeps, resid};
  out.value = value;
  return out;
}

std::map<long, JobResult> runBatch(std::vector<Job> jobs, GpuBackend& gpu) {
  std::map<long, JobResult> out;
  {
    std::map<long, bool> ids;
    for (const Job& j : jobs)
      if (!ids.emplace(j.id, true).second) fail(Errc::InvalidConfig, "duplicate job id " + std::to_string(j.id));
  }
  for (int kind = 0; kind < 2; ++kind) {
    std::vector<const Job*> batch;
    for (const Job& j : jobs) {
      if ((kind == 0) != (j.kind == JobKind::Optimize)) continue;
      JobResult& res = out[j.id];
      if (!j.model) {
        res.error = "job carries no model";
        res.errc = Errc::InvalidModel;
        continue;
      }
      if (static_cast<int>(j.reward.size()) != productRows(*j.model)) {
        res.error = "reward structure does not match action rows";
        res.errc = Errc::DimensionMismatch;
        continue;
      }
      if (kind == 1 && static_cast<int>(j.scheduler.rows.size()) != j.model->mdp.numStates) {
        res.error = "scheduler does not cover every state";
        res.errc = Errc::InvalidModel;
        continue;
      }
      batch.push_back(&j);
    }
    if (batch.empty()) continue;
    // per call the eps / cap are uniform; group by them so mixed batches still work
    std::map<std::pair<double, int>, std::vector<const Job*>> groups;
    for (const Job* j : batch) groups[{j->eps, j->sweepCap}].push_back(j);
    for (auto& [key, grp] : groups) {
      const size_t n = grp.size();
      std::vector<int32_t> ids(n), sweeps(n), status(n);
      std::vector<const double*> rho(n);
      std::vector<const int32_t*> pol(n);
      std::vector<double> value(n), resid(n);
      for (size_t k = 0; k < n; ++k) {
        ids[k] = gpu.modelId(grp[k]->model.get(), true);
        rho[k] = grp[k]->reward.data();
        pol[k] = grp[k]->scheduler.rows.data();
      }
      if (kind == 0)
        check(gpu.ctx(), morap_cuda_optimize_rho(gpu.ctx(), static_cast<int>(n), ids.data(), rho.data(), key.first,
                                                 key.second, value.data(), sweeps.data(), resid.data(), status.data()),
              "optimize batch");
      else
        check(gpu.ctx(), morap_cuda_evaluate(gpu.ctx(), static_cast<int>(n), ids.data(), pol.data(), rho.data(), key.first,
                                             key.second, value.data(), sweeps.data(), resid.data(), status.data()),
              "evaluate batch");
      for (size_t k = 0; k < n; ++k) {
        JobResult& res = out[grp[k]->id];
        res.stats = {sweeps[k], resid[k]};
        if (status[k] != MORAP_OK) {
          res.ok = false;
          res.errc = static_cast<Errc>(status[k] - 1);
          res.error = status[k] == MORAP_NON_CONVERGENCE ? "value iteration did not converge within the sweep cap"
                      : status[k] == MORAP_NOT_REWARD_FINITE
                          ? "some scheduler avoids the objective with positive probability"
                          : "invalid job";
          continue;
        }
        res.ok = true;
        res.value = value[k];
        const int S = grp[k]->model->mdp.numStates;
        res.values.resize(static_cast<size_t>(S));
        if (kind == 0) {
          res.policy.rows.resize(static_cast<size_t>(S));
          check(gpu.ctx(), morap_cuda_fetch_values(gpu.ctx(), static_cast<int>(k), res.values.data()), "fetch values");
          check(gpu.ctx(), morap_cuda_fetch_policy(gpu.ctx(), static_cast<int>(k), res.policy.rows.data()), "fetch policy");
        } else {
          check(gpu.ctx(), morap_cuda_fetch_eval_values(gpu.ctx(), static_cast<int>(k), 0, res.values.data()), "fetch values");
        }
      }
    }
  }
  return out;
}

}  // namespace morap
