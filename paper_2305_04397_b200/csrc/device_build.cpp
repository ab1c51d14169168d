// buildInstance (instance.hpp:42-91) with the products built on the GPU.
//
// The host side keeps what is cheap and sequential: validation (the same checks and error
// texts as buildInstance / buildProduct), the alphabets the device kernel indexes (distinct
// probabilities, costs, action names and label sets over all agents, by exact bits / value),
// each task's letter per label set (letterMaskFor), the reject / dedup pass in (i, j) order
// and the slim ProductMdp records. morap_cuda_build_products does the rest: a measure pass
// over every pair (sizes, reward finiteness, identity hash), then the write pass over the
// distinct products only -- on one device, or split over the shards' devices.
#include <chrono>
#include <cstring>
#include <map>

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

uint64_t bitsOf(double d) {
  uint64_t b;
  std::memcpy(&b, &d, sizeof b);
  return b;
}

template <class K>
int intern(std::map<K, int>& ids, const K& key) {
  return ids.emplace(key, static_cast<int>(ids.size())).first->second;
}

bool traceOn() { return std::getenv("MORAP_TRACE") != nullptr; }

}  // namespace

struct DeviceBuild::Inputs {
  struct AgentArrays {
    std::vector<int32_t> pc, cc, name, lset;
  };
  struct TaskArrays {
    std::vector<uint8_t> flags;
    std::vector<int32_t> letter;
  };
  std::vector<AgentArrays> aa;
  std::vector<TaskArrays> ta;
  std::vector<double> probs, costs;
  std::vector<morap_build_agent> agents;
  std::vector<morap_build_task> tasks;
  morap_build_alphabet alpha{};
  std::vector<int32_t> pairs;          // distinct products' (agent, task)
  std::vector<morap_build_info> info;  // their measure results
};

DeviceBuild::DeviceBuild() = default;
DeviceBuild::~DeviceBuild() = default;

std::unique_ptr<DeviceBuild> planDeviceBuild(GpuBackend& gpu, std::vector<Mdp> agents, std::vector<RewardStructure> costs,
                                             std::vector<Dfa> tasks) {
  if (agents.empty()) fail(Errc::InvalidModel, "instance needs at least one agent");
  if (agents.size() != costs.size()) fail(Errc::DimensionMismatch, "one cost structure per agent required");
  if (tasks.size() > agents.size()) fail(Errc::InvalidModel, "more tasks than agents; drop tasks or add agents");
  const auto t0 = std::chrono::steady_clock::now();
  auto since = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  auto plan = std::make_unique<DeviceBuild>();
  plan->in = std::make_unique<DeviceBuild::Inputs>();
  MorapInstance& inst = plan->inst;
  DeviceBuild::Inputs& in = *plan->in;
  inst.n = static_cast<int>(agents.size());
  inst.realTasks = static_cast<int>(tasks.size());
  inst.agents = std::move(agents);
  inst.costs = std::move(costs);
  inst.tasks = std::move(tasks);
  for (int i = 0; i < inst.n; ++i) {
    validateMdp(inst.agents[i]);
    if (static_cast<int>(inst.costs[i].size()) != inst.agents[i].numActions())
      fail(Errc::DimensionMismatch, "cost structure does not match agent action rows");
  }
  if (inst.realTasks < inst.n) inst.tasks.resize(static_cast<size_t>(inst.n), insertPreSinks(formulaToDfa(fTrue())));
  const int n = inst.n;
  // buildProduct's task checks, in the order the products would be built: (0, 0), (0, 1), ...
  for (int j = 0; j < n; ++j) checkPreSinks(inst.tasks[j]);

  // alphabets shared by every product of the instance
  std::map<uint64_t, int> probIds, costIds;
  std::map<std::string, int> nameIds;
  std::map<std::vector<std::string>, int> labelIds;
  intern(probIds, bitsOf(1.0));  // pre-sink steps
  const int internalName = intern(nameIds, kInternalAction);
  in.aa.resize(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    const Mdp& m = inst.agents[i];
    auto& a = in.aa[i];
    a.pc.resize(m.prob.size());
    for (size_t k = 0; k < m.prob.size(); ++k) a.pc[k] = intern(probIds, bitsOf(m.prob[k]));
    a.cc.resize(inst.costs[i].size());
    a.name.resize(inst.costs[i].size());
    for (size_t r = 0; r < inst.costs[i].size(); ++r) {
      a.cc[r] = intern(costIds, bitsOf(inst.costs[i][r]));
      a.name[r] = intern(nameIds, m.actionName[r]);
    }
    a.lset.resize(static_cast<size_t>(m.numStates));
    for (int s = 0; s < m.numStates; ++s) a.lset[s] = intern(labelIds, m.labels[s]);
  }
  in.probs.resize(probIds.size());
  in.costs.resize(costIds.size());
  for (const auto& [b, id] : probIds) std::memcpy(&in.probs[id], &b, 8);
  for (const auto& [b, id] : costIds) std::memcpy(&in.costs[id], &b, 8);
  std::vector<const std::vector<std::string>*> sets(labelIds.size());
  for (const auto& [labels, id] : labelIds) sets[id] = &labels;

  in.agents.resize(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    const Mdp& m = inst.agents[i];
    const auto& a = in.aa[i];
    in.agents[i] = morap_build_agent{m.numStates,     m.numActions(),     static_cast<int32_t>(m.succ.size()),
                                     m.initial,       m.rowOffset.data(), m.trnOffset.data(),
                                     m.succ.data(),   a.pc.data(),        a.cc.data(),
                                     a.name.data(),   a.lset.data()};
  }
  in.ta.resize(static_cast<size_t>(n));
  in.tasks.resize(static_cast<size_t>(n));
  for (int j = 0; j < n; ++j) {
    const Dfa& d = inst.tasks[j];
    auto& t = in.ta[j];
    t.flags.resize(static_cast<size_t>(d.numLocations));
    for (int q = 0; q < d.numLocations; ++q)
      t.flags[q] = static_cast<uint8_t>((d.accepting[q] ? 1 : 0) | (d.trap[q] ? 2 : 0) | (d.preSink[q] ? 4 : 0));
    t.letter.resize(sets.size());
    for (size_t l = 0; l < sets.size(); ++l) t.letter[l] = static_cast<int32_t>(letterMaskFor(d, *sets[l]));
    in.tasks[j] = morap_build_task{d.numLocations, d.numLetters(), d.initial, d.delta.data(), t.flags.data(),
                                   t.letter.data()};
  }
  in.alpha = morap_build_alphabet{static_cast<int32_t>(in.probs.size()), static_cast<int32_t>(in.costs.size()),
                                  internalName, static_cast<int32_t>(sets.size()), in.probs.data(), in.costs.data()};
  const size_t total = static_cast<size_t>(n) * n;
  std::vector<int32_t> pairs(2 * total);
  for (size_t k = 0; k < total; ++k) {
    pairs[2 * k] = static_cast<int32_t>(k / n);
    pairs[2 * k + 1] = static_cast<int32_t>(k % n);
  }
  const double prepS = since();
  std::vector<morap_build_info> info(total);
  check(gpu.ctx(),
        morap_cuda_build_products(gpu.ctx(), n, in.agents.data(), n, in.tasks.data(), &in.alpha,
                                  static_cast<int>(total), pairs.data(), 0, info.data(), nullptr),
        "device product build (measure)");

  // reject / deduplicate in (i, j) order (buildInstance; identity = hash + dimensions, as for
  // every product whose arrays live on the device only)
  inst.products.assign(static_cast<size_t>(n), std::vector<std::shared_ptr<const ProductMdp>>(static_cast<size_t>(n)));
  std::map<uint64_t, std::vector<std::shared_ptr<ProductMdp>>> byHash;
  for (size_t k = 0; k < total; ++k) {
    const int i = static_cast<int>(k / n), j = static_cast<int>(k % n);
    const morap_build_info& b = info[k];
    if (b.status != MORAP_OK)
      fail(Errc::InvalidConfig, "device product builder: product of agent " + std::to_string(i) + " and task " +
                                    std::to_string(j) + " has no compact layout (more than 256 probabilities)");
    if (!b.reward_finite)
      fail(Errc::NotRewardFinite,
           "product of agent " + std::to_string(i) + " and task " + std::to_string(j) + " can cycle without finishing");
    auto& bucket = byHash[b.hash];
    std::shared_ptr<ProductMdp> share;
    for (const auto& cand : bucket)
      if (cand->mdp.numStates == b.num_states && cand->slimRows == b.num_rows && cand->slimNnz == b.nnz) {
        share = cand;
        break;
      }
    if (!share) {
      share = std::make_shared<ProductMdp>();
      ProductMdp& p = *share;
      p.agentId = i;
      p.taskId = j;
      p.mdp.numStates = b.num_states;
      p.mdp.initial = 0;  // the BFS root
      p.rewardFinite = true;
      p.structuralHash = b.hash;
      p.slim = true;
      p.slimRows = b.num_rows;
      p.slimNnz = b.nnz;
      bucket.push_back(share);
      plan->distinct.push_back(share.get());
      in.pairs.push_back(i);
      in.pairs.push_back(j);
      in.info.push_back(b);
      ++inst.distinctProducts;
    }
    inst.products[i][j] = share;
  }
  if (traceOn())
    std::fprintf(stderr, "[morap] planDeviceBuild: %zu pairs, %d distinct: host prep %.3f s, measure %.3f s\n", total,
                 inst.distinctProducts, prepS, since() - prepS);
  return plan;
}

void DeviceBuild::write(GpuBackend& gpu, const std::vector<size_t>& which) const {
  if (which.empty()) return;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<int32_t> pairs;
  std::vector<morap_build_info> info;
  for (size_t k : which) {
    pairs.push_back(in->pairs[2 * k]);
    pairs.push_back(in->pairs[2 * k + 1]);
    info.push_back(in->info[k]);
  }
  std::vector<int32_t> ids(which.size());
  const int n = inst.n;
  check(gpu.ctx(),
        morap_cuda_build_products(gpu.ctx(), n, in->agents.data(), n, in->tasks.data(), &in->alpha,
                                  static_cast<int>(which.size()), pairs.data(), 1, info.data(), ids.data()),
        "device product build (write)");
  for (size_t q = 0; q < which.size(); ++q) gpu.adopt(distinct[which[q]]->uid, ids[q]);
  if (traceOn())
    std::fprintf(stderr, "[morap] DeviceBuild::write: %zu products on device %d in %.3f s\n", which.size(),
                 gpu.device(),
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
}

MorapInstance buildInstanceOnDevice(GpuBackend& gpu, std::vector<Mdp> agents, std::vector<RewardStructure> costs,
                                    std::vector<Dfa> tasks) {
  auto plan = planDeviceBuild(gpu, std::move(agents), std::move(costs), std::move(tasks));
  std::vector<size_t> all(plan->distinct.size());
  for (size_t k = 0; k < all.size(); ++k) all[k] = k;
  plan->write(gpu, all);
  return std::move(plan->inst);
}

}  // namespace morap
