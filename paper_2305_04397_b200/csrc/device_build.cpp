// buildInstance (instance.hpp:42-91) with the products built on the GPU.
//
// The host side keeps what is cheap and sequential: validation (the same checks and error
// texts as buildInstance / buildProduct), the alphabets the device kernel indexes (distinct
// probabilities, costs, action names and label sets over all agents, by exact bits / value),
// each task's letter per label set (letterMaskFor), the reject / dedup pass in (i, j) order
// and the slim ProductMdp records. morap_cuda_build_products does the rest: a measure pass
// over every pair (sizes, reward finiteness, identity hash), then the write pass over the
// distinct products only.
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

}  // namespace

MorapInstance buildInstanceOnDevice(GpuBackend& gpu, std::vector<Mdp> agents, std::vector<RewardStructure> costs,
                                    std::vector<Dfa> tasks) {
  if (agents.empty()) fail(Errc::InvalidModel, "instance needs at least one agent");
  if (agents.size() != costs.size()) fail(Errc::DimensionMismatch, "one cost structure per agent required");
  if (tasks.size() > agents.size()) fail(Errc::InvalidModel, "more tasks than agents; drop tasks or add agents");
  const bool trace = std::getenv("MORAP_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto since = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  MorapInstance inst;
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
  struct AgentArrays {
    std::vector<int32_t> pc, cc, name, lset;
  };
  std::vector<AgentArrays> aa(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    const Mdp& m = inst.agents[i];
    AgentArrays& a = aa[i];
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
  std::vector<double> probs(probIds.size()), costVals(costIds.size());
  for (const auto& [b, id] : probIds) std::memcpy(&probs[id], &b, 8);
  for (const auto& [b, id] : costIds) std::memcpy(&costVals[id], &b, 8);
  std::vector<const std::vector<std::string>*> sets(labelIds.size());
  for (const auto& [labels, id] : labelIds) sets[id] = &labels;

  std::vector<morap_build_agent> ba(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    const Mdp& m = inst.agents[i];
    ba[i] = morap_build_agent{m.numStates,         m.numActions(),      static_cast<int32_t>(m.succ.size()),
                              m.initial,           m.rowOffset.data(),  m.trnOffset.data(),
                              m.succ.data(),       aa[i].pc.data(),     aa[i].cc.data(),
                              aa[i].name.data(),   aa[i].lset.data()};
  }
  struct TaskArrays {
    std::vector<uint8_t> flags;
    std::vector<int32_t> letter;
  };
  std::vector<TaskArrays> ta(static_cast<size_t>(n));
  std::vector<morap_build_task> bt(static_cast<size_t>(n));
  for (int j = 0; j < n; ++j) {
    const Dfa& d = inst.tasks[j];
    ta[j].flags.resize(static_cast<size_t>(d.numLocations));
    for (int q = 0; q < d.numLocations; ++q)
      ta[j].flags[q] = static_cast<uint8_t>((d.accepting[q] ? 1 : 0) | (d.trap[q] ? 2 : 0) | (d.preSink[q] ? 4 : 0));
    ta[j].letter.resize(sets.size());
    for (size_t l = 0; l < sets.size(); ++l) ta[j].letter[l] = static_cast<int32_t>(letterMaskFor(d, *sets[l]));
    bt[j] = morap_build_task{d.numLocations, d.numLetters(), d.initial, d.delta.data(), ta[j].flags.data(),
                             ta[j].letter.data()};
  }
  const morap_build_alphabet alpha{static_cast<int32_t>(probs.size()), static_cast<int32_t>(costVals.size()),
                                   internalName, static_cast<int32_t>(sets.size()), probs.data(), costVals.data()};
  const size_t total = static_cast<size_t>(n) * n;
  std::vector<int32_t> pairs(2 * total);
  for (size_t k = 0; k < total; ++k) {
    pairs[2 * k] = static_cast<int32_t>(k / n);
    pairs[2 * k + 1] = static_cast<int32_t>(k % n);
  }
  const double prepS = since();
  std::vector<morap_build_info> info(total);
  check(gpu.ctx(),
        morap_cuda_build_products(gpu.ctx(), n, ba.data(), n, bt.data(), &alpha, static_cast<int>(total), pairs.data(), 0,
                                  info.data(), nullptr),
        "device product build (measure)");
  const double measureS = since();

  // reject / deduplicate in (i, j) order (buildInstance; identity = hash + dimensions, as for
  // every product whose arrays live on the device only)
  inst.products.assign(static_cast<size_t>(n), std::vector<std::shared_ptr<const ProductMdp>>(static_cast<size_t>(n)));
  std::map<uint64_t, std::vector<std::shared_ptr<ProductMdp>>> byHash;
  std::vector<int32_t> freshPairs;
  std::vector<morap_build_info> freshInfo;
  std::vector<ProductMdp*> fresh;
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
      fresh.push_back(share.get());
      freshPairs.push_back(i);
      freshPairs.push_back(j);
      freshInfo.push_back(b);
      ++inst.distinctProducts;
    }
    inst.products[i][j] = share;
  }
  std::vector<int32_t> ids(fresh.size());
  check(gpu.ctx(),
        morap_cuda_build_products(gpu.ctx(), n, ba.data(), n, bt.data(), &alpha, static_cast<int>(fresh.size()),
                                  freshPairs.data(), 1, freshInfo.data(), ids.data()),
        "device product build (write)");
  for (size_t k = 0; k < fresh.size(); ++k) gpu.adopt(fresh[k]->uid, ids[k]);
  if (trace)
    std::fprintf(stderr,
                 "[morap] buildInstanceOnDevice: %zu pairs, %d distinct: host prep %.3f s, measure %.3f s, write %.3f s\n",
                 total, inst.distinctProducts, prepS, measureS - prepS, since() - measureS);
  return inst;
}

}  // namespace morap
