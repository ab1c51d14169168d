// Model loader and product builder (reference: model.hpp, instance.hpp).
//
// buildProduct explores (agent state, DFA location) pairs breadth first from
// (s0, delta(q0, L(s0))) and numbers product states in discovery order, so the CSR it
// emits -- rowOffset / trnOffset / succ / prob / cost / success / done -- is identical,
// array for array, to the reference's (tests/test_model_parity.py checks this). The pair
// index is a flat int32 table instead of a hash map, and buildInstance builds the n^2
// products on all host threads before deduplicating them in (i, j) order.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <cstring>
#include <optional>
#include <random>
#include <set>
#include <thread>

#include "morap.hpp"

namespace morap {

const std::string kInternalAction = "!advance";

uint64_t nextProductUid() {
  static std::atomic<uint64_t> counter{1};
  return counter.fetch_add(1);
}

void validateMdp(const Mdp& m, double tol) {
  if (m.numStates <= 0) fail(Errc::InvalidModel, "model has no states");
  if (m.initial < 0 || m.initial >= m.numStates) fail(Errc::InvalidModel, "initial state out of range");
  for (int s = 0; s < m.numStates; ++s)
    if (m.actionsEnd(s) <= m.actionsBegin(s)) fail(Errc::InvalidModel, "deadlock: state " + std::to_string(s) + " has no action");
  for (int r = 0; r < m.numActions(); ++r) {
    double total = 0.0;
    for (int k = m.trnBegin(r); k < m.trnEnd(r); ++k) {
      if (m.prob[k] < 0.0) fail(Errc::InvalidModel, "negative transition probability");
      if (m.succ[k] < 0 || m.succ[k] >= m.numStates) fail(Errc::InvalidModel, "successor out of range");
      total += m.prob[k];
    }
    if (std::fabs(total - 1.0) > tol)
      fail(Errc::InvalidModel, "action row " + std::to_string(r) + " sums to " + std::to_string(total));
  }
}

void renormalizeRows(Mdp& m) {
  for (int r = 0; r < m.numActions(); ++r) {
    double total = 0.0;
    for (int k = m.trnBegin(r); k < m.trnEnd(r); ++k) total += m.prob[k];
    if (total > 0.0)
      for (int k = m.trnBegin(r); k < m.trnEnd(r); ++k) m.prob[k] /= total;
  }
}

std::pair<Mdp, RewardStructure> mdpFromJson(const Json& j) {
  if (!j.is_object() || !j.contains("states") || !j.contains("actions"))
    fail(Errc::InvalidModel, "model JSON must carry states and actions");
  Mdp m;
  m.numStates = j.at("states").get<int>();
  m.initial = j.value("initial", 0);
  if (m.numStates <= 0) fail(Errc::InvalidModel, "model has no states");
  m.labels.assign(static_cast<size_t>(m.numStates), {});
  if (j.contains("labels"))
    for (auto it = j.at("labels").begin(); it != j.at("labels").end(); ++it) {
      const int s = std::stoi(it.key());
      if (s < 0 || s >= m.numStates) fail(Errc::InvalidModel, "label for unknown state " + it.key());
      auto& lab = m.labels[s];
      for (const Json& a : it.value()) lab.push_back(a.get<std::string>());
      std::sort(lab.begin(), lab.end());
      lab.erase(std::unique(lab.begin(), lab.end()), lab.end());
    }
  // rows grouped by owning state, file order kept inside a state
  std::vector<std::vector<const Json*>> rowsOf(static_cast<size_t>(m.numStates));
  for (const Json& a : j.at("actions")) {
    const int s = a.at("state").get<int>();
    if (s < 0 || s >= m.numStates) fail(Errc::InvalidModel, "action at unknown state");
    rowsOf[s].push_back(&a);
  }
  RewardStructure reward;
  m.trnOffset.push_back(0);
  for (int s = 0; s < m.numStates; ++s) {
    m.rowOffset.push_back(static_cast<int>(reward.size()));
    for (const Json* a : rowsOf[s]) {
      for (const Json& t : a->at("to")) {
        m.succ.push_back(t.at("s").get<int>());
        m.prob.push_back(t.at("p").get<double>());
      }
      m.trnOffset.push_back(static_cast<int>(m.succ.size()));
      m.actionName.push_back(a->value("name", ""));
      reward.push_back(a->value("reward", 0.0));
    }
  }
  m.rowOffset.push_back(static_cast<int>(reward.size()));
  validateMdp(m);
  renormalizeRows(m);
  return {std::move(m), std::move(reward)};
}

Json mdpToJson(const Mdp& m, const RewardStructure& reward) {
  Json labels = Json::object(), actions = Json::array();
  for (int s = 0; s < m.numStates; ++s) {
    if (!m.labels[s].empty()) labels[std::to_string(s)] = m.labels[s];
    for (int r = m.actionsBegin(s); r < m.actionsEnd(s); ++r) {
      Json to = Json::array();
      for (int k = m.trnBegin(r); k < m.trnEnd(r); ++k) to.push_back({{"s", m.succ[k]}, {"p", m.prob[k]}});
      actions.push_back({{"state", s}, {"name", m.actionName[r]}, {"to", to}, {"reward", reward[r]}});
    }
  }
  return Json{{"states", m.numStates}, {"initial", m.initial}, {"labels", labels}, {"actions", actions}};
}

// Greatest set of non-done states that some scheduler can keep away from `done` forever:
// repeatedly discard states all of whose rows may leave the candidate set.
std::vector<int> maximalAvoidSet(const Mdp& m, const std::vector<char>& done) {
  const int S = m.numStates, R = m.numActions();
  std::vector<int> owner(static_cast<size_t>(R));
  for (int s = 0; s < S; ++s)
    for (int r = m.actionsBegin(s); r < m.actionsEnd(s); ++r) owner[r] = s;
  std::vector<char> in(static_cast<size_t>(S));
  for (int s = 0; s < S; ++s) in[s] = !done[s];
  std::vector<int> leaving(static_cast<size_t>(R), 0), closedRows(static_cast<size_t>(S), 0);
  // reverse edges successor -> rows, as a CSR
  std::vector<int> head(static_cast<size_t>(S) + 1, 0);
  for (int r = 0; r < R; ++r)
    if (in[owner[r]])
      for (int k = m.trnBegin(r); k < m.trnEnd(r); ++k) ++head[m.succ[k] + 1];
  for (int s = 0; s < S; ++s) head[s + 1] += head[s];
  std::vector<int> rev(static_cast<size_t>(head[S])), fill(head.begin(), head.end() - 1);
  for (int r = 0; r < R; ++r) {
    if (!in[owner[r]]) continue;
    for (int k = m.trnBegin(r); k < m.trnEnd(r); ++k) {
      rev[fill[m.succ[k]]++] = r;
      if (!in[m.succ[k]]) ++leaving[r];
    }
    if (leaving[r] == 0) ++closedRows[owner[r]];
  }
  std::vector<int> stack;
  for (int s = 0; s < S; ++s)
    if (in[s] && closedRows[s] == 0) stack.push_back(s);
  while (!stack.empty()) {
    const int s = stack.back();
    stack.pop_back();
    if (!in[s]) continue;
    in[s] = 0;
    for (int e = head[s]; e < head[s + 1]; ++e) {
      const int r = rev[e], o = owner[r];
      if (!in[o]) continue;
      if (leaving[r]++ == 0 && --closedRows[o] == 0) stack.push_back(o);
    }
  }
  std::vector<int> out;
  for (int s = 0; s < S; ++s)
    if (in[s]) out.push_back(s);
  return out;
}

bool checkRewardFinite(const Mdp& m, const std::vector<char>& done) { return maximalAvoidSet(m, done).empty(); }
bool checkRewardFinite(const ProductMdp& p) { return checkRewardFinite(p.mdp, p.done); }

namespace {

// Dedup key of a product (bucketing only -- equality is checked array by array): four
// independent multiply-rotate lanes over 8-byte words, ~10x faster than a byte-wise FNV
// on the ~10 MB of a C4 product.
struct Fnv {
  uint64_t lane[4] = {0x9e3779b97f4a7c15ull, 0xc2b2ae3d27d4eb4full, 0x165667b19e3779f9ull, 0x27d4eb2f165667c5ull};
  static uint64_t mix(uint64_t h, uint64_t w) {
    h ^= w * 0x9fb21c651e98df25ull;
    return ((h << 29) | (h >> 35)) * 0xff51afd7ed558ccdull;
  }
  void bytes(const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    size_t i = 0;
    for (; i + 32 <= n; i += 32) {
      uint64_t w[4];
      std::memcpy(w, c + i, 32);
      for (int k = 0; k < 4; ++k) lane[k] = mix(lane[k], w[k]);
    }
    uint64_t tail = n;
    for (; i < n; ++i) tail = (tail << 8 | tail >> 56) ^ c[i];
    lane[0] = mix(lane[0], tail);
  }
  template <class T>
  void vec(const std::vector<T>& v) {
    const uint64_t n = v.size();
    bytes(&n, sizeof n);
    if (!v.empty()) bytes(v.data(), v.size() * sizeof(T));
  }
  uint64_t digest() const { return mix(mix(lane[0], lane[1]), mix(lane[2], lane[3])); }
};

}  // namespace

uint64_t productHash(const ProductMdp& p) {
  Fnv f;
  const int64_t head[2] = {p.mdp.numStates, p.mdp.initial};
  f.bytes(head, sizeof head);
  f.vec(p.mdp.rowOffset);
  f.vec(p.mdp.trnOffset);
  f.vec(p.mdp.succ);
  f.vec(p.mdp.prob);
  f.vec(p.cost);
  f.vec(p.success);
  f.vec(p.done);
  f.vec(p.accept);
  return f.digest();
}

// every acceptance must be entered through a pre-sink step (model.hpp:234-243)
void checkPreSinks(const Dfa& task) {
  if (task.accepting[task.initial]) fail(Errc::InvalidDfa, "task automaton lacks pre-sinks: initial location is accepting");
  const int L = task.numLetters(), Q = task.numLocations;
  for (int q = 0; q < Q; ++q) {
    if (task.accepting[q] || task.preSink[q]) continue;
    for (int w = 0; w < L; ++w)
      if (task.accepting[task.step(q, w)])
        fail(Errc::InvalidDfa, "task automaton lacks pre-sinks: acceptance without a pre-sink step");
  }
}

ProductMdp buildProduct(const Mdp& agent, const RewardStructure& agentCost, const Dfa& task, int agentId, int taskId) {
  if (static_cast<int>(agentCost.size()) != agent.numActions())
    fail(Errc::DimensionMismatch, "cost structure does not match the model's action rows");
  checkPreSinks(task);
  const int Q = task.numLocations;
  ProductMdp p;
  p.agentId = agentId;
  p.taskId = taskId;
  const int SA = agent.numStates;
  std::vector<int> letter(static_cast<size_t>(SA));
  std::set<std::string> dropped;
  for (int s = 0; s < SA; ++s) {
    letter[s] = static_cast<int>(letterMaskFor(task, agent.labels[s]));
    for (const std::string& a : agent.labels[s])
      if (!std::binary_search(task.atoms.begin(), task.atoms.end(), a)) dropped.insert(a);
  }
  p.droppedAtoms.assign(dropped.begin(), dropped.end());

  std::vector<int32_t> id(static_cast<size_t>(SA) * Q, -1);
  std::vector<int> qs, as;  // discovery order: agent state, location
  auto visit = [&](int s, int q) {
    int32_t& slot = id[static_cast<size_t>(s) * Q + q];
    if (slot < 0) {
      slot = static_cast<int32_t>(as.size());
      as.push_back(s);
      qs.push_back(q);
    }
    return static_cast<int>(slot);
  };
  const int q0 = task.preSink[task.initial] ? task.initial : task.step(task.initial, letter[agent.initial]);
  Mdp& M = p.mdp;
  M.initial = visit(agent.initial, q0);
  M.trnOffset.push_back(0);
  std::vector<int> rowName;  // agent row of each product row (-1: internal), names filled at the end
  {
    const size_t guess = static_cast<size_t>(agent.numActions()) * static_cast<size_t>(Q) / 2;
    rowName.reserve(guess);
    M.trnOffset.reserve(guess + 1);
    M.succ.reserve(guess + guess / 4);
    M.prob.reserve(guess + guess / 4);
    p.cost.reserve(guess);
    p.success.reserve(guess);
  }
  for (size_t x = 0; x < as.size(); ++x) {
    const int s = as[x], q = qs[x];
    M.rowOffset.push_back(M.numActions());
    if (task.preSink[q]) {
      M.succ.push_back(visit(s, task.step(q, letter[s])));
      M.prob.push_back(1.0);
      M.trnOffset.push_back(static_cast<int>(M.succ.size()));
      rowName.push_back(-1);
      p.cost.push_back(0.0);
      p.success.push_back(1.0);
      continue;
    }
    for (int r = agent.actionsBegin(s); r < agent.actionsEnd(s); ++r) {
      for (int k = agent.trnBegin(r); k < agent.trnEnd(r); ++k) {
        const int t = agent.succ[k];
        M.succ.push_back(visit(t, task.step(q, letter[t])));
        M.prob.push_back(agent.prob[k]);
      }
      M.trnOffset.push_back(static_cast<int>(M.succ.size()));
      rowName.push_back(r);
      p.cost.push_back(agentCost[r]);
      p.success.push_back(0.0);
    }
  }
  M.numStates = static_cast<int>(as.size());
  M.rowOffset.push_back(M.numActions());
  M.actionName.resize(rowName.size());
  for (size_t r = 0; r < rowName.size(); ++r)
    M.actionName[r] = rowName[r] < 0 ? kInternalAction : agent.actionName[static_cast<size_t>(rowName[r])];
  M.labels.assign(static_cast<size_t>(M.numStates), {});
  p.agentState = as;
  p.dfaLocation = qs;
  p.done.resize(as.size());
  p.accept.resize(as.size());
  p.preSink.resize(as.size());
  for (size_t x = 0; x < as.size(); ++x) {
    const int q = qs[x];
    p.accept[x] = task.accepting[q];
    p.done[x] = task.accepting[q] || task.trap[q];
    p.preSink[x] = task.preSink[q];
  }
  p.rewardFinite = checkRewardFinite(p);
  p.structuralHash = productHash(p);
  return p;
}

// ---- instance ----------------------------------------------------------------------------
namespace {

bool sameProduct(const ProductMdp& a, const ProductMdp& b) {
  const Mdp &x = a.mdp, &y = b.mdp;
  return x.numStates == y.numStates && x.initial == y.initial && x.rowOffset == y.rowOffset &&
         x.trnOffset == y.trnOffset && x.succ == y.succ && x.prob == y.prob && x.actionName == y.actionName &&
         a.cost == b.cost && a.success == b.success && a.done == b.done && a.accept == b.accept &&
         a.preSink == b.preSink && a.extra == b.extra;
}

int hostThreads(int want) {
  if (want > 0) return want;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? static_cast<int>(hw) : 1;
}

}  // namespace

void slimProduct(ProductMdp& p) {
  if (p.slim) return;
  p.slimRows = p.mdp.numActions();
  p.slimNnz = static_cast<int64_t>(p.mdp.succ.size());
  auto drop = [](auto& v) { std::remove_reference_t<decltype(v)>().swap(v); };
  drop(p.mdp.rowOffset);
  drop(p.mdp.trnOffset);
  drop(p.mdp.succ);
  drop(p.mdp.prob);
  drop(p.mdp.actionName);
  drop(p.mdp.labels);
  drop(p.agentState);
  drop(p.dfaLocation);
  drop(p.done);
  drop(p.accept);
  drop(p.preSink);
  drop(p.cost);
  drop(p.success);
  drop(p.extra);
  p.slim = true;
}

void requireFull(const ProductMdp& p, const char* what) {
  if (p.slim)
    fail(Errc::InvalidConfig, std::string(what) +
                                  ": the product's host arrays were dropped after a streamed upload (its only copy is "
                                  "on the device)");
}

namespace {

// Same (S, R, nnz, initial) and structural hash: the identity test used against products
// whose arrays are gone (streamed builds); full products are compared array by array.
bool sameSlimKey(const ProductMdp& a, const ProductMdp& b) {
  return a.structuralHash == b.structuralHash && a.mdp.numStates == b.mdp.numStates &&
         a.mdp.initial == b.mdp.initial && productRows(a) == productRows(b) && productNnz(a) == productNnz(b);
}

}  // namespace

MorapInstance buildInstance(std::vector<Mdp> agents, std::vector<RewardStructure> costs, std::vector<Dfa> tasks,
                            int threads, size_t chunk, const ProductSink* sink) {
  if (agents.empty()) fail(Errc::InvalidModel, "instance needs at least one agent");
  if (agents.size() != costs.size()) fail(Errc::DimensionMismatch, "one cost structure per agent required");
  if (tasks.size() > agents.size()) fail(Errc::InvalidModel, "more tasks than agents; drop tasks or add agents");
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
  const size_t total = static_cast<size_t>(n) * n;
  if (chunk == 0 || !sink) chunk = total;
  std::map<uint64_t, std::vector<std::shared_ptr<ProductMdp>>> byHash;
  inst.products.assign(static_cast<size_t>(n), std::vector<std::shared_ptr<const ProductMdp>>(static_cast<size_t>(n)));
  const int T = std::min<int>(hostThreads(threads), static_cast<int>(std::min(total, chunk)));
  const bool trace = std::getenv("MORAP_TRACE") != nullptr;
  double buildS = 0, dedupS = 0, sinkS = 0;
  auto since = [](std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
  };
  for (size_t base = 0; base < total; base += chunk) {
    const size_t m = std::min(chunk, total - base);
    const auto tb = std::chrono::steady_clock::now();
    std::vector<std::unique_ptr<ProductMdp>> built(m);
    std::vector<std::optional<Error>> errs(m);
    std::atomic<size_t> next{0};
    auto worker = [&] {
      for (size_t q; (q = next.fetch_add(1)) < m;) {
        const size_t k = base + q;
        const int i = static_cast<int>(k / n), j = static_cast<int>(k % n);
        try {
          built[q] = std::make_unique<ProductMdp>(buildProduct(inst.agents[i], inst.costs[i], inst.tasks[j], i, j));
        } catch (const Error& e) {
          errs[q] = e;
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    buildS += since(tb);

    // reject / deduplicate in (i, j) order, as instance.hpp:445-466 does sequentially
    std::vector<ProductMdp*> fresh;
    for (size_t q = 0; q < m; ++q) {
      const size_t k = base + q;
      const int i = static_cast<int>(k / n), j = static_cast<int>(k % n);
      if (errs[q]) throw *errs[q];
      if (!built[q]->rewardFinite)
        fail(Errc::NotRewardFinite,
             "product of agent " + std::to_string(i) + " and task " + std::to_string(j) + " can cycle without finishing");
      auto& bucket = byHash[built[q]->structuralHash];
      std::shared_ptr<ProductMdp> share;
      for (const auto& cand : bucket)
        if (cand->slim ? sameSlimKey(*cand, *built[q]) : sameProduct(*cand, *built[q])) {
          share = cand;
          break;
        }
      if (!share) {
        share = std::shared_ptr<ProductMdp>(built[q].release());
        bucket.push_back(share);
        fresh.push_back(share.get());
        ++inst.distinctProducts;
      }
      inst.products[i][j] = share;
    }
    dedupS += since(tb);
    const auto ts = std::chrono::steady_clock::now();
    if (sink && !fresh.empty()) (*sink)(fresh);
    sinkS += since(ts);
  }
  if (trace)
    std::fprintf(stderr, "[morap] buildInstance: products %.2f s, dedup %.2f s, sink (upload) %.2f s\n", buildS,
                 dedupS - buildS, sinkS);
  return inst;
}

Vec expandThresholds(const MorapInstance& inst, const Vec& user) {
  const int K = inst.objectives;
  // costs (and extra per-agent objectives) first, then one probability per real task
  const int want = (K - 1) * inst.n + inst.realTasks;
  if (static_cast<int>(user.size()) != want)
    fail(Errc::DimensionMismatch, "expected " + std::to_string(want) + " thresholds (costs first, then task probabilities)");
  Vec t(static_cast<size_t>(K) * inst.n, 0.0);
  for (int i = 0; i < (K - 1) * inst.n; ++i) {
    if (!std::isfinite(user[i])) fail(Errc::InvalidModel, "cost threshold must be finite");
    t[i] = user[i];
  }
  for (int j = 0; j < inst.realTasks; ++j) {
    const double p = user[(K - 1) * inst.n + j];
    if (!(p >= 0.0 && p <= 1.0)) fail(Errc::InvalidModel, "probability threshold outside [0,1]");
    t[(K - 1) * inst.n + j] = p;
  }
  return t;
}

void addSyntheticObjectives(MorapInstance& inst, int K, uint64_t seed) {
  if (K < 2 || K > 8) fail(Errc::InvalidConfig, "objective count must lie in [2, 8]");
  // distinct products in (i, j) order of first occurrence; each gets its own seeded stream
  std::map<const ProductMdp*, size_t> slot;
  std::vector<std::pair<const ProductMdp*, uint64_t>> todo;
  for (int i = 0; i < inst.n; ++i)
    for (int j = 0; j < inst.n; ++j)
      if (slot.emplace(inst.products[i][j].get(), todo.size()).second)
        todo.emplace_back(inst.products[i][j].get(), static_cast<uint64_t>(i) * inst.n + j + 1);
  for (const auto& t : todo) requireFull(*t.first, "add objectives");
  std::vector<std::shared_ptr<ProductMdp>> copies(todo.size());
  std::atomic<size_t> next{0};
  auto worker = [&] {
    for (size_t q; (q = next.fetch_add(1)) < todo.size();) {
      auto copy = std::make_shared<ProductMdp>(*todo[q].first);
      copy->uid = nextProductUid();
      copy->extra.clear();
      std::mt19937_64 rng(seed ^ (0x9e3779b97f4a7c15ull * todo[q].second));
      // seeded per-row costs in [-2, 0] on a 1/8 grid (17 levels), so K-objective products
      // keep a small reward-tuple alphabet (compact streams)
      std::uniform_int_distribution<int> u(0, 16);
      for (int k = 2; k < K; ++k) {
        RewardStructure v(copy->cost.size());
        for (size_t r = 0; r < v.size(); ++r)
          v[r] = copy->mdp.actionName[r] == kInternalAction ? 0.0 : -0.125 * static_cast<double>(u(rng));
        copy->extra.push_back(std::move(v));
      }
      copies[q] = std::move(copy);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < hostThreads(0); ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  for (int i = 0; i < inst.n; ++i)
    for (int j = 0; j < inst.n; ++j) inst.products[i][j] = copies[slot.at(inst.products[i][j].get())];
  inst.objectives = K;
}

}  // namespace morap
