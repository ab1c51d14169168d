// morap.hpp -- host C++ API of the B200 MORAP hot path (libmorap_host.so).
//
// Same surface as the reference library (/root/reference/proj/include/morap/*.hpp): the
// model loader (mdpFromJson, buildProduct, buildInstance, generateInstance), the
// per-model solve (optimalScheduler, evaluateScheduler, runBatch) and the Pareto-point
// query (supportingPoint, paretoPoint, verifyOnly, synthesize). Names, argument meaning
// and error codes follow the reference; the implementation is new. Every Bellman solve
// goes through the C ABI of libmorap_cuda.so (include/morap_cuda.h) -- there is no CPU
// solver in this library.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <type_traits>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "json.hpp"

#include "morap_cuda.h"  // morap_ctx, morap_csr_view

namespace morap {

using Json = nlohmann::json;

// ---- errors (common.hpp:12-45) ----------------------------------------------------------
enum class Errc {
  Syntax, NotCoSafe, ClosureBlowup, InvalidDfa, InvalidModel, NotRewardFinite, NonConvergence,
  SingularSystem, DimensionMismatch, NonSquare, NotBistochastic, NoPerfectMatching, NotPositiveDefinite,
  SolverFailure, DegenerateDirection, SizeGuard, CycleGuard, InvalidConfig, GenerationFailure,
  NoCertificate, Io,
};

class Error : public std::runtime_error {
 public:
  Error(Errc c, const std::string& what) : std::runtime_error(what), code_(c) {}
  Errc code() const noexcept { return code_; }

 private:
  Errc code_;
};

[[noreturn]] void fail(Errc c, const std::string& msg);
inline int statusOf(Errc c) { return static_cast<int>(c) + 1; }

using Vec = std::vector<double>;

struct Mat {
  int rows = 0, cols = 0;
  Vec a;
  Mat() = default;
  Mat(int r, int c, double v = 0.0) : rows(r), cols(c), a(static_cast<size_t>(r) * c, v) {}
  double& operator()(int r, int c) { return a[static_cast<size_t>(r) * cols + c]; }
  double operator()(int r, int c) const { return a[static_cast<size_t>(r) * cols + c]; }
};

// ---- dense linear algebra (common.hpp:47-125) --------------------------------------------
double dot(const Vec& x, const Vec& y);
Vec matVec(const Mat& m, const Vec& x);
double maxAbs(const Vec& v);
Vec solveDense(Mat A, Vec b, double pivotTol = 1e-12);
Vec solveDenseInPlace(Mat& A, Vec& b, double pivotTol = 1e-12);  // A and b are destroyed
// A recorded elimination of solveDense: the row swap and the nonzero multipliers of every
// pivot step, and the upper triangle (left in the caller's matrix, row-major, leading
// dimension lda), so the same system can be solved again for another right-hand side with
// exactly the arithmetic a fresh elimination performs.
struct DenseLU {
  int n = 0, lda = 0;
  double* U = nullptr;  // caller-owned
  std::vector<int> piv;
  // step k's multipliers: (rows[i], f[i]) for i in [stepOff[k], stepOff[k + 1]), rows ascending
  std::vector<int> stepOff, rows;
  std::vector<double> f;
  void reset(int dim) {
    n = dim;
    piv.assign(static_cast<size_t>(dim), 0);
    stepOff.assign(static_cast<size_t>(dim) + 1, 0);
    rows.clear();
    f.clear();
  }
  void beginStep(int k, int p) {
    piv[k] = p;
    stepOff[k] = static_cast<int>(rows.size());
  }
  void log(int, int r, double fv) {
    rows.push_back(r);
    f.push_back(fv);
  }
  void logMany(const int* r, const double* fv, int m) {
    rows.insert(rows.end(), r, r + m);
    f.insert(f.end(), fv, fv + m);
  }
  void finish() { stepOff[n] = static_cast<int>(rows.size()); }
};
// solveDenseInPlace on a row-major A (n x n, leading dimension lda) that records `lu`
Vec solveDenseRecorded(double* A, int n, int lda, Vec& b, DenseLU& lu, double pivotTol = 1e-12);
// x of the recorded system for another right-hand side (bitwise a fresh solve)
Vec solveLU(const DenseLU& lu, Vec b);

// 0: blocked + host threads for n >= 128 (bitwise the unblocked elimination), 1: unblocked
// only (A/B and tests; env MORAP_DENSE=unblocked)
int& denseSolveMode();
// fn(0 .. n-1) on the host worker pool (the dense solve's threads); returns when all are done
void parallelFor(int n, const std::function<void(int)>& fn);
bool choleskyLower(const Mat& m, Mat& lower);

// ---- task logic (logic.hpp) --------------------------------------------------------------
enum class FKind : uint8_t { True, False, Atom, NotAtom, And, Or, Next, Until, Eventually };

struct Formula {
  FKind kind = FKind::True;
  std::string atom;
  std::vector<Formula> kids;
};
int cmpFormula(const Formula& a, const Formula& b);
bool operator==(const Formula& a, const Formula& b);
bool operator<(const Formula& a, const Formula& b);
Formula fTrue();
Formula fFalse();
Formula fAtom(std::string a);
Formula fNotAtom(std::string a);
Formula fAnd(std::vector<Formula> kids);
Formula fOr(std::vector<Formula> kids);
Formula fNext(Formula f);
Formula fUntil(Formula l, Formula r);
Formula fEventually(Formula f);
Formula negate(const Formula& f);
Formula parseCoSafe(const std::string& src);
Formula progressMask(const Formula& f, uint32_t letter, const std::vector<std::string>& atoms);

struct Dfa {
  std::vector<std::string> atoms;  // sorted; letters are bitmasks over them
  int numLocations = 0;
  int initial = 0;
  std::vector<char> accepting, trap, preSink;
  std::vector<int> delta;  // numLocations x numLetters
  int numLetters() const { return 1 << static_cast<int>(atoms.size()); }
  int step(int q, int letter) const { return delta[static_cast<size_t>(q) * numLetters() + letter]; }
};
uint32_t letterMaskFor(const Dfa& d, const std::vector<std::string>& sortedLabels);
Dfa formulaToDfa(const Formula& phi, size_t locationCap = 1000000);
Dfa insertPreSinks(const Dfa& d);
Dfa withDeadline(const Dfa& d, int k);
bool acceptsWord(const Dfa& d, const std::vector<uint32_t>& word);
Json dfaToJson(const Dfa& d);
Dfa dfaFromJson(const Json& j);

// ---- models (model.hpp) ------------------------------------------------------------------
struct Mdp {
  int numStates = 0;
  int initial = 0;
  std::vector<int> rowOffset, trnOffset, succ;
  std::vector<double> prob;
  std::vector<std::string> actionName;
  std::vector<std::vector<std::string>> labels;
  int numActions() const { return static_cast<int>(trnOffset.size()) - 1; }
  int actionsBegin(int s) const { return rowOffset[s]; }
  int actionsEnd(int s) const { return rowOffset[s + 1]; }
  int trnBegin(int r) const { return trnOffset[r]; }
  int trnEnd(int r) const { return trnOffset[r + 1]; }
};
using RewardStructure = Vec;

void validateMdp(const Mdp& m, double rowSumTol = 1e-9);
void renormalizeRows(Mdp& m);
std::pair<Mdp, RewardStructure> mdpFromJson(const Json& j);
Json mdpToJson(const Mdp& m, const RewardStructure& reward);

uint64_t nextProductUid();  // process-unique identity of a built product

struct ProductMdp {
  Mdp mdp;
  std::vector<int> agentState, dfaLocation;
  std::vector<char> done, accept, preSink;
  RewardStructure cost, success;
  std::vector<RewardStructure> extra;  // objectives beyond cost/success (K > 2 extension)
  bool rewardFinite = false;
  std::vector<std::string> droppedAtoms;
  int agentId = -1, taskId = -1;
  uint64_t structuralHash = 0;
  uint64_t uid = nextProductUid();  // device-model key (addresses can be reused after free)
  // Streamed instances (C4): once a product is resident on the device its host arrays are
  // dropped; numStates / initial / rewardFinite / hash stay, rows and nnz are kept here.
  bool slim = false;
  int slimRows = 0;
  int64_t slimNnz = 0;
};
inline int productRows(const ProductMdp& p) { return p.slim ? p.slimRows : p.mdp.numActions(); }
inline int64_t productNnz(const ProductMdp& p) { return p.slim ? p.slimNnz : static_cast<int64_t>(p.mdp.succ.size()); }
void slimProduct(ProductMdp& p);  // drop host arrays (the device copy is the only one left)
void requireFull(const ProductMdp& p, const char* what);  // InvalidConfig on a slim product
extern const std::string kInternalAction;

std::vector<int> maximalAvoidSet(const Mdp& m, const std::vector<char>& done);
bool checkRewardFinite(const Mdp& m, const std::vector<char>& done);
bool checkRewardFinite(const ProductMdp& p);
uint64_t productHash(const ProductMdp& p);
void checkPreSinks(const Dfa& task);  // buildProduct's InvalidDfa checks (model.hpp:234-243)
ProductMdp buildProduct(const Mdp& agent, const RewardStructure& agentCost, const Dfa& task, int agentId = -1,
                        int taskId = -1);

// ---- instance (instance.hpp) -------------------------------------------------------------
struct MorapInstance {
  std::vector<Mdp> agents;
  std::vector<RewardStructure> costs;
  std::vector<Dfa> tasks;
  int n = 0;
  int realTasks = 0;
  std::vector<std::vector<std::shared_ptr<const ProductMdp>>> products;  // [agent][task]
  int distinctProducts = 0;
  int objectives = 2;  // K: cost, success (+ extras)
};
// Called with each chunk's newly built distinct products (streamed builds): the sink
// uploads them and may slim them. Later chunks deduplicate against slim products by
// (structural hash, S, R, nnz, initial) instead of a full array compare.
using ProductSink = std::function<void(const std::vector<ProductMdp*>&)>;
MorapInstance buildInstance(std::vector<Mdp> agents, std::vector<RewardStructure> costs, std::vector<Dfa> tasks,
                            int threads = 0, size_t chunk = 0, const ProductSink* sink = nullptr);
Vec expandThresholds(const MorapInstance& inst, const Vec& user);
// K-objective extension: attach K-2 extra seeded per-row objectives in
// [-2, 0] to every product (not in the reference; parity for K > 2 is unpinned).
void addSyntheticObjectives(MorapInstance& inst, int K, uint64_t seed);

// ---- warehouse generator (warehouse.hpp) --------------------------------------------------
struct WarehouseConfig {
  int width = 0, height = 0, agents = 1;
  double slip = 0.05;
  std::vector<std::array<int, 2>> racks;
  std::array<int, 2> feed{0, 0};
  uint64_t seed = 0;
  int deadline = -1;
};
void validateWarehouseConfig(const WarehouseConfig& cfg);
std::pair<Mdp, RewardStructure> generateAgent(const WarehouseConfig& cfg, int agentIndex);
Formula generateTask(const WarehouseConfig& cfg, int rackIndex);
Dfa taskAutomaton(const WarehouseConfig& cfg, int rackIndex);
MorapInstance generateInstance(const WarehouseConfig& cfg, int threads = 0, size_t chunk = 0,
                               const ProductSink* sink = nullptr, const std::function<void()>* onRetry = nullptr);
// the seeded retry loop of generateInstance (warehouse.hpp) around any instance builder
using InstanceBuilder =
    std::function<MorapInstance(std::vector<Mdp>, std::vector<RewardStructure>, std::vector<Dfa>)>;
MorapInstance generateInstanceWith(const WarehouseConfig& cfg, const InstanceBuilder& build,
                                   const std::function<void()>* onRetry = nullptr);
WarehouseConfig warehouseConfigFromJson(const Json& j);

// ---- per-model solve on the GPU (numerics.hpp, engine.hpp) --------------------------------
// Allocator that default-initialises (no zero fill): scheduler rows are always written in
// full right after they are sized (a C2 query sizes 10 x ~0.3 MB of them per iteration).
template <class T>
struct DefaultInitAllocator : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInitAllocator<U>;
  };
  DefaultInitAllocator() = default;
  template <class U>
  DefaultInitAllocator(const DefaultInitAllocator<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept(std::is_nothrow_default_constructible<U>::value) {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};
using SchedulerRows = std::vector<int, DefaultInitAllocator<int>>;

struct Scheduler {  // deterministic: one action row per state (the solver only produces these)
  SchedulerRows rows;
};
Scheduler makeDeterministic(std::vector<int> rows);
struct SweepStats {
  int sweeps = 0;
  double residual = 0.0;
};
struct OptimizeResult {
  Vec values;
  Scheduler policy;
  SweepStats stats;
  double value = 0.0;
};
struct EvaluateResult {
  Vec values;
  SweepStats stats;
  double value = 0.0;
};
RewardStructure weightedReward(const std::vector<const RewardStructure*>& parts, const Vec& w);

// Device-resident model store + the CUDA context: the accelerator queue of the engine.
class GpuBackend {
 public:
  explicit GpuBackend(int device = 0);
  ~GpuBackend();
  GpuBackend(const GpuBackend&) = delete;
  GpuBackend& operator=(const GpuBackend&) = delete;
  // device model of p, uploaded on first use; full = with its fp64 arrays (explicit-reward jobs)
  int modelId(const ProductMdp* p, bool full = false);
  void uploadInstance(const MorapInstance& inst);  // all distinct products in one batch
  void uploadProducts(const std::vector<const ProductMdp*>& products, bool lean);  // skips resident ones
  // the same through a cached packed image: re-uploading the same products (after release())
  // is one host-to-device copy
  void uploadCached(const std::vector<const ProductMdp*>& products, bool lean);
  void setLean(bool on);  // default for query uploads (on): compact products without fp64 arrays
  bool lean() const { return leanDefault_; }
  int modelIdFor(uint64_t uid, const morap_csr_view& view);  // any model keyed by a process-unique id
  morap_ctx* ctx() const { return ctx_; }
  int device() const { return device_; }
  void release();
  void adopt(uint64_t uid, int id) { ids_[uid] = id; }  // a model built on the device for product uid

 private:
  morap_ctx* ctx_ = nullptr;
  int device_ = 0;
  std::map<uint64_t, int> ids_;      // ProductMdp::uid -> device model id (query uploads)
  std::map<uint64_t, int> fullIds_;  // full copies of lean products (explicit-reward jobs)
  bool leanDefault_ = true;
  morap_image* image_ = nullptr;   // cached packed image of the last uploaded instance
  std::vector<uint64_t> imageKey_;  // lean flag + product uids it holds
  bool isLean(int id);
};

// buildInstance (instance.hpp:42-91) with every product built on the GPU (morap_cuda_build_products):
// the products stay device-resident as lean compact models, the instance holds slim products
// (dimensions, reward finiteness, identity hash). Two objectives only (cost, success).
// In two steps for sharded builds: planDeviceBuild validates, measures every pair on `gpu`
// and rejects / deduplicates (the instance and its distinct products, nothing registered
// yet); DeviceBuild::write builds a subset of the distinct products on any device.
struct DeviceBuild {
  MorapInstance inst;
  std::vector<ProductMdp*> distinct;  // first-occurrence order
  struct Inputs;                      // agents / tasks / alphabets in the ABI layout
  std::unique_ptr<Inputs> in;
  void write(GpuBackend& gpu, const std::vector<size_t>& which) const;  // indices into `distinct`
  DeviceBuild();
  ~DeviceBuild();
};
std::unique_ptr<DeviceBuild> planDeviceBuild(GpuBackend& gpu, std::vector<Mdp> agents,
                                             std::vector<RewardStructure> costs, std::vector<Dfa> tasks);
MorapInstance buildInstanceOnDevice(GpuBackend& gpu, std::vector<Mdp> agents, std::vector<RewardStructure> costs,
                                    std::vector<Dfa> tasks);

OptimizeResult optimalScheduler(GpuBackend& gpu, const ProductMdp& p, const RewardStructure& rho, double eps = 1e-6,
                                int sweepCap = 100000);
EvaluateResult evaluateScheduler(GpuBackend& gpu, const ProductMdp& p, const Scheduler& mu, const RewardStructure& rho,
                                 double eps = 1e-6, int sweepCap = 100000);

enum class JobKind { Optimize, Evaluate };
struct Job {
  long id = 0;
  JobKind kind = JobKind::Optimize;
  std::shared_ptr<const ProductMdp> model;
  RewardStructure reward;
  Scheduler scheduler;
  double eps = 1e-6;
  int sweepCap = 100000;
};
struct JobResult {
  bool ok = false;
  std::string error;
  std::optional<Errc> errc;
  double value = 0.0;
  Vec values;
  Scheduler policy;
  SweepStats stats;
};
// engine.hpp:370 on the GPU: all jobs of one kind in one device batch.
std::map<long, JobResult> runBatch(std::vector<Job> jobs, GpuBackend& gpu);

// ---- assignment (assignment.hpp) ---------------------------------------------------------
struct Assignment {
  std::vector<int> agentOf;
  double value = 0.0;
};
Assignment maxAssignment(const Mat& c);
bool validateBistochastic(const Mat& x, double entryTol = 1e-9, double sumTol = 1e-6);

// ---- geometry (geometry.hpp) -------------------------------------------------------------
struct NormMatrix {
  Mat m;
  explicit NormMatrix(Mat mat);
  static NormMatrix identity(int dim);
  int dim() const { return m.rows; }
};
double normDistance(const NormMatrix& norm, const Vec& v);
struct LowerApprox {
  std::vector<Vec> points;
};
struct Halfspace {
  Vec w, r;
};
struct UpperApprox {
  std::vector<Halfspace> cuts;
};
struct ProjectionResult {
  Vec x, lambda;
  double distance = 0.0;
};
ProjectionResult projectToLowerApprox(const Vec& t, const LowerApprox& phi, const NormMatrix& norm);
Vec weightVector(const Vec& t, const Vec& tUp, const NormMatrix& norm);
Vec projectToUpperApprox(const Vec& t, const UpperApprox& upper, const NormMatrix& norm);

// ---- solver (solver.hpp) -----------------------------------------------------------------
struct SupportingPoint {
  Vec r;
  Assignment assignment;
  std::vector<Scheduler> schedulers;
};
struct IterationRecord {
  Vec w, r;
  Assignment assignment;
  std::vector<Scheduler> schedulers;
  Vec tUp, tDown;
};
struct ParetoResult {
  bool feasible = false, converged = false;
  Vec thresholds, tUp, tDown;
  LowerApprox phi;
  UpperApprox lambda;
  std::vector<IterationRecord> iterations;
  Vec lambdaStar;
  double eps = 0.0;
};
struct SynthesisTerm {
  double p = 0.0;
  Assignment assignment;
  std::vector<Scheduler> schedulers;
};
struct SynthesisResult {
  std::vector<SynthesisTerm> terms;
  Mat marginal;
};
struct QueryStats {  // per-query instrumentation (bench)
  long optimizeJobs = 0, evaluateJobs = 0;
  double optimizeBackups = 0, evaluateStateBackups = 0;
  double optimizeSeconds = 0, evaluateSeconds = 0, hostSeconds = 0;
  double evaluateSweepSeconds = 0;  // inside evaluateSeconds: the fused evaluate batch alone
};

using QueryFn = std::function<SupportingPoint(const Vec& w)>;

SupportingPoint supportingPoint(const MorapInstance& inst, const Vec& w, GpuBackend& gpu, QueryStats* stats = nullptr);
ParetoResult runParetoCore(Vec expandedThresholds, const NormMatrix& norm, double eps, int iterationCap,
                           bool verifyMode, bool* verdict, const QueryFn& query);
ParetoResult paretoPoint(const MorapInstance& inst, const Vec& thresholds, const NormMatrix& norm, double eps,
                         GpuBackend& gpu, int iterationCap = 500, QueryStats* stats = nullptr);
bool verifyOnly(const MorapInstance& inst, const Vec& thresholds, const NormMatrix& norm, double eps,
                GpuBackend& gpu, int iterationCap = 500);
SynthesisResult synthesize(const ParetoResult& result);

// ---- sharded supporting points (multi-GPU, csrc/shard.cpp) --------------------------------
// exchange(send, count, recv): recv[r * count + k] = shard r's send[k] for every shard r (an
// allgather: NCCL / gloo through a callback, or in-process)
using Exchange = std::function<void(const double* send, int count, double* recv)>;
// owner shard of every pair i * n + j: distinct products by longest-processing-time on nnz
std::vector<int> lptOwners(const MorapInstance& inst, int world);
class Shard {  // the pairs of one shard on one GPU
 public:
  Shard(const MorapInstance& inst, GpuBackend& gpu, std::vector<int> owner, int rank);
  void upload();  // this shard's products (lean when the objectives allow)
  // initial-state values of the pairs owned here and a mask per pair: 1 owned, 0 not,
  // 2 + status when the pair's job failed (so every rank raises the same error)
  void optimize(const Vec& w, double* values, double* mask, QueryStats* stats);
  // the K values of the assigned pairs owned here (r coordinates), mask per coordinate,
  // and their schedulers
  void evaluate(const Assignment& a, double* r, double* mask, std::vector<Scheduler>& schedulers, QueryStats* stats);
  const MorapInstance& instance() const { return inst_; }
  int rank() const { return rank_; }
  const std::vector<int>& owners() const { return owner_; }

 private:
  const MorapInstance& inst_;
  GpuBackend& gpu_;
  std::vector<int> owner_;
  int rank_;
  std::vector<int> jobIJ_;  // local optimize job of each owned pair (last optimize)
};
SupportingPoint shardedSupportingPoint(Shard& shard, int world, const Exchange& exchange, const Vec& w,
                                       QueryStats* stats = nullptr);
ParetoResult paretoPointSharded(Shard& shard, int world, const Exchange& exchange, const Vec& thresholds,
                                const NormMatrix& norm, double eps, int iterationCap = 500, QueryStats* stats = nullptr);
SupportingPoint multiSupportingPoint(const std::vector<Shard*>& shards, const Vec& w, QueryStats* stats = nullptr);
ParetoResult paretoPointMulti(const std::vector<Shard*>& shards, const Vec& thresholds, const NormMatrix& norm,
                              double eps, int iterationCap = 500, QueryStats* stats = nullptr);
Json resultToJson(const ParetoResult& result, const SynthesisResult* synthesis = nullptr);

// instance file (cli.hpp:84-117): agents inline or as paths, tasks as LTL strings / DFA JSON.
// `build` (optional): the instance builder to use instead of buildInstance (device builds)
MorapInstance instanceFromJson(const Json& j, const std::string& baseDir = ".", const InstanceBuilder* build = nullptr);

// ---- centralised model (centralised.hpp) -------------------------------------------------
// One MDP over (agent block i, task j, product state, assigned-agent mask) with the control
// rows b1 (assign the current task to agent i), b2 (pass it to the next free agent) and b3
// (advance to the next task once the current one ended). Its Pareto query runs the same
// device sweeps as the decentralised one, on a single large model.
struct CentralisedMdp {
  Mdp mdp;
  int n = 0, realTasks = 0;
  std::vector<char> taskEnded, done;
  std::vector<RewardStructure> rewards;  // n agent costs, then n task successes
  bool rewardFinite = false;
  std::vector<int> agentIdx, taskIdx, productState;
  std::vector<uint32_t> assigned;  // bitmask over agents
  uint64_t uid = nextProductUid();
};
CentralisedMdp buildCentralised(const MorapInstance& inst, long stateGuard = 10000000);
SupportingPoint centralisedSupportingPoint(const CentralisedMdp& c, const Vec& w, GpuBackend& gpu,
                                           double valueEps = 1e-6, QueryStats* stats = nullptr);
ParetoResult centralisedParetoPoint(const CentralisedMdp& c, const Vec& thresholds, const NormMatrix& norm,
                                    double eps, GpuBackend& gpu, int iterationCap = 500,
                                    QueryStats* stats = nullptr);

}  // namespace morap
