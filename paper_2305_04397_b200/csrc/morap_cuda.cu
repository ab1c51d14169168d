// libmorap_cuda.so -- sm_100a value-iteration backend behind include/morap_cuda.h.
//
// What runs on the GPU (reference functions replaced, /root/reference/proj/include/morap):
//   k_class_rho / k_weighted_reward   weightedReward             numerics.hpp:224-234
//   k_greedy_sweep_cmp (+ k_select)   optimalSchedulerOn sweep   numerics.hpp:84-113 (compact models)
//   k_greedy_sweep_tma                the same, fp64 streams     (non-compact models, explicit rewards)
//   k_greedy_sweep_*<true>            final argmax scheduler     numerics.hpp:96-102,114-115
//   k_chain_* + k_eval_interleaved / k_eval_persistent / k_eval_sweep_tma / k_eval_sweep
//                                     evaluateSchedulerOn sweep  numerics.hpp:138-162 (multi-RHS)
//   stop tests (delta <= eps, sweep cap -> NonConvergence, numerics.hpp:105-112) inside
//   k_select / the persistent kernels / k_finalize
//
// Files (one translation unit): device_types.cuh (HBM layout),
// kernels_optimize.cuh (K1, K3), kernels_evaluate.cuh + eval_interleaved.cuh (K2),
// upload_prep.cuh (host tiling / compact streams), this file (context, batch loops, upload
// pipeline, C ABI).
//
// Execution: jobs advance in lock step, one sweep per launch over the tiles of still-active
// jobs (frozen tiles skipped exactly), so converged jobs cost nothing and there is no
// per-sweep host synchronisation; sweeps go out as CUDA graphs and the host polls the
// active count between rounds. Evaluate batches run as one cooperative launch.
//
// Bitwise parity: every product and sum is an explicitly rounded __dmul_rn/__dadd_rn
// (no FMA contraction; also built with -fmad=false), rows are accumulated left to right
// from rho[r], the per-state argmax scans rows in order keeping the first strict max, and
// delta is a max (order independent). Hence values, sweeps, residuals and policies
// equal the reference CPU solver bit for bit.
#include <cuda_runtime.h>

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <thread>
#include <cstdint>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/morap_cuda.h"

namespace {
#include "device_types.cuh"
#include "kernels_optimize.cuh"
#include "kernels_evaluate.cuh"

// --------------------------------------------------------------------------------------
// host side

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) return ctx->cudaFail(e_, #call, __LINE__);                 \
  } while (0)

struct HostModel {
  int32_t S, R, nnz, initial, ntiles, K, rewardFinite;
  int32_t maxRowNnz;  // transitions of the widest row
  int32_t nOutGrp;    // entries of the model's out-of-window group lists (frozen-tile skipping)
  int32_t needB;      // its sweeps read the upload's segment B (non-compact / oversized tiles)
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
};

}  // namespace

struct morap_ctx {
  int device = 0;
  int numSMs = 148;
  int sweepBlocks = 0;  // grid of the tile-parallel helper kernels (weighted reward, policy chains)
  int evalBlocks = 0;   // persistent grid of the evaluate sweep kernel
  int tmaBlocks = 0;    // persistent grid of the TMA-pipelined sweep kernel
  int evalTmaBlocks = 0;
  static constexpr bool useTma = true;  // every sweep is a TMA-pipelined one on sm_100a
  bool evalTma = false;  // current evaluate batch runs the pipelined chain kernel
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;           // policy prefetch copies (overlap the evaluate sweeps)
  cudaEvent_t polReady = nullptr, polCopied = nullptr;
  cudaStream_t upload = nullptr;    // segment B copies of image uploads (not the policy side stream)
  cudaEvent_t segBReady = nullptr;  // segment B of the last image upload is on the device
  bool segBPending = false;         // ... and the stream has not waited for it yet
  std::vector<int32_t> polPrefetched;    // jobs whose policies sit in polStage (in this order)
  std::vector<size_t> polOff;
  std::string err;
  bool profiling = false;
  bool trace = std::getenv("MORAP_TRACE") != nullptr;
  double stats[12] = {0};  // [11]: device-to-host bytes copied
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  std::vector<HostModel> hm;
  std::vector<DevModel> dm;
  std::vector<void*> modelAllocs;
  std::vector<size_t> modelAllocBytes;
  // released model blocks kept for reuse: cudaFree of ~1 GB costs up to ~0.8 s on B200
  std::vector<std::pair<void*, size_t>> freeModelAllocs;
  DevModel* dModels = nullptr;
  size_t dModelsCap = 0;

  // optimize batch state
  int optJobs = 0;
  std::vector<int32_t> optModel;
  std::vector<int32_t> optSweeps;
  std::vector<int32_t> optStatus;
  std::vector<int32_t> optPolicyReady;
  void* optArena = nullptr;
  size_t optArenaBytes = 0;
  OptJob* dOptJobs = nullptr;
  std::vector<OptJob> hOptJobs;

  // evaluate batch state
  int evalJobs = 0;
  int evalSplitG = 1, evalSplitChunk = 0;  // evaluate_optimized split each job's RHS into G sub-jobs
  std::vector<EvalJob> hEvalJobs;
  std::vector<int32_t> evalSweeps;  // njobs * MAX_RHS
  void* evalArena = nullptr;
  size_t evalArenaBytes = 0;

  // control arrays (shared by optimize/evaluate loops, sized to max jobs)
  size_t ctlCap = 0;
  int32_t* dList = nullptr;
  int32_t* dPrefix = nullptr;
  int32_t* dJobModel = nullptr;
  unsigned long long* dDelta = nullptr;
  uint32_t* dMask = nullptr;
  int32_t* dNrhs = nullptr;
  int32_t* dSweeps = nullptr;
  double* dResidual = nullptr;
  double* dGather = nullptr;   // packed batch results (pack_result), 24 B per entry
  double* hGather = nullptr;   // pinned twin
  int32_t* dStatus = nullptr;
  int32_t* dAlive = nullptr;
  void* evalStage = nullptr;
  size_t evalStageBytes = 0;
  void* stage = nullptr;  // pinned host staging for uploads
  size_t stageBytes = 0;
  std::vector<cudaEvent_t> evPool;  // per-sweep start/stop events (profiling, no graphs)
  static constexpr int kKeyPtrs = 19;
  struct GraphKey {
    int kind, B, cap, variant, ncand;
    double eps;
    bool timed;
    const void* ptrs[kKeyPtrs];
    bool operator==(const GraphKey& o) const {
      if (kind != o.kind || B != o.B || cap != o.cap || variant != o.variant || ncand != o.ncand || eps != o.eps ||
          timed != o.timed)
        return false;
      for (int i = 0; i < kKeyPtrs; ++i)
        if (ptrs[i] != o.ptrs[i]) return false;
      return true;
    }
  };
  struct Graph {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    std::vector<cudaEvent_t> ev;
  };
  std::vector<Graph> graphs;  // cached sweep batches
  bool useGraphs = true;
  int lastOptSweeps = 0;      // sweeps the previous optimize batch needed (run_loop's first round)
  int launchedOptSweeps = 0;  // sweep launches of the previous optimize batch (>= its sweeps)
  bool useCompact = true;  // compact u8 probability / reward-class streams where possible
  bool lean = false;       // compact models uploaded without their fp64 prob / objective arrays
  bool optCompact = false; // current optimize batch runs the deep compact pipeline
  int cmpBlocks = 0;
  bool skip = true;        // frozen-tile skipping in compact optimize sweeps (k_select)
  // profiling: the events bracket the sweep kernel alone (k_select outside); MORAP_TIME_SELECT=1
  // brackets k_select + sweep
  bool timeSweepOnly = true;  // profiling events around the sweep kernel only (k_select outside)
  bool optSkip = false;    // current optimize batch uses it
  int selBlocks = 0;
  int2* dSel = nullptr;    // (job, tile) pairs of the current sweep
  int4* dCand = nullptr;   // candidates of the current optimize batch (k_build_cand)
  int32_t* dCandOut = nullptr;  // per candidate: offset of its absolute out-group stamps in dCandOutG
  int32_t* dCandOutG = nullptr;
  size_t candOutGCap = 0;
  int32_t* dStampAll = nullptr;  // stamps of the current optimize batch (inside optArena)
  int nCand = 0;
  void* dTrace = nullptr;  // diagnostics: per-CTA sweep timeline (morap_cuda_debug_cta_trace)
  size_t selCap = 0;
  bool usePersistent = true;  // evaluate batches as one cooperative launch
  int persistBlocks = 0;
  bool usePersistCache = false;
  bool useInterleaved = false;  // k_eval_interleaved for cached-chain evaluate batches
  int evalDirect = 0;  // current evaluate batch builds its chains in-kernel from the policies: 1 via
                       // the model CSR (segment B), 2 via the sweep streams (segment A only)
  bool evalModelRewards = false;  // current evaluate batch: rewards are the models' own objectives
  unsigned* dBar = nullptr;   // grid-barrier counter + generation
  unsigned* dFinCount = nullptr;  // CTAs done in the current compact sweep (fused finalize)
  void* persistArena = nullptr;
  size_t persistArenaBytes = 0;
  void* buildWs = nullptr;  // device product builder: per-CTA workspaces
  size_t buildWsBytes = 0;
  void* polStage = nullptr;  // pinned staging for batched policy reads
  size_t polStageBytes = 0;
  Ctl* dCtl = nullptr;
  Ctl* hCtl = nullptr;  // pinned mirror
  void* dEvalJobsRaw = nullptr;
  size_t dEvalJobsCap = 0;
  size_t dOptJobsCap = 0;

  int cudaFail(cudaError_t e, const char* what, int line) {
    err = std::string("CUDA error ") + cudaGetErrorString(e) + " at morap_cuda.cu:" + std::to_string(line) + " (" +
          what + ")";
    return MORAP_CUDA_ERROR;
  }
  int fail(int code, const std::string& msg) {
    err = msg;
    return code;
  }
};

namespace {

// Every device-to-host copy of the library goes through here and is counted (stats[11]),
// so the end-to-end bench reports the D2H bytes it actually moved.
cudaError_t d2h(morap_ctx* ctx, void* dst, const void* src, size_t bytes, bool sync = false) {
  ctx->stats[11] += static_cast<double>(bytes);
  return sync ? cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost)
              : cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream);
}

// Small host-to-device copies (job tables, lists, masks) from pageable memory: the driver
// takes the bytes immediately (the source may be freed on return) and does not wait for the
// device. (A pinned staging ring was slower: its copies queue behind an image upload's
// segment-B copy on the copy engine, while small pageable copies travel inline.)
int h2d(morap_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return MORAP_OK;
}
#define H2D(dst, src, bytes)                                   \
  do {                                                         \
    const int rcH_ = h2d(ctx, (dst), (src), (bytes));          \
    if (rcH_) return rcH_;                                     \
  } while (0)

// The stream waits for the last image upload's segment B before a kernel that reads it.
int wait_segment_b(morap_ctx* ctx) {
  if (!ctx->segBPending) return MORAP_OK;
  CK(cudaStreamWaitEvent(ctx->stream, ctx->segBReady, 0));
  ctx->segBPending = false;
  return MORAP_OK;
}

int ensure_ctl(morap_ctx* ctx, size_t njobs) {
  if (njobs <= ctx->ctlCap && ctx->dCtl) return MORAP_OK;
  size_t cap = std::max<size_t>(njobs, 64);
  cudaFree(ctx->dList);
  cudaFree(ctx->dPrefix);
  cudaFree(ctx->dJobModel);
  cudaFree(ctx->dDelta);
  cudaFree(ctx->dMask);
  cudaFree(ctx->dNrhs);
  cudaFree(ctx->dSweeps);
  cudaFree(ctx->dResidual);
  cudaFree(ctx->dStatus);
  cudaFree(ctx->dGather);
  cudaFree(ctx->dAlive);
  CK(cudaMalloc(&ctx->dGather, cap * MORAP_MAX_RHS * 3 * sizeof(double)));
  if (ctx->hGather) cudaFreeHost(ctx->hGather);
  CK(cudaMallocHost(&ctx->hGather, cap * MORAP_MAX_RHS * 3 * sizeof(double)));
  CK(cudaMalloc(&ctx->dAlive, cap * sizeof(int32_t)));
  CK(cudaMalloc(&ctx->dList, cap * sizeof(int32_t)));
  CK(cudaMalloc(&ctx->dPrefix, (cap + 1) * sizeof(int32_t)));
  CK(cudaMalloc(&ctx->dJobModel, cap * sizeof(int32_t)));
  CK(cudaMalloc(&ctx->dDelta, cap * MORAP_MAX_RHS * sizeof(unsigned long long)));
  CK(cudaMalloc(&ctx->dMask, cap * sizeof(uint32_t)));
  CK(cudaMalloc(&ctx->dNrhs, cap * sizeof(int32_t)));
  CK(cudaMalloc(&ctx->dSweeps, cap * MORAP_MAX_RHS * sizeof(int32_t)));
  CK(cudaMalloc(&ctx->dResidual, cap * MORAP_MAX_RHS * sizeof(double)));
  CK(cudaMalloc(&ctx->dStatus, cap * MORAP_MAX_RHS * sizeof(int32_t)));
  if (!ctx->dCtl) {
    CK(cudaMalloc(&ctx->dCtl, sizeof(Ctl)));
    CK(cudaMallocHost(&ctx->hCtl, sizeof(Ctl)));
  }
  ctx->ctlCap = cap;
  return MORAP_OK;
}

#include "upload_prep.cuh"
#include "kernels_build.cuh"

int upload_models_table(morap_ctx* ctx) {
  if (ctx->dm.size() > ctx->dModelsCap) {
    cudaFree(ctx->dModels);
    size_t cap = std::max<size_t>(ctx->dm.size() * 2, 16);
    CK(cudaMalloc(&ctx->dModels, cap * sizeof(DevModel)));
    ctx->dModelsCap = cap;
  }
  H2D(ctx->dModels, ctx->dm.data(), ctx->dm.size() * sizeof(DevModel));
  return MORAP_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int ensure_arena(morap_ctx* ctx, void** arena, size_t* have, size_t need) {
  if (need <= *have) return MORAP_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(*arena);
  *arena = nullptr;
  size_t cap = std::max(need, *have + *have / 2);
  cudaError_t e = cudaMalloc(arena, cap);
  if (e != cudaSuccess) {
    cap = need;
    CK(cudaMalloc(arena, cap));
  }
  *have = cap;
  return MORAP_OK;
}


// Enqueues B (sweep, finalize) pairs on the context stream; with `ev` (2B events) every
// sweep launch is bracketed by CUDA events.
int enqueue_sweeps(morap_ctx* ctx, int kind, double eps, int cap, int B, const cudaEvent_t* ev, bool capturing) {
  const unsigned evFlags = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
  for (int i = 0; i < B; ++i) {
    const bool selTimed = !(kind == 0 && ctx->useTma && ctx->optCompact && ctx->optSkip && ctx->timeSweepOnly);
    if (ev && selTimed) CK(cudaEventRecordWithFlags(ev[2 * i], ctx->stream, evFlags));
    if (kind == 0 && ctx->useTma && ctx->optCompact) {
      const FinArgs fin{ctx->dFinCount, ctx->dJobModel, eps, cap, ctx->dSweeps, ctx->dResidual, ctx->dStatus};
      if (ctx->optSkip) {
        k_select<<<ctx->selBlocks, kSelThreads, 0, ctx->stream>>>(
            ctx->dModels, ctx->dOptJobs, ctx->dAlive, ctx->dCand, ctx->dCandOut, ctx->dCandOutG, ctx->dStampAll,
            ctx->nCand, ctx->dCtl, ctx->dSel, ctx->dDelta, eps, cap, ctx->dSweeps, ctx->dResidual, ctx->dStatus);
        CK(cudaGetLastError());
      }
      if (ev && !selTimed) CK(cudaEventRecordWithFlags(ev[2 * i], ctx->stream, evFlags));
      k_greedy_sweep_cmp<false><<<ctx->cmpBlocks, kTmaThreads, kCmpSmemBytes, ctx->stream>>>(
          ctx->dModels, ctx->dOptJobs, ctx->dList, ctx->dPrefix, ctx->dCtl, nullptr, ctx->dDelta,
          ctx->optSkip ? ctx->dSel : nullptr, fin);
    } else if (kind == 0) {
      k_greedy_sweep_tma<false><<<ctx->tmaBlocks, kTmaThreads, kTmaSmemBytes, ctx->stream>>>(
          ctx->dModels, ctx->dOptJobs, ctx->dList, ctx->dPrefix, ctx->dCtl, nullptr, ctx->dDelta);
    } else if (ctx->evalTma) {
      k_eval_sweep_tma<<<ctx->evalTmaBlocks, kTmaThreads, kEvSmemBytes, ctx->stream>>>(
          ctx->dModels, (const EvalJob*)ctx->dEvalJobsRaw, ctx->dList, ctx->dPrefix, ctx->dCtl, ctx->dMask, ctx->dDelta);
    } else {
      k_eval_sweep<<<ctx->evalBlocks, kBlock, 0, ctx->stream>>>(ctx->dModels, (const EvalJob*)ctx->dEvalJobsRaw,
                                                                ctx->dList, ctx->dPrefix, ctx->dCtl, ctx->dMask,
                                                                ctx->dDelta);
    }
    CK(cudaGetLastError());
    if (ev) CK(cudaEventRecordWithFlags(ev[2 * i + 1], ctx->stream, evFlags));
    if (kind == 0 && ctx->useTma && ctx->optCompact)
      ;  // finalize fused into the compact sweep's last CTA
    else if (kind == 0)
      k_finalize<false><<<1, kFinBlock, 0, ctx->stream>>>(ctx->dModels, ctx->dJobModel, ctx->dList, ctx->dPrefix,
                                                         ctx->dCtl, ctx->dDelta, ctx->dMask, ctx->dNrhs, eps, cap,
                                                         ctx->dSweeps, ctx->dResidual, ctx->dStatus);
    else
      k_finalize<true><<<1, kFinBlock, 0, ctx->stream>>>(ctx->dModels, ctx->dJobModel, ctx->dList, ctx->dPrefix,
                                                        ctx->dCtl, ctx->dDelta, ctx->dMask, ctx->dNrhs, eps, cap,
                                                        ctx->dSweeps, ctx->dResidual, ctx->dStatus);
    CK(cudaGetLastError());
  }
  return MORAP_OK;
}

// A batch of B sweep/finalize pairs as one CUDA graph (kernel arguments are the same for
// every batch of a call: all per-sweep state lives in device memory). Cached per
// (kind, B, eps, cap, profiling, kernel variant, buffer addresses).
int batch_graph(morap_ctx* ctx, int kind, double eps, int cap, int B, bool timed, morap_ctx::Graph** out) {
  morap_ctx::GraphKey key{};
  key.kind = kind;
  key.B = B;
  key.eps = eps;
  key.cap = cap;
  key.timed = timed;
  key.variant = (ctx->useTma ? 1 : 0) | (ctx->evalTma ? 2 : 0) | (ctx->optCompact ? 4 : 0) | (ctx->optSkip ? 8 : 0);
  key.ncand = kind == 0 && ctx->optSkip ? ctx->nCand : 0;
  const void* ptrs[] = {ctx->dModels, ctx->dOptJobs, ctx->dList,  ctx->dPrefix,    ctx->dCtl,      ctx->dDelta,
                        ctx->dMask,   ctx->dNrhs,    ctx->dSweeps, ctx->dResidual, ctx->dStatus,   ctx->dJobModel,
                        ctx->dEvalJobsRaw, ctx->stream, ctx->dSel, ctx->dCand, ctx->dCandOut, ctx->dCandOutG,
                        ctx->dStampAll};
  static_assert(sizeof(ptrs) / sizeof(ptrs[0]) == morap_ctx::kKeyPtrs, "graph key size");
  for (int i = 0; i < morap_ctx::kKeyPtrs; ++i) key.ptrs[i] = ptrs[i];
  for (auto& g : ctx->graphs)
    if (g.key == key) {
      *out = &g;
      return MORAP_OK;
    }
  if (ctx->graphs.size() >= 24) {
    for (auto& g : ctx->graphs) {
      cudaGraphExecDestroy(g.exec);
      for (cudaEvent_t e : g.ev) cudaEventDestroy(e);
    }
    ctx->graphs.clear();
  }
  morap_ctx::Graph g;
  g.key = key;
  if (timed) {
    g.ev.resize(2 * B);
    for (auto& e : g.ev) CK(cudaEventCreate(&e));
  }
  cudaGraph_t graph = nullptr;
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  const int rc = enqueue_sweeps(ctx, kind, eps, cap, B, timed ? g.ev.data() : nullptr, true);
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  if (rc) return rc;
  if (e != cudaSuccess) return ctx->cudaFail(e, "graph capture", __LINE__);
  e = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return ctx->cudaFail(e, "graph instantiate", __LINE__);
  ctx->graphs.push_back(std::move(g));
  *out = &ctx->graphs.back();
  return MORAP_OK;
}

// Runs sweeps (+finalize) until no job is active. kind 0 optimize, 1 evaluate.
// Sweep/finalize pairs go out as CUDA graphs of 4, 8, 16 or 32 pairs and the 4-byte active
// count is polled between rounds of graphs (converged jobs are already frozen on the device,
// so overshooting only costs empty launches). The optimize batches of one Pareto query need
// similar sweep counts from call to call, so the first round launches (previous call's count
// - 2) pairs at once and later rounds 4, 8, 16, 32; without a history, 4, 8, 16, 32. With
// profiling on, every sweep launch inside the graphs is bracketed by CUDA events; only
// launches that still had active jobs are counted.
int run_loop(morap_ctx* ctx, int kind, double eps, int cap) {
  const bool timed = ctx->profiling;
  const int start = ctx->hCtl->sweepsDone;
  int before = start;
  double ms = 0.0;
  int launched = 0;
  int ahead = kind == 0 && ctx->lastOptSweeps > 6 ? ((ctx->lastOptSweeps - 2 + 3) & ~3) : 4;
  int next = 4;
  for (;;) {
    // this round: `ahead` pairs as graphs of 32 / 16 / 8 / 4
    std::vector<int> pieces;
    for (int left = ahead; left > 0;) {
      const int b = left >= 32 ? 32 : left >= 16 ? 16 : left >= 8 ? 8 : 4;
      pieces.push_back(b);
      left -= b;
    }
    std::vector<const cudaEvent_t*> evs;
    if (timed && !ctx->useGraphs)  // pointers into the pool stay valid for the whole round
      while (ctx->evPool.size() < 2u * 32u * pieces.size()) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        ctx->evPool.push_back(e);
      }
    for (int b : pieces) {
      morap_ctx::Graph* g = nullptr;
      int rc = ctx->useGraphs ? batch_graph(ctx, kind, eps, cap, b, timed, &g) : MORAP_OK;
      if (rc) return rc;
      if (g) {
        CK(cudaGraphLaunch(g->exec, ctx->stream));
        evs.push_back(g->ev.data());
      } else {
        const cudaEvent_t* ev = timed ? ctx->evPool.data() + 2 * evs.size() * 32 : nullptr;
        if ((rc = enqueue_sweeps(ctx, kind, eps, cap, b, ev, false))) return rc;
        evs.push_back(ev);
      }
      launched += b;
      ctx->stats[8] += (kind == 0 && ctx->useTma && ctx->optCompact ? (ctx->optSkip ? 2 : 1) : 2) * b;
    }
    CK(d2h(ctx, ctx->hCtl, ctx->dCtl, sizeof(Ctl)));
    CK(cudaStreamSynchronize(ctx->stream));
    if (timed) {
      int worked = ctx->hCtl->sweepsDone - before;
      for (size_t q = 0; q < pieces.size() && worked > 0; ++q)
        for (int i = 0; i < pieces[q] && worked > 0; ++i, --worked) {
          float t = 0.f;
          CK(cudaEventElapsedTime(&t, evs[q][2 * i], evs[q][2 * i + 1]));
          ms += t;
        }
    }
    before = ctx->hCtl->sweepsDone;
    if (ctx->hCtl->nactive == 0) break;
    ahead = next;
    next = std::min(next * 2, 32);
  }
  if (kind == 0) {
    ctx->lastOptSweeps = ctx->hCtl->sweepsDone - start;
    ctx->launchedOptSweeps = launched;
  }
  if (timed) ctx->stats[kind == 0 ? 1 : 5] += ms;
  return MORAP_OK;
}

// Host-built initial active list: jobs listed in `active` (order kept), tile prefix.
int init_ctl(morap_ctx* ctx, const std::vector<int32_t>& active, const std::vector<int32_t>& jobModel) {
  std::vector<int32_t> prefix(active.size() + 1, 0);
  for (size_t a = 0; a < active.size(); ++a) prefix[a + 1] = prefix[a] + ctx->hm[jobModel[active[a]]].ntiles;
  if (!active.empty()) H2D(ctx->dList, active.data(), active.size() * 4);
  H2D(ctx->dPrefix, prefix.data(), prefix.size() * 4);
  H2D(ctx->dJobModel, jobModel.data(), jobModel.size() * 4);
  Ctl c{};
  c.nactive = static_cast<int32_t>(active.size());
  c.totalTiles = prefix.back();
  c.sweepsDone = 0;
  *ctx->hCtl = c;
  CK(cudaMemcpyAsync(ctx->dCtl, ctx->hCtl, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
  return MORAP_OK;
}

// Shared body of the two optimize entry points. rhoHost == nullptr -> weights mode.
int optimize_impl(morap_ctx* ctx, int njobs, const int32_t* model_ids, const double* weights, int K,
                  const double* const* rhoHost, double eps, int cap, double* value_out, int32_t* sweeps_out,
                  double* residual_out, int32_t* status_out) {
  if (njobs < 0) return ctx->fail(MORAP_INVALID_CONFIG, "negative job count");
  if (!(eps >= 0.0)) return ctx->fail(MORAP_INVALID_CONFIG, "eps must be nonnegative");
  if (cap < 1) return ctx->fail(MORAP_INVALID_CONFIG, "sweep cap must be positive");
  if (!rhoHost && (K < 0 || K > MORAP_MAX_OBJECTIVES)) return ctx->fail(MORAP_DIMENSION_MISMATCH, "bad objective count");
  CK(cudaEventSynchronize(ctx->polCopied));  // policy buffers are about to be rewritten
  ctx->polPrefetched.clear();
  ctx->optJobs = 0;
  if (njobs == 0) return MORAP_OK;
  {
    bool needB = rhoHost != nullptr;  // explicit rewards: the fp64 arrays
    for (int j = 0; j < njobs && !needB; ++j)
      needB = model_ids[j] >= 0 && model_ids[j] < static_cast<int>(ctx->hm.size()) && ctx->hm[model_ids[j]].needB;
    int rcB;
    if (needB && (rcB = wait_segment_b(ctx))) return rcB;
  }
  for (int j = 0; j < njobs; ++j) {
    if (model_ids[j] < 0 || model_ids[j] >= static_cast<int>(ctx->hm.size()))
      return ctx->fail(MORAP_INVALID_CONFIG, "job " + std::to_string(j) + ": unknown model id");
    if (!rhoHost && K != ctx->hm[model_ids[j]].K)
      return ctx->fail(MORAP_DIMENSION_MISMATCH, "one weight per reward structure (numerics.hpp:225)");
    if (rhoHost && !ctx->dm[model_ids[j]].prob)
      return ctx->fail(MORAP_INVALID_CONFIG, "lean models take weighted jobs only (no explicit reward vectors)");
  }
  // arena regions: [rho of every job][x0|x1 of every job][policy of every job] so the
  // x region is zeroed with one memset (x = y = 0 at the start, numerics.hpp:81)
  size_t rhoBytes = 0, xBytes = 0, polBytes = 0;
  std::vector<size_t> offRho(njobs), offX(njobs), offPol(njobs);
  std::vector<int32_t> stampOff(njobs);
  size_t stampInts = 0;  // stamps of every job, contiguous (k_select indexes them absolutely)
  // compact sweeps read rho_w per reward class only: no per-row rho vector then
  bool allCompact = ctx->useCompact && ctx->useTma && !rhoHost;
  for (int j = 0; j < njobs && allCompact; ++j)
    if (!ctx->dm[model_ids[j]].compact) allCompact = false;
  for (int j = 0; j < njobs; ++j) {
    const HostModel& m = ctx->hm[model_ids[j]];
    offRho[j] = rhoBytes;
    const bool lean = !ctx->dm[model_ids[j]].prob;  // lean compact model: class table only
    if (!lean && !allCompact) rhoBytes += align_up(sizeof(double) * m.R, 256);
    offX[j] = xBytes;
    xBytes += 2 * align_up(sizeof(double) * m.S, 256);  // x0 | x1
    stampOff[j] = static_cast<int32_t>(stampInts);
    stampInts += static_cast<size_t>(((m.S + 31) / 32 + 7) & ~3);
    offPol[j] = polBytes;
    polBytes += align_up(sizeof(int32_t) * m.S, 256);
  }
  if (stampInts >= (1u << 31)) return ctx->fail(MORAP_SIZE_GUARD, "stamp array exceeds 2^31 entries");
  const size_t xJobBytes = xBytes;
  xBytes += align_up(sizeof(int32_t) * stampInts, 256);  // zeroed with x
  std::vector<size_t> offClass(njobs);  // rho_w per reward class, per job
  size_t classBytes = 0;
  for (int j = 0; j < njobs; ++j) {
    offClass[j] = classBytes;
    classBytes += align_up(sizeof(double) * std::max(1, ctx->dm[model_ids[j]].nclass), 256);
  }
  const size_t need = rhoBytes + xBytes + polBytes + classBytes;
  int rc;
  if ((rc = ensure_arena(ctx, &ctx->optArena, &ctx->optArenaBytes, need))) return rc;
  if ((rc = ensure_ctl(ctx, njobs))) return rc;
  if (static_cast<size_t>(njobs) > ctx->dOptJobsCap) {
    cudaFree(ctx->dOptJobs);
    ctx->dOptJobsCap = std::max<size_t>(njobs, 64);
    CK(cudaMalloc(&ctx->dOptJobs, ctx->dOptJobsCap * sizeof(OptJob)));
  }
  ctx->hOptJobs.assign(njobs, OptJob{});
  ctx->optModel.assign(model_ids, model_ids + njobs);
  std::vector<int32_t> active, statusInit(njobs, MORAP_OK), zeroI(njobs, 0);
  char* base = static_cast<char*>(ctx->optArena);
  for (int j = 0; j < njobs; ++j) {
    const HostModel& m = ctx->hm[model_ids[j]];
    OptJob& J = ctx->hOptJobs[j];
    J.model = model_ids[j];
    J.rho = (ctx->dm[model_ids[j]].prob && !allCompact) ? reinterpret_cast<double*>(base + offRho[j]) : nullptr;
    J.buf[0] = reinterpret_cast<double*>(base + rhoBytes + offX[j]);
    J.buf[1] = reinterpret_cast<double*>(base + rhoBytes + offX[j] + align_up(sizeof(double) * m.S, 256));
    J.policy = reinterpret_cast<int32_t*>(base + rhoBytes + xBytes + offPol[j]);
    J.stampOff = stampOff[j];
    J.stamp = reinterpret_cast<int32_t*>(base + rhoBytes + xJobBytes) + stampOff[j];
    J.outGrp = ctx->dm[model_ids[j]].outGrp;
    J.bytesPerSweep = ctx->dm[model_ids[j]].bytesPerSweep;
    J.nnz = m.nnz;
    J.classRho = (!rhoHost && ctx->dm[model_ids[j]].compact)
                     ? reinterpret_cast<double*>(base + rhoBytes + xBytes + polBytes + offClass[j])
                     : nullptr;
    if (!rhoHost)
      for (int o = 0; o < K; ++o) J.w[o] = weights[static_cast<size_t>(j) * K + o];
    if (!m.rewardFinite) statusInit[j] = MORAP_NOT_REWARD_FINITE;  // numerics.hpp:79-80
    else active.push_back(j);
  }
  CK(cudaMemsetAsync(base + rhoBytes, 0, xBytes, ctx->stream));
  ctx->optCompact = allCompact;
  ctx->optSkip = allCompact && ctx->skip;
  for (int j = 0; j < njobs && ctx->optSkip; ++j)
    if (ctx->hm[model_ids[j]].ntiles >= (1 << kCandLtBits)) ctx->optSkip = false;  // k_build_cand packing
  ctx->dStampAll = reinterpret_cast<int32_t*>(base + rhoBytes + xJobBytes);
  if (ctx->optSkip) {
    size_t tiles = 0, outs = 0;
    for (int j : active) {
      tiles += static_cast<size_t>(ctx->hm[model_ids[j]].ntiles);
      ctx->hOptJobs[j].outBase = static_cast<int32_t>(outs);
      outs += static_cast<size_t>(ctx->hm[model_ids[j]].nOutGrp);
    }
    if (outs >= (1u << 31)) ctx->optSkip = false;
    if (outs > ctx->candOutGCap) {
      CK(cudaStreamSynchronize(ctx->stream));
      cudaFree(ctx->dCandOutG);
      ctx->dCandOutG = nullptr;
      ctx->candOutGCap = std::max(outs, ctx->candOutGCap + ctx->candOutGCap / 2);
      CK(cudaMalloc(&ctx->dCandOutG, ctx->candOutGCap * sizeof(int32_t)));
    }
    if (tiles > ctx->selCap) {
      CK(cudaStreamSynchronize(ctx->stream));
      cudaFree(ctx->dSel);
      cudaFree(ctx->dCand);
      cudaFree(ctx->dCandOut);
      ctx->dSel = nullptr;
      ctx->dCand = nullptr;
      ctx->dCandOut = nullptr;
      ctx->selCap = std::max(tiles, ctx->selCap + ctx->selCap / 2);
      CK(cudaMalloc(&ctx->dSel, ctx->selCap * sizeof(int2)));
      CK(cudaMalloc(&ctx->dCand, ctx->selCap * sizeof(int4)));
      CK(cudaMalloc(&ctx->dCandOut, ctx->selCap * sizeof(int32_t)));
    }
    ctx->nCand = static_cast<int>(tiles);
  }
  if (!ctx->optSkip)
    for (int j = 0; j < njobs; ++j) ctx->hOptJobs[j].stamp = nullptr;
  if (!ctx->optCompact)
    for (int j = 0; j < njobs; ++j)
      if (!ctx->dm[model_ids[j]].prob)
        return ctx->fail(MORAP_INVALID_CONFIG, "a batch with lean models cannot include non-compact models");
  H2D(ctx->dOptJobs, ctx->hOptJobs.data(), njobs * sizeof(OptJob));
  H2D(ctx->dStatus, statusInit.data(), njobs * 4);
  CK(cudaMemsetAsync(ctx->dSweeps, 0, njobs * 4, ctx->stream));
  CK(cudaMemsetAsync(ctx->dDelta, 0, 2 * njobs * sizeof(unsigned long long), ctx->stream));  // two parities
  CK(cudaMemsetAsync(ctx->dResidual, 0, njobs * sizeof(double), ctx->stream));
  if ((rc = init_ctl(ctx, active, ctx->optModel))) return rc;
  if (ctx->optSkip && !active.empty()) {
    std::vector<int32_t> alive(njobs, 0);  // act: 1 while the job iterates
    for (int j : active) alive[j] = 1;
    H2D(ctx->dAlive, alive.data(), njobs * 4);
    int maxTiles = 0;
    for (int j : active) maxTiles = std::max(maxTiles, ctx->hm[model_ids[j]].ntiles);
    for (size_t s0 = 0; s0 < active.size(); s0 += 65535) {  // gridDim.y limit
      const dim3 grid((maxTiles + kSelThreads - 1) / kSelThreads, static_cast<unsigned>(std::min<size_t>(65535, active.size() - s0)));
      k_build_cand<<<grid, kSelThreads, 0, ctx->stream>>>(ctx->dModels, ctx->dOptJobs, ctx->dList, ctx->dPrefix,
                                                          ctx->dCand, ctx->dCandOut, ctx->dCandOutG,
                                                          static_cast<int>(s0));
      CK(cudaGetLastError());
      ctx->stats[8] += 1;
    }
  }

  // rho: device-side weighted reward, or host-provided vectors
  if (rhoHost) {
    for (int j = 0; j < njobs; ++j) {
      const HostModel& m = ctx->hm[model_ids[j]];
      if (m.R) CK(cudaMemcpyAsync(ctx->hOptJobs[j].rho, rhoHost[j], sizeof(double) * m.R, cudaMemcpyHostToDevice, ctx->stream));
    }
  } else if (!active.empty() && allCompact) {  // rho_w per reward class only: one CTA per job
    k_class_rho<<<static_cast<int>(active.size()), kBlock, 0, ctx->stream>>>(ctx->dModels, ctx->dOptJobs, ctx->dList);
    CK(cudaGetLastError());
    ctx->stats[8] += 1;
  } else if (!active.empty()) {
    k_weighted_reward<<<ctx->sweepBlocks, kBlock, 0, ctx->stream>>>(ctx->dModels, ctx->dOptJobs, ctx->dList,
                                                                    ctx->dPrefix, ctx->hCtl->nactive,
                                                                    ctx->hCtl->totalTiles);
    CK(cudaGetLastError());
    ctx->stats[8] += 1;
  }
  if (!active.empty()) {
    if ((rc = run_loop(ctx, 0, eps, cap))) return rc;
    if (ctx->trace)
      std::fprintf(stderr, "[morap] optimize batch: %d jobs, %d sweeps, %d sweep launches\n", njobs,
                   ctx->lastOptSweeps, ctx->launchedOptSweeps);
  }

  // results: one gather kernel packs them, one copy into pinned memory, one synchronisation
  ctx->optSweeps.assign(njobs, 0);
  ctx->optStatus.assign(njobs, 0);
  k_gather_opt<<<(njobs + 255) / 256, 256, 0, ctx->stream>>>(ctx->dModels, ctx->dOptJobs, njobs, ctx->dSweeps,
                                                             ctx->dStatus, ctx->dResidual, ctx->dGather);
  CK(cudaGetLastError());
  CK(d2h(ctx, ctx->hGather, ctx->dGather, 24ull * njobs));
  CK(d2h(ctx, ctx->hCtl, ctx->dCtl, sizeof(Ctl)));
  CK(cudaStreamSynchronize(ctx->stream));
  const int32_t* gi = reinterpret_cast<const int32_t*>(ctx->hGather + 2ull * njobs);
  double backups = 0;
  for (int j = 0; j < njobs; ++j) {
    ctx->optSweeps[j] = gi[j];
    ctx->optStatus[j] = gi[njobs + j];
    value_out[j] = ctx->hGather[j];
    if (sweeps_out) sweeps_out[j] = ctx->optSweeps[j];
    if (residual_out) residual_out[j] = ctx->hGather[njobs + j];
    if (status_out) status_out[j] = ctx->optStatus[j];
    backups += static_cast<double>(ctx->optSweeps[j]) * ctx->hm[model_ids[j]].nnz;
  }
  // bytes: what the sweeps actually streamed; backups: sweeps x nnz of every job (the
  // reference's work for the same results); [10]: backups actually executed
  ctx->stats[0] += ctx->hCtl->sweepsDone;
  ctx->stats[2] += static_cast<double>(ctx->optSkip ? ctx->hCtl->execBytes : ctx->hCtl->bytes);
  ctx->stats[3] += backups;
  ctx->stats[10] += ctx->optSkip ? static_cast<double>(ctx->hCtl->execBackups) : backups;
  ctx->optPolicyReady.assign(njobs, 0);
  ctx->optJobs = njobs;
  return MORAP_OK;
}

// Computes final-sweep argmax policies for the listed optimize jobs (on the device).
int extract_policies(morap_ctx* ctx, const std::vector<int32_t>& jobsIn) {
  for (int j : jobsIn)  // compact all-fit models: the policy sweep reads segment A only
    if (!ctx->optCompact || ctx->hm[ctx->optModel[j]].needB) {
      int rcB;
      if ((rcB = wait_segment_b(ctx))) return rcB;
      break;
    }
  std::vector<int32_t> jobs;
  for (int j : jobsIn)
    if (!ctx->optPolicyReady[j] && ctx->optSweeps[j] > 0) jobs.push_back(j);
  if (jobs.empty()) return MORAP_OK;
  int rc;
  if ((rc = init_ctl(ctx, jobs, ctx->optModel))) return rc;
  H2D(ctx->dSweeps, ctx->optSweeps.data(), ctx->optSweeps.size() * 4);
  if (ctx->optCompact)
    k_greedy_sweep_cmp<true><<<ctx->cmpBlocks, kTmaThreads, kCmpSmemBytes, ctx->stream>>>(
        ctx->dModels, ctx->dOptJobs, ctx->dList, ctx->dPrefix, ctx->dCtl, ctx->dSweeps, nullptr, nullptr, FinArgs{});
  else
    k_greedy_sweep_tma<true><<<ctx->tmaBlocks, kTmaThreads, kTmaSmemBytes, ctx->stream>>>(
        ctx->dModels, ctx->dOptJobs, ctx->dList, ctx->dPrefix, ctx->dCtl, ctx->dSweeps, nullptr);
  CK(cudaGetLastError());
  ctx->stats[8] += 1;
  for (int j : jobs) ctx->optPolicyReady[j] = 1;
  return MORAP_OK;
}

// Copy the final policies of `jobs` to the pinned staging area on the side stream (after
// the policy kernel on the main stream); morap_cuda_fetch_policies then only waits for them.
int prefetch_policies(morap_ctx* ctx, const std::vector<int32_t>& jobs) {
  size_t bytes = 0;
  for (int j : jobs) bytes += align_up(sizeof(int32_t) * ctx->hm[ctx->optModel[j]].S, 256);
  if (bytes > ctx->polStageBytes) {
    CK(cudaStreamSynchronize(ctx->side));
    cudaFreeHost(ctx->polStage);
    ctx->polStage = nullptr;
    ctx->polStageBytes = 0;
    CK(cudaMallocHost(&ctx->polStage, bytes));
    ctx->polStageBytes = bytes;
  }
  CK(cudaEventRecord(ctx->polReady, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->side, ctx->polReady, 0));
  ctx->polOff.assign(jobs.size(), 0);
  size_t o = 0;
  for (size_t q = 0; q < jobs.size(); ++q) {
    const size_t n = sizeof(int32_t) * ctx->hm[ctx->optModel[jobs[q]]].S;
    ctx->polOff[q] = o;
    ctx->stats[11] += static_cast<double>(n);  // counted like d2h()
    CK(cudaMemcpyAsync(static_cast<char*>(ctx->polStage) + o, ctx->hOptJobs[jobs[q]].policy, n, cudaMemcpyDeviceToHost,
                       ctx->side));
    o += align_up(n, 256);
  }
  CK(cudaEventRecord(ctx->polCopied, ctx->side));
  ctx->polPrefetched = jobs;
  return MORAP_OK;
}

// Whole evaluate batch in one cooperative launch (k_eval_persistent). The policy chains
// must already be built; dMask / dSweeps / dResidual / dStatus are initialised.
// States per CTA of the persistent evaluate grid when every job's chains can be cached in
// shared memory (rows of <= 2 transitions, the CTA's share fits), else 0.
int eval_cache_states(morap_ctx* ctx, int njobs, size_t* cacheBytesOut = nullptr) {
  long long total = 0;
  bool narrow = true;
  for (int j = 0; j < njobs; ++j) {
    total += ctx->hm[ctx->hEvalJobs[j].model].S;
    narrow = narrow && ctx->hm[ctx->hEvalJobs[j].model].maxRowNnz <= 2;
  }
  const long long per = (total + ctx->persistBlocks - 1) / ctx->persistBlocks;
  const size_t cacheBytes = static_cast<size_t>((per + 15) & ~15ll) + 24ull * static_cast<size_t>(per) + 16;
  if (cacheBytesOut) *cacheBytesOut = cacheBytes;
  return (narrow && ctx->usePersistCache && cacheBytes <= kPersistCacheBytes) ? static_cast<int>(per) : 0;
}

int run_eval_persistent(morap_ctx* ctx, int njobs, double eps, int cap) {
  std::vector<long long> prefix(static_cast<size_t>(njobs) + 1, 0);
  for (int j = 0; j < njobs; ++j) prefix[j + 1] = prefix[j] + ctx->hm[ctx->hEvalJobs[j].model].S;
  const size_t slotBytes = 3ull * njobs * MORAP_MAX_RHS * sizeof(unsigned long long);
  int maxRhs = 1;
  for (int j = 0; j < njobs; ++j) maxRhs = std::max(maxRhs, ctx->hEvalJobs[j].nrhs);
  const int R = maxRhs <= 2 ? 2 : 4;
  const size_t interBytes = 3ull * prefix[njobs] * R * sizeof(double);  // xi (2 parities) + rhoI
  const size_t need = align_up(slotBytes, 256) + align_up(8ull * (njobs + 1), 256) + align_up(interBytes, 256);
  int rc;
  if ((rc = ensure_arena(ctx, &ctx->persistArena, &ctx->persistArenaBytes, need))) return rc;
  char* base = static_cast<char*>(ctx->persistArena);
  unsigned long long* slots = reinterpret_cast<unsigned long long*>(base);
  long long* dPrefix = reinterpret_cast<long long*>(base + align_up(slotBytes, 256));
  CK(cudaMemsetAsync(slots, 0, slotBytes, ctx->stream));
  H2D(dPrefix, prefix.data(), 8ull * (njobs + 1));
  PersistArgs a{};
  a.models = ctx->dModels;
  a.jobs = static_cast<const EvalJob*>(ctx->dEvalJobsRaw);
  a.statePrefix = dPrefix;
  a.njobs = njobs;
  a.eps = eps;
  a.cap = cap;
  a.mask = ctx->dMask;
  a.slots = slots;
  a.sweeps = ctx->dSweeps;
  a.residual = ctx->dResidual;
  a.status = ctx->dStatus;
  a.ctl = ctx->dCtl;
  a.barCount = ctx->dBar;
  a.barGen = ctx->dBar + 1;
  // shared-memory chains when every job's rows have <= 2 transitions and a CTA's states fit
  size_t cacheBytes = 0;
  a.cacheStates = eval_cache_states(ctx, njobs, &cacheBytes);
  // interleaved RHS (k_eval_interleaved) whenever the chains are cached: every job <= 4 RHS
  // here; `direct`: the kernel reads each state's chosen row from the policy itself (the
  // chain CSR was not built)
  InterArgs ia{a, nullptr, nullptr, R, ctx->evalDirect};
  const bool inter = a.cacheStates > 0 && ctx->useInterleaved;
  if (inter) {
    char* ib = base + align_up(slotBytes, 256) + align_up(8ull * (njobs + 1), 256);
    ia.xi = reinterpret_cast<double*>(ib);
    ia.rhoI = ia.xi + 2ull * prefix[njobs] * R;
    CK(cudaMemsetAsync(ia.xi, 0, 2ull * prefix[njobs] * R * sizeof(double), ctx->stream));
  }
  void* args[] = {&a};
  void* iargs[] = {&ia};
  const bool timed = ctx->profiling;
  if (timed) CK(cudaEventRecord(ctx->ev0, ctx->stream));
  if (inter)
    CK(cudaLaunchCooperativeKernel(R == 2 ? reinterpret_cast<void*>(k_eval_interleaved<2>)
                                          : reinterpret_cast<void*>(k_eval_interleaved<4>),
                                   dim3(ctx->persistBlocks), dim3(kPersistThreads), iargs, cacheBytes, ctx->stream));
  else
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_eval_persistent), dim3(ctx->persistBlocks),
                                   dim3(kPersistThreads), args, a.cacheStates ? cacheBytes : 0, ctx->stream));
  if (timed) CK(cudaEventRecord(ctx->ev1, ctx->stream));
  ctx->stats[8] += 1;
  CK(d2h(ctx, ctx->hCtl, ctx->dCtl, sizeof(Ctl)));
  CK(cudaStreamSynchronize(ctx->stream));
  if (timed) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    ctx->stats[5] += ms;
  }
  return MORAP_OK;
}

int evaluate_impl(morap_ctx* ctx, int njobs, const std::vector<EvalJob>& proto, double eps, int cap,
                  double* value_out, int32_t* sweeps_out, double* residual_out, int32_t* status_out,
                  const std::vector<uint32_t>& maskInit, const std::vector<int32_t>& statusInit) {
  int rc;
  if ((rc = ensure_ctl(ctx, njobs))) return rc;
  if (static_cast<size_t>(njobs) > ctx->dEvalJobsCap) {
    cudaFree(ctx->dEvalJobsRaw);
    ctx->dEvalJobsCap = std::max<size_t>(njobs, 64);
    CK(cudaMalloc(&ctx->dEvalJobsRaw, ctx->dEvalJobsCap * sizeof(EvalJob)));
  }
  // arena: [x/y buffers of every job and RHS][policy chains][tile counts]
  size_t xBytes = 0, chainBytes = 0, totalTiles = 0;
  bool tmaOk = ctx->useTma;
  for (int j = 0; j < njobs; ++j) {
    const HostModel& m = ctx->hm[proto[j].model];
    xBytes += 2 * proto[j].nrhs * align_up(sizeof(double) * m.S, 256);
    chainBytes += align_up(4ull * (m.S + 1), 256) + align_up(4ull * m.nnz, 256) + align_up(8ull * m.nnz, 256) +
                  proto[j].nrhs * align_up(8ull * m.S, 256);
    totalTiles += m.ntiles;
    if (proto[j].nrhs > kEvRhs) tmaOk = false;
  }
  const size_t need = xBytes + chainBytes + align_up(4ull * (totalTiles + 1), 256);
  if ((rc = ensure_arena(ctx, &ctx->evalArena, &ctx->evalArenaBytes, need))) return rc;
  ctx->hEvalJobs = proto;
  char* p = static_cast<char*>(ctx->evalArena);
  char* pc = p + xBytes;
  int32_t* tileCount = reinterpret_cast<int32_t*>(pc + chainBytes);
  std::vector<int32_t> jobModel(njobs), active, nrhs(njobs);
  for (int j = 0; j < njobs; ++j) {
    EvalJob& J = ctx->hEvalJobs[j];
    const HostModel& m = ctx->hm[J.model];
    const size_t sz = align_up(sizeof(double) * m.S, 256);
    for (int o = 0; o < J.nrhs; ++o) {
      J.buf[o][0] = reinterpret_cast<double*>(p);
      p += sz;
      J.buf[o][1] = reinterpret_cast<double*>(p);
      p += sz;
    }
    J.chainOff = reinterpret_cast<int32_t*>(pc);
    pc += align_up(4ull * (m.S + 1), 256);
    J.chainSucc = reinterpret_cast<int32_t*>(pc);
    pc += align_up(4ull * m.nnz, 256);
    J.chainProb = reinterpret_cast<double*>(pc);
    pc += align_up(8ull * m.nnz, 256);
    for (int o = 0; o < J.nrhs; ++o) {
      J.rhoC[o] = reinterpret_cast<double*>(pc);
      pc += align_up(8ull * m.S, 256);
    }
    jobModel[j] = J.model;
    nrhs[j] = J.nrhs;
    if (maskInit[j]) active.push_back(j);
  }
  if (xBytes) CK(cudaMemsetAsync(ctx->evalArena, 0, xBytes, ctx->stream));
  H2D(ctx->dEvalJobsRaw, ctx->hEvalJobs.data(), njobs * sizeof(EvalJob));
  H2D(ctx->dMask, maskInit.data(), njobs * 4);
  H2D(ctx->dNrhs, nrhs.data(), njobs * 4);
  H2D(ctx->dStatus, statusInit.data(), njobs * MORAP_MAX_RHS * 4);
  CK(cudaMemsetAsync(ctx->dSweeps, 0, njobs * MORAP_MAX_RHS * 4, ctx->stream));
  CK(cudaMemsetAsync(ctx->dDelta, 0, njobs * MORAP_MAX_RHS * sizeof(unsigned long long), ctx->stream));
  CK(cudaMemsetAsync(ctx->dResidual, 0, njobs * MORAP_MAX_RHS * sizeof(double), ctx->stream));
  if ((rc = init_ctl(ctx, active, jobModel))) return rc;
  const auto tq0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!ctx->trace) return;
    cudaStreamSynchronize(ctx->stream);
    std::fprintf(stderr, "[morap] evaluate_impl: %s at %.3f ms\n", what,
                 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - tq0).count());
  };
  lap("setup");
  ctx->evalTma = tmaOk;
  const bool persistent = tmaOk && ctx->usePersistent && njobs <= kPersistMaxJobs;
  // the interleaved kernel builds its shared-memory chains from the policies directly; from
  // the compact sweep streams when every model has them (and all its tiles fit) and the
  // rewards are the models' objectives (their class tables) -- then nothing in this batch
  // reads the upload's segment B
  ctx->evalDirect = persistent && ctx->useInterleaved && eval_cache_states(ctx, njobs) > 0 ? 1 : 0;
  if (ctx->evalDirect && ctx->evalModelRewards) {
    bool streams = true;
    for (int j = 0; j < njobs && streams; ++j)
      streams = ctx->dm[proto[j].model].compact && !ctx->hm[proto[j].model].needB;
    if (streams) ctx->evalDirect = 2;
  }
  if (ctx->evalDirect != 2 && (rc = wait_segment_b(ctx))) return rc;
  if (tmaOk && !active.empty() && !ctx->evalDirect) {
    // policy chains of the active jobs (count, per-job scan, fill)
    const int nl = ctx->hCtl->nactive, tt = ctx->hCtl->totalTiles;
    const EvalJob* ej = static_cast<const EvalJob*>(ctx->dEvalJobsRaw);
    k_chain_count<<<ctx->sweepBlocks, kBlock, 0, ctx->stream>>>(ctx->dModels, ej, ctx->dList, ctx->dPrefix, nl, tt,
                                                                tileCount);
    k_chain_scan<<<nl, 1024, 0, ctx->stream>>>(ctx->dModels, ej, ctx->dList, ctx->dPrefix, tileCount);
    k_chain_fill<<<ctx->sweepBlocks, kBlock, 0, ctx->stream>>>(ctx->dModels, ej, ctx->dList, ctx->dPrefix, nl, tt,
                                                               tileCount);
    CK(cudaGetLastError());
    ctx->stats[8] += 3;
  }
  lap("chains");
  if (!active.empty()) {
    if (persistent) {
      if ((rc = run_eval_persistent(ctx, njobs, eps, cap))) return rc;
    } else if ((rc = run_loop(ctx, 1, eps, cap))) {
      return rc;
    }
  }

  lap("sweeps");
  const int mres = njobs * MORAP_MAX_RHS;
  ctx->evalSweeps.assign(static_cast<size_t>(mres), 0);
  k_gather_eval<<<(mres + 255) / 256, 256, 0, ctx->stream>>>(ctx->dModels, (const EvalJob*)ctx->dEvalJobsRaw, njobs,
                                                              ctx->dSweeps, ctx->dStatus, ctx->dResidual,
                                                              ctx->dGather);
  CK(cudaGetLastError());
  CK(d2h(ctx, ctx->hGather, ctx->dGather, 24ull * mres));
  CK(d2h(ctx, ctx->hCtl, ctx->dCtl, sizeof(Ctl)));
  CK(cudaStreamSynchronize(ctx->stream));
  const double* vals = ctx->hGather;
  const double* res = ctx->hGather + mres;
  const int32_t* gi = reinterpret_cast<const int32_t*>(ctx->hGather + 2ull * mres);
  const int32_t* st = gi + mres;
  for (int q2 = 0; q2 < mres; ++q2) ctx->evalSweeps[q2] = gi[q2];
  double backups = 0;
  size_t q = 0;  // outputs: every job's RHS in order (j * nrhs + o for a uniform batch)
  for (int j = 0; j < njobs; ++j) {
    const EvalJob& J = ctx->hEvalJobs[j];
    for (int o = 0; o < J.nrhs; ++o, ++q) {
      const size_t s = static_cast<size_t>(j) * MORAP_MAX_RHS + o;
      value_out[q] = vals[s];
      if (sweeps_out) sweeps_out[q] = ctx->evalSweeps[s];
      if (residual_out) residual_out[q] = res[s];
      if (status_out) status_out[q] = st[s];
      backups += static_cast<double>(ctx->evalSweeps[s]) * ctx->hm[J.model].S;
    }
  }
  ctx->stats[4] += ctx->hCtl->sweepsDone;
  ctx->stats[6] += static_cast<double>(ctx->hCtl->bytes);
  ctx->stats[7] += backups;
  ctx->evalJobs = njobs;
  return MORAP_OK;
}

// ---- upload pipeline: prepare (validate, tile, compact) -> pack -> copy -> register ----
// A batch of models is packed into one device block; `morap_image` keeps a packed batch in
// pinned host memory with its DevModel records relative to kImageBase, so re-uploading the
// same products is one H2D copy (the product builder's device-layout output).

struct UploadPrep {
  std::vector<std::vector<int32_t>> tiles;
  std::vector<std::vector<TileDesc>> descs;
  std::vector<CompactStream> compact;
  std::vector<int32_t> maxRowNnz;
  // The block has two segments: A = what the compact sweeps read (tiles, dictionaries, the
  // per-tile streams, stamp groups, the out-of-window successors), B = the rest (rowOffset,
  // trnOffset, succ, done, probIdx, rclass, and the fp64 arrays of full uploads),
  // needed by the chain-CSR evaluate paths and by non-compact sweeps. An image upload copies
  // A on the stream and B on the upload stream, overlapped with the query.
  std::vector<size_t> offA, offB;  // byte offset of each model in its segment
  std::vector<size_t> lenA, lenB;
  std::vector<char> lean;          // stored without fp64 prob / objectives
  std::vector<char> needB;         // the model's sweeps read segment B (non-compact / oversized tiles)
  size_t bytesA = 0, bytes = 0;    // segment B starts at bytesA
};

int prepare_models(morap_ctx* ctx, int nmodels, const morap_csr_view* models, UploadPrep& P) {
  P.tiles.assign(nmodels, {});
  P.descs.assign(nmodels, {});
  P.compact.assign(nmodels, CompactStream{});
  P.maxRowNnz.assign(nmodels, 0);
  auto& tiles = P.tiles;
  auto& descs = P.descs;
  auto& compact = P.compact;
  auto& maxRowNnz = P.maxRowNnz;
  std::vector<int> status(nmodels, MORAP_OK);
  std::vector<std::string> why(nmodels);
  const auto tu0 = std::chrono::steady_clock::now();
  auto lapU = [&](const char* what) {
    if (ctx->trace)
      std::fprintf(stderr, "[morap] upload %d models: %s at %.3f ms\n", nmodels, what,
                   1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - tu0).count());
  };
  std::atomic<long long> phaseNs[4] = {0, 0, 0, 0};  // trace: validate, tiles, compact, streams
  parallel_for(nmodels, [&](int m) {
    morap_ctx scratch;  // per-model error text
    auto tp = std::chrono::steady_clock::now();
    auto lapP = [&](int k) {
      if (!ctx->trace) return;
      const auto now = std::chrono::steady_clock::now();
      phaseNs[k] += std::chrono::duration_cast<std::chrono::nanoseconds>(now - tp).count();
      tp = now;
    };
    status[m] = validate_view(&scratch, models[m], m);
    lapP(0);
    if (status[m]) {
      why[m] = scratch.err;
      return;
    }
    make_tiles(models[m], tiles[m], descs[m]);
    for (int r = 0; r < models[m].num_rows; ++r)
      maxRowNnz[m] = std::max(maxRowNnz[m], models[m].trn_offset[r + 1] - models[m].trn_offset[r]);
    lapP(1);
    if (ctx->useCompact) {
      build_compact(models[m], compact[m]);
      lapP(2);
      if (compact[m].ok) layout_streams(models[m], descs[m], compact[m]);
      lapP(3);
    }
  });
  if (ctx->trace)
    std::fprintf(stderr, "[morap] upload prep thread-ms: validate %.1f, tiles %.1f, compact %.1f, streams %.1f\n",
                 phaseNs[0] * 1e-6, phaseNs[1] * 1e-6, phaseNs[2] * 1e-6, phaseNs[3] * 1e-6);
  for (int m = 0; m < nmodels; ++m)
    if (status[m]) return ctx->fail(status[m], why[m]);
  lapU("validated, tiled, compacted");
  // every array of the batch in one block (two segments, see UploadPrep)
  P.offA.assign(nmodels, 0);
  P.offB.assign(nmodels, 0);
  P.lenA.assign(nmodels, 0);
  P.lenB.assign(nmodels, 0);
  P.lean.assign(nmodels, 0);
  P.needB.assign(nmodels, 0);
  size_t totA = 0, totB = 0;
  for (int m = 0; m < nmodels; ++m) {
    const morap_csr_view& v = models[m];
    const bool lean = ctx->lean && compact[m].ok && ctx->useTma;
    P.lean[m] = lean;
    bool fitsAll = true;
    for (const TileDesc& d : descs[m]) fitsAll = fitsAll && (d.fits || d.s0 == v.num_states);
    P.needB[m] = !compact[m].ok || !fitsAll;
    size_t a = align_up(4ull * tiles[m].size(), 256) + align_up(sizeof(TileDesc) * descs[m].size(), 256);
    size_t b = align_up(4ull * v.nnz, 256) + align_up(4ull * (v.num_states + 1), 256) + align_up(4ull * (v.num_rows + 1), 256) +
               (lean ? 0 : align_up(8ull * v.nnz, 256)) + align_up(1ull * v.num_states, 256) +
               (lean ? 0 : static_cast<size_t>(v.num_objectives) * align_up(8ull * v.num_rows, 256));
    if (compact[m].ok) {
      a += align_up(8ull * compact[m].dict.size(), 256) + align_up(8ull * compact[m].table.size(), 256) +
           align_up(4ull * compact[m].nTrW, 256) + align_up(4ull * compact[m].nStW, 256) +
           align_up(4ull * compact[m].nRowW, 256) + align_up(sizeof(TilePos) * compact[m].pos.size(), 256) +
           align_up(4ull * compact[m].outIdx.size(), 256) + align_up(4ull * compact[m].outGrp.size(), 256) +
           align_up(4ull * compact[m].outSucc.size(), 256);
      b += align_up(v.nnz, 256) + align_up(2ull * v.num_rows, 256);
    }
    P.offA[m] = totA;
    P.offB[m] = totB;
    P.lenA[m] = a;
    P.lenB[m] = b;
    totA += a;
    totB += b;
  }
  P.bytesA = totA;
  P.bytes = totA + totB;
  return MORAP_OK;
}

// Packs every model into `host` (layout of P) with DevModel pointers into `devBase`; with
// `dev` set, each model's block is copied as soon as it is packed (copies overlap packing).
void pack_models(morap_ctx* ctx, int nmodels, const morap_csr_view* models, const UploadPrep& P, char* host,
                 char* devBase, bool copy, std::vector<DevModel>& built, std::atomic<bool>& copyFailed,
                 std::atomic<long long>& uploadBytes) {
  const auto& tiles = P.tiles;
  const auto& descs = P.descs;
  const auto& compact = P.compact;
  void* dev = devBase;
  parallel_for(nmodels, [&](int m) {
    const morap_csr_view& v = models[m];
    char* hA = host + P.offA[m];
    char* dA = static_cast<char*>(dev) + P.offA[m];
    char* hB = host + P.bytesA + P.offB[m];
    char* dB = static_cast<char*>(dev) + P.bytesA + P.offB[m];
    DevModel dmod{};
    // src == nullptr: reserve (filled by the caller); seg 0 = A, 1 = B
    auto put = [&](int seg, const void* src, size_t n) {
      char*& h = seg ? hB : hA;
      char*& d = seg ? dB : dA;
      if (n && src) std::memcpy(h, src, n);
      char* at = d;
      const size_t a = align_up(n, 256);
      h += a;
      d += a;
      return at;
    };
    dmod.rowOffset = reinterpret_cast<const int32_t*>(put(1, v.row_offset, 4ull * (v.num_states + 1)));
    dmod.trnOffset = reinterpret_cast<const int32_t*>(put(1, v.trn_offset, 4ull * (v.num_rows + 1)));
    dmod.succ = reinterpret_cast<const int32_t*>(put(1, v.succ, 4ull * v.nnz));
    const bool lean = P.lean[m];  // fp64 prob / objectives live in the tables
    if (!lean) dmod.prob = reinterpret_cast<const double*>(put(1, v.prob, 8ull * v.nnz));
    dmod.done = reinterpret_cast<const uint8_t*>(put(1, v.done, v.num_states));
    if (!lean)
      for (int o = 0; o < v.num_objectives; ++o)
        dmod.obj[o] = reinterpret_cast<const double*>(put(1, v.rewards[o], 8ull * v.num_rows));
    dmod.tileStart = reinterpret_cast<const int32_t*>(put(0, tiles[m].data(), 4ull * tiles[m].size()));
    dmod.tiles = reinterpret_cast<const TileDesc*>(put(0, descs[m].data(), sizeof(TileDesc) * descs[m].size()));
    dmod.S = v.num_states;
    dmod.R = v.num_rows;
    dmod.nnz = v.nnz;
    dmod.initial = v.initial;
    dmod.ntiles = static_cast<int32_t>(tiles[m].size() - 1);
    dmod.K = v.num_objectives;
    dmod.rewardFinite = v.reward_finite ? 1 : 0;
    // succ 4 + prob 8 per nnz; trnOffset 4 + rho 8 per row;
    // rowOffset 4 + done 1 + x 8 + y 8 per state.
    dmod.bytesPerSweep = 12ull * v.nnz + 12ull * v.num_rows + 21ull * v.num_states;
    const CompactStream& c = compact[m];
    if (c.ok) {
      dmod.compact = 1;
      dmod.probIdx = reinterpret_cast<const uint8_t*>(put(1, c.idx.data(), c.idx.size()));
      dmod.probDict = reinterpret_cast<const double*>(put(0, c.dict.data(), 8ull * c.dict.size()));
      dmod.rclass = reinterpret_cast<const uint16_t*>(put(1, c.cls.data(), 2ull * c.cls.size()));
      dmod.classTable = reinterpret_cast<const double*>(put(0, c.table.data(), 8ull * c.table.size()));
      dmod.nclass = static_cast<int32_t>(c.table.size() / std::max(1, v.num_objectives));
      dmod.nOutSucc = static_cast<int32_t>(c.outSucc.size());
      dmod.nDict = static_cast<int32_t>(c.dict.size());
      dmod.nStW = static_cast<int32_t>(c.nStW);
      dmod.nRowW = static_cast<int32_t>(c.nRowW);
      dmod.nTrW = static_cast<int32_t>(c.nTrW);
      uint32_t* hs = reinterpret_cast<uint32_t*>(hA);
      dmod.stW = reinterpret_cast<const uint32_t*>(put(0, nullptr, 4ull * c.nStW));
      uint32_t* hr = reinterpret_cast<uint32_t*>(hA);
      dmod.rowW = reinterpret_cast<const uint32_t*>(put(0, nullptr, 4ull * c.nRowW));
      uint32_t* ht = reinterpret_cast<uint32_t*>(hA);
      dmod.trW = reinterpret_cast<const uint32_t*>(put(0, nullptr, 4ull * c.nTrW));
      fill_streams(v, descs[m], c, hs, hr, ht);  // straight into the staging buffer
      dmod.tilePos = reinterpret_cast<const TilePos*>(put(0, c.pos.data(), sizeof(TilePos) * c.pos.size()));
      dmod.outIdx = reinterpret_cast<const int32_t*>(put(0, c.outIdx.data(), 4ull * c.outIdx.size()));
      dmod.outGrp = reinterpret_cast<const int32_t*>(put(0, c.outGrp.data(), 4ull * c.outGrp.size()));
      dmod.outSucc = reinterpret_cast<const int32_t*>(put(0, c.outSucc.data(), 4ull * c.outSucc.size()));
      // compact stream: one 4-byte word per transition (window offset | index) and per row
      // (transition end | class) and per state (row end | transition end | done) + x 8 + y 8
      dmod.bytesPerSweep = 4ull * v.nnz + 4ull * v.num_rows + 20ull * v.num_states;
    }
    // evaluate, one RHS over the policy chain: chainOff 4 + done 1 + rhoC 8 + x 8 + y 8 per
    // state + 12 per chosen transition (mean nnz per row)
    const double nnzPerRow = v.num_rows ? static_cast<double>(v.nnz) / v.num_rows : 0.0;
    dmod.bytesPerEval = static_cast<unsigned long long>(v.num_states * (29.0 + 12.0 * nnzPerRow));
    built[m] = dmod;
    // this model's two parts go out as soon as they are packed (copies overlap the packing)
    uploadBytes += static_cast<long long>(P.lenA[m] + P.lenB[m]);
    if (!copy) return;
    cudaSetDevice(ctx->device);  // packing runs on pool threads
    if (cudaMemcpyAsync(static_cast<char*>(dev) + P.offA[m], host + P.offA[m], P.lenA[m], cudaMemcpyHostToDevice,
                        ctx->stream) != cudaSuccess ||
        cudaMemcpyAsync(static_cast<char*>(dev) + P.bytesA + P.offB[m], host + P.bytesA + P.offB[m], P.lenB[m],
                        cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
      copyFailed = true;
  });
}

// Appends the packed models to the context's model list and refreshes the device table.
int register_models(morap_ctx* ctx, const std::vector<DevModel>& built, const std::vector<HostModel>& hmods,
                    int32_t* ids_out) {
  const int first = static_cast<int>(ctx->hm.size());
  for (size_t m = 0; m < built.size(); ++m) {
    ctx->dm.push_back(built[m]);
    ctx->hm.push_back(hmods[m]);
    if (ids_out) ids_out[m] = first + static_cast<int>(m);
  }
  int rc;
  if ((rc = upload_models_table(ctx))) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return MORAP_OK;
}

std::vector<HostModel> host_models(const std::vector<DevModel>& built, const UploadPrep& P) {
  std::vector<HostModel> out(built.size());
  for (size_t m = 0; m < built.size(); ++m) {
    const DevModel& d = built[m];
    out[m] = HostModel{d.S, d.R, d.nnz, d.initial, d.ntiles, d.K, d.rewardFinite, P.maxRowNnz[m],
                       static_cast<int32_t>(P.compact[m].outGrp.size()), P.needB[m] ? 1 : 0};
  }
  return out;
}

// Device block for `bytes`: a released block that fits (cudaFree of ~1 GB costs up to ~0.8 s
// on B200), else a fresh allocation.
int acquire_block(morap_ctx* ctx, size_t bytes, void** out) {
  void* dev = nullptr;
  int best = -1;
  for (int q = 0; q < static_cast<int>(ctx->freeModelAllocs.size()); ++q)
    if (ctx->freeModelAllocs[q].second >= bytes &&
        (best < 0 || ctx->freeModelAllocs[q].second < ctx->freeModelAllocs[best].second))
      best = q;
  if (best >= 0) {
    dev = ctx->freeModelAllocs[best].first;
    ctx->modelAllocs.push_back(dev);
    ctx->modelAllocBytes.push_back(ctx->freeModelAllocs[best].second);
    ctx->freeModelAllocs.erase(ctx->freeModelAllocs.begin() + best);
  } else {
    if (cudaMalloc(&dev, bytes) != cudaSuccess) {  // give the cached blocks back, retry once
      cudaGetLastError();
      for (auto& f : ctx->freeModelAllocs) cudaFree(f.first);
      ctx->freeModelAllocs.clear();
      CK(cudaMalloc(&dev, bytes));
    }
    ctx->modelAllocs.push_back(dev);
    ctx->modelAllocBytes.push_back(bytes);
  }
  *out = dev;
  return MORAP_OK;
}

char* const kImageBase = reinterpret_cast<char*>(uintptr_t{1} << 40);  // DevModel pointers of an image

template <class T>
void relocate(T*& p, char* to) {
  if (p) p = reinterpret_cast<T*>(to + (reinterpret_cast<const char*>(p) - kImageBase));
}

DevModel relocated(DevModel d, char* to) {
  relocate(d.rowOffset, to);
  relocate(d.trnOffset, to);
  relocate(d.succ, to);
  relocate(d.prob, to);
  relocate(d.done, to);
  for (auto& o : d.obj) relocate(o, to);
  relocate(d.tiles, to);
  relocate(d.tileStart, to);
  relocate(d.probIdx, to);
  relocate(d.probDict, to);
  relocate(d.rclass, to);
  relocate(d.classTable, to);
  relocate(d.stW, to);
  relocate(d.rowW, to);
  relocate(d.trW, to);
  relocate(d.tilePos, to);
  relocate(d.outIdx, to);
  relocate(d.outGrp, to);
  relocate(d.outSucc, to);
  return d;
}

}  // namespace

struct morap_image {
  int device = 0;
  size_t bytes = 0, bytesA = 0;  // segment B = [bytesA, bytes)
  void* host = nullptr;           // pinned
  std::vector<DevModel> dm;       // pointers relative to kImageBase
  std::vector<HostModel> hm;
  ~morap_image() {
    if (host) cudaFreeHost(host);
  }
};

namespace {
}  // namespace

// ======================================================================================
// C ABI

extern "C" {

int morap_cuda_create(int device, morap_ctx** out) {
  if (!out) return MORAP_INVALID_CONFIG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return MORAP_CUDA_ERROR;
  if (device < 0 || device >= ndev) return MORAP_INVALID_CONFIG;
  morap_ctx* ctx = new morap_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete ctx; return MORAP_CUDA_ERROR; }
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) {
    delete ctx;
    return MORAP_CUDA_ERROR;  // built for sm_100a only
  }
  ctx->numSMs = prop.multiProcessorCount;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_chain_fill, kBlock, 0);
  int occE = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occE, k_eval_sweep, kBlock, 0);
  ctx->sweepBlocks = ctx->numSMs * std::max(1, occ);
  ctx->evalBlocks = ctx->numSMs * std::max(1, occE);
  // TMA-pipelined sweep: two ~28 KB shared-memory stages per CTA
  cudaFuncSetAttribute(k_greedy_sweep_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmemBytes);
  cudaFuncSetAttribute(k_greedy_sweep_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmemBytes);
  int occT = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occT, k_greedy_sweep_tma<false>, kTmaThreads, kTmaSmemBytes);
  ctx->tmaBlocks = ctx->numSMs * std::max(1, occT);
  cudaFuncSetAttribute(k_greedy_sweep_cmp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCmpSmemBytes);
  cudaFuncSetAttribute(k_greedy_sweep_cmp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCmpSmemBytes);
  int occC = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occC, k_greedy_sweep_cmp<false>, kTmaThreads, kCmpSmemBytes);
  ctx->cmpBlocks = ctx->numSMs * std::max(1, occC);
  int occP = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occP, k_eval_persistent, kPersistThreads, 0);
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
  cudaFuncSetAttribute(k_eval_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, kPersistCacheBytes);
  cudaFuncSetAttribute(k_eval_interleaved<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPersistCacheBytes);
  cudaFuncSetAttribute(k_eval_interleaved<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPersistCacheBytes);
  {
    int o2 = 0, o4 = 0;  // the interleaved kernel must keep the cooperative grid resident too
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_eval_interleaved<2>, kPersistThreads, kPersistCacheBytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o4, k_eval_interleaved<4>, kPersistThreads, kPersistCacheBytes);
    const char* ie = std::getenv("MORAP_EVAL_INTERLEAVED");  // "0": per-RHS layout (A/B)
    ctx->useInterleaved = std::min(o2, o4) >= std::max(1, occP) && !(ie && std::string(ie) == "0");
  }
  {
    int occCache = 0;  // the chain cache must not cost the cooperative grid its residency
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occCache, k_eval_persistent, kPersistThreads, kPersistCacheBytes);
    const char* pc = std::getenv("MORAP_PERSIST_CACHE");  // "0" disables the shared-memory chains (A/B)
    ctx->usePersistCache = occCache >= occP && occP > 0 && !(pc && std::string(pc) == "0");
  }
  int persistPerSm = std::max(1, occP);
#ifdef MORAP_DIAGNOSTICS
  if (const char* pc = std::getenv("MORAP_PERSIST_CTAS")) persistPerSm = std::max(1, std::min(occP, std::atoi(pc)));
  if (std::getenv("MORAP_TIME_SELECT")) ctx->timeSweepOnly = false;
#endif
  ctx->persistBlocks = ctx->numSMs * persistPerSm;
  const char* psel = std::getenv("MORAP_PERSISTENT");  // "0" keeps per-sweep launches (A/B)
  ctx->usePersistent = coop && occP > 0 && !(psel && std::string(psel) == "0");
  if (cudaMalloc(&ctx->dFinCount, sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(ctx->dFinCount, 0, sizeof(unsigned)) != cudaSuccess) {
    morap_cuda_destroy(ctx);
    return MORAP_CUDA_ERROR;
  }
  if (cudaMalloc(&ctx->dBar, 2 * sizeof(unsigned)) != cudaSuccess || cudaMemset(ctx->dBar, 0, 2 * sizeof(unsigned)) != cudaSuccess)
    ctx->usePersistent = false;
  cudaFuncSetAttribute(k_eval_sweep_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kEvSmemBytes);
  int occV = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occV, k_eval_sweep_tma, kTmaThreads, kEvSmemBytes);
  ctx->evalTmaBlocks = ctx->numSMs * std::max(1, occV);
  if (occT <= 0) {  // the fp64 TMA sweep cannot be resident: not an sm_100a device
    morap_cuda_destroy(ctx);
    return MORAP_CUDA_ERROR;
  }
  const char* gsel = std::getenv("MORAP_GRAPHS");  // "0" launches sweeps one by one (A/B)
  ctx->useGraphs = !(gsel && std::string(gsel) == "0");
#ifdef MORAP_DIAGNOSTICS
  if (const char* dry = std::getenv("MORAP_DEBUG_DRY")) {
    const int on = std::atoi(dry);
    cudaMemcpyToSymbol(g_dryRun, &on, sizeof(int));
  }
#endif
  const char* csel = std::getenv("MORAP_COMPACT");  // "0" keeps the plain fp64 streams (A/B)
  ctx->useCompact = !(csel && std::string(csel) == "0");
  const char* ksel = std::getenv("MORAP_SKIP");  // "0" sweeps every tile every sweep (A/B)
  ctx->skip = !(ksel && std::string(ksel) == "0");
  ctx->selBlocks = ctx->numSMs * 4;
  if (cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking) != cudaSuccess) { delete ctx; return MORAP_CUDA_ERROR; }
  if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->polReady, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->polCopied, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->segBReady, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->upload, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return MORAP_CUDA_ERROR;
  }
  ctx->stream = ctx->own;
  cudaEventCreate(&ctx->ev0);
  cudaEventCreate(&ctx->ev1);
  *out = ctx;
  return MORAP_OK;
}

int morap_cuda_destroy(morap_ctx* ctx) {
  if (!ctx) return MORAP_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (void* p : ctx->modelAllocs) cudaFree(p);
  for (auto& f : ctx->freeModelAllocs) cudaFree(f.first);
  cudaFree(ctx->dModels);
  cudaFree(ctx->buildWs);
  cudaFree(ctx->optArena);
  cudaFree(ctx->evalArena);
  cudaFree(ctx->dOptJobs);
  cudaFree(ctx->dEvalJobsRaw);
  cudaFree(ctx->dList);
  cudaFree(ctx->dPrefix);
  cudaFree(ctx->dJobModel);
  cudaFree(ctx->dDelta);
  cudaFree(ctx->dMask);
  cudaFree(ctx->dNrhs);
  cudaFree(ctx->dSweeps);
  cudaFree(ctx->dResidual);
  cudaFree(ctx->dStatus);
  cudaFree(ctx->dGather);
  if (ctx->hGather) cudaFreeHost(ctx->hGather);
  cudaFree(ctx->evalStage);
  cudaFreeHost(ctx->stage);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
  }
  if (ctx->polReady) cudaEventDestroy(ctx->polReady);
  if (ctx->polCopied) cudaEventDestroy(ctx->polCopied);
  if (ctx->segBReady) cudaEventDestroy(ctx->segBReady);
  if (ctx->upload) {
    cudaStreamSynchronize(ctx->upload);
    cudaStreamDestroy(ctx->upload);
  }
  cudaFree(ctx->dBar);
  cudaFree(ctx->dFinCount);
  cudaFree(ctx->persistArena);
  cudaFreeHost(ctx->polStage);
  for (cudaEvent_t e : ctx->evPool) cudaEventDestroy(e);
  for (auto& g : ctx->graphs) {
    cudaGraphExecDestroy(g.exec);
    for (cudaEvent_t e : g.ev) cudaEventDestroy(e);
  }
  cudaFree(ctx->dSel);
  cudaFree(ctx->dCand);
  cudaFree(ctx->dCandOut);
  cudaFree(ctx->dCandOutG);
  cudaFree(ctx->dTrace);
  cudaFree(ctx->dCtl);
  cudaFreeHost(ctx->hCtl);
  cudaEventDestroy(ctx->ev0);
  cudaEventDestroy(ctx->ev1);
  cudaStreamDestroy(ctx->own);
  delete ctx;
  return MORAP_OK;
}

int morap_cuda_set_stream(morap_ctx* ctx, void* s) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
  return MORAP_OK;
}

const char* morap_cuda_last_error(morap_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int morap_cuda_upload(morap_ctx* ctx, int nmodels, const morap_csr_view* models, int32_t* ids_out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  if (nmodels < 0 || (nmodels > 0 && !models)) return ctx->fail(MORAP_INVALID_CONFIG, "bad model list");
  if (nmodels == 0) return MORAP_OK;
  cudaSetDevice(ctx->device);
  int rc;
  UploadPrep P;
  const auto tu0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (ctx->trace)
      std::fprintf(stderr, "[morap] upload %d models: %s at %.3f ms\n", nmodels, what,
                   1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - tu0).count());
  };
  if ((rc = prepare_models(ctx, nmodels, models, P))) return rc;
  void* dev = nullptr;
  if ((rc = acquire_block(ctx, P.bytes, &dev))) return rc;
  lap("device block");
  if (P.bytes > ctx->stageBytes) {  // pinned staging, grow-only (reused by later uploads)
    // with headroom: pinning ~1 GB costs ~1 s, and the chunks of a streamed build differ
    // by a few percent (each new maximum used to re-pin the whole buffer)
    const size_t cap = P.bytes + P.bytes / 4;
    cudaFreeHost(ctx->stage);
    ctx->stage = nullptr;
    ctx->stageBytes = 0;
    CK(cudaMallocHost(&ctx->stage, cap));
    ctx->stageBytes = cap;
  }
  std::vector<DevModel> built(nmodels);
  std::atomic<bool> copyFailed{false};
  std::atomic<long long> uploadBytes{0};
  pack_models(ctx, nmodels, models, P, static_cast<char*>(ctx->stage), static_cast<char*>(dev), true, built, copyFailed,
              uploadBytes);
  lap("packed, copies queued");
  ctx->stats[9] += static_cast<double>(uploadBytes.load());
  cudaError_t e = copyFailed ? cudaErrorUnknown : cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return ctx->cudaFail(e, "upload copy", __LINE__);
  lap("copied");
  rc = register_models(ctx, built, host_models(built, P), ids_out);
  lap("registered");
  return rc;
}

int morap_cuda_build_image(morap_ctx* ctx, int nmodels, const morap_csr_view* models, morap_image** out) {
  if (!ctx || !out) return MORAP_INVALID_CONFIG;
  *out = nullptr;
  if (nmodels < 0 || (nmodels > 0 && !models)) return ctx->fail(MORAP_INVALID_CONFIG, "bad model list");
  cudaSetDevice(ctx->device);
  int rc;
  UploadPrep P;
  if (nmodels > 0 && (rc = prepare_models(ctx, nmodels, models, P))) return rc;
  auto img = std::make_unique<morap_image>();
  img->device = ctx->device;
  img->bytes = P.bytes;
  img->bytesA = P.bytesA;
  if (P.bytes) CK(cudaMallocHost(&img->host, P.bytes));
  img->dm.resize(nmodels);
  std::atomic<bool> copyFailed{false};
  std::atomic<long long> uploadBytes{0};
  if (nmodels > 0)
    pack_models(ctx, nmodels, models, P, static_cast<char*>(img->host), kImageBase, false, img->dm, copyFailed,
                uploadBytes);
  img->hm = host_models(img->dm, P);
  *out = img.release();
  return MORAP_OK;
}

int morap_cuda_upload_image(morap_ctx* ctx, const morap_image* img, int32_t* ids_out) {
  if (!ctx || !img) return MORAP_INVALID_CONFIG;
  if (img->device != ctx->device) return ctx->fail(MORAP_INVALID_CONFIG, "image was built for another device");
  if (img->dm.empty()) return MORAP_OK;
  cudaSetDevice(ctx->device);
  int rc;
  void* dev = nullptr;
  if ((rc = acquire_block(ctx, img->bytes, &dev))) return rc;
  // segment A (what the compact sweeps read) on the stream; segment B (evaluate paths,
  // non-compact sweeps) on the upload stream, overlapping the query -- the stream waits for
  // it before the first kernel that reads it (wait_segment_b)
  CK(cudaMemcpyAsync(dev, img->host, img->bytesA, cudaMemcpyHostToDevice, ctx->stream));
  if (img->bytes > img->bytesA) {
    CK(cudaMemcpyAsync(static_cast<char*>(dev) + img->bytesA, static_cast<const char*>(img->host) + img->bytesA,
                       img->bytes - img->bytesA, cudaMemcpyHostToDevice, ctx->upload));
    CK(cudaEventRecord(ctx->segBReady, ctx->upload));
    ctx->segBPending = true;
  }
  ctx->stats[9] += static_cast<double>(img->bytes);
  std::vector<DevModel> built(img->dm.size());
  for (size_t m = 0; m < built.size(); ++m) built[m] = relocated(img->dm[m], static_cast<char*>(dev));
  return register_models(ctx, built, img->hm, ids_out);
}

void morap_cuda_free_image(morap_image* img) { delete img; }

int morap_cuda_release_models(morap_ctx* ctx) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamSynchronize(ctx->upload);  // an image upload's segment B may still be copying
  ctx->segBPending = false;
  for (size_t q = 0; q < ctx->modelAllocs.size(); ++q)
    ctx->freeModelAllocs.emplace_back(ctx->modelAllocs[q], ctx->modelAllocBytes[q]);
  ctx->modelAllocs.clear();
  ctx->modelAllocBytes.clear();
  ctx->dm.clear();
  ctx->hm.clear();
  ctx->optJobs = 0;
  ctx->evalJobs = 0;
  ctx->evalSplitG = 1;
  ctx->evalSplitChunk = 0;
  return MORAP_OK;
}

int morap_cuda_build_products(morap_ctx* ctx, int nagents, const morap_build_agent* agents, int ntasks,
                              const morap_build_task* tasks, const morap_build_alphabet* alpha, int npairs,
                              const int32_t* pairs, int write, morap_build_info* info, int32_t* model_ids_out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  if (npairs < 0 || (npairs && (!agents || !tasks || !alpha || !pairs || !info)) || (write && npairs && !model_ids_out))
    return ctx->fail(MORAP_INVALID_CONFIG, "build_products: null argument");
  if (npairs == 0) return MORAP_OK;
  cudaSetDevice(ctx->device);
  {
    const cudaError_t stale = cudaPeekAtLastError();
    if (stale != cudaSuccess) return ctx->cudaFail(stale, "stale error before build_products", __LINE__);
  }
  const auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (ctx->trace)
      std::fprintf(stderr, "[morap] build_products (%d pairs, %s): %s at %.1f ms\n", npairs, write ? "write" : "measure",
                   what, 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  };
  if (alpha->num_probs < 1 || alpha->num_probs > kBuildMaxCand || alpha->num_costs < 0 ||
      alpha->num_costs >= kBuildMaxCand || alpha->num_label_sets < 1 || !alpha->probs ||
      (alpha->num_costs && !alpha->costs))
    return ctx->fail(MORAP_INVALID_CONFIG, "build_products: alphabet sizes out of range");
  int probOne = -1;
  {
    const double d1 = 1.0;
    uint64_t one;
    std::memcpy(&one, &d1, 8);
    for (int c = 0; c < alpha->num_probs; ++c) {
      uint64_t b;
      std::memcpy(&b, &alpha->probs[c], 8);
      if (b == one) probOne = c;
    }
  }
  if (probOne < 0) return ctx->fail(MORAP_INVALID_CONFIG, "build_products: the probability alphabet lacks 1.0");
  // per agent: the widest state (rows, transitions); validation of the index arrays
  std::vector<int64_t> maxRows(nagents, 1), maxEdges(nagents, 1);
  for (int a = 0; a < nagents; ++a) {
    const morap_build_agent& g = agents[a];
    const std::string who = "build_products: agent " + std::to_string(a);
    if (g.num_states < 1 || g.num_rows < 0 || g.nnz < 0 || g.initial < 0 || g.initial >= g.num_states ||
        !g.row_offset || !g.trn_offset || !g.label_set || (g.num_rows && (!g.cost_cand || !g.name_id)) ||
        (g.nnz && (!g.succ || !g.prob_cand)) || g.row_offset[0] != 0 || g.row_offset[g.num_states] != g.num_rows ||
        g.trn_offset[0] != 0 || g.trn_offset[g.num_rows] != g.nnz)
      return ctx->fail(MORAP_INVALID_MODEL, who + " is not a valid CSR");
    for (int s = 0; s < g.num_states; ++s) {
      const int r0 = g.row_offset[s], r1 = g.row_offset[s + 1];
      if (r1 < r0 || g.label_set[s] < 0 || g.label_set[s] >= alpha->num_label_sets)
        return ctx->fail(MORAP_INVALID_MODEL, who + ": row offsets / label sets");
      maxRows[a] = std::max<int64_t>(maxRows[a], r1 - r0);
      maxEdges[a] = std::max<int64_t>(maxEdges[a], g.trn_offset[r1] - g.trn_offset[r0]);
    }
    for (int r = 0; r < g.num_rows; ++r)
      if (g.trn_offset[r + 1] < g.trn_offset[r] || g.cost_cand[r] < 0 || g.cost_cand[r] >= alpha->num_costs)
        return ctx->fail(MORAP_INVALID_MODEL, who + ": rows");
    for (int k = 0; k < g.nnz; ++k)
      if (g.succ[k] < 0 || g.succ[k] >= g.num_states || g.prob_cand[k] < 0 || g.prob_cand[k] >= alpha->num_probs)
        return ctx->fail(MORAP_INVALID_MODEL, who + ": transitions");
  }
  for (int t = 0; t < ntasks; ++t) {
    const morap_build_task& d = tasks[t];
    const std::string who = "build_products: task " + std::to_string(t);
    if (d.num_locations < 1 || d.num_letters < 1 || d.initial < 0 || d.initial >= d.num_locations || !d.delta ||
        !d.flags || !d.letter_of_set)
      return ctx->fail(MORAP_INVALID_DFA, who + " is not a valid DFA");
    for (int64_t i = 0; i < static_cast<int64_t>(d.num_locations) * d.num_letters; ++i)
      if (d.delta[i] < 0 || d.delta[i] >= d.num_locations) return ctx->fail(MORAP_INVALID_DFA, who + ": transition out of range");
    for (int l = 0; l < alpha->num_label_sets; ++l)
      if (d.letter_of_set[l] < 0 || d.letter_of_set[l] >= d.num_letters)
        return ctx->fail(MORAP_INVALID_DFA, who + ": letter out of range");
  }
  // tiles: every tile but the last ends because the next state would overflow one of its caps
  // (kBlock states, kRowCap rows, kNnzCap transitions), so it holds at least kBlock states,
  // kRowCap - (widest state's rows) rows or kNnzCap - (widest state's transitions) transitions
  int64_t SQmax = 1, Rmax = 1, Nmax = 1, SAmax = 1, Tmax = 1;
  for (int k = 0; k < npairs; ++k) {
    const int a = pairs[2 * k], t = pairs[2 * k + 1];
    if (a < 0 || a >= nagents || t < 0 || t >= ntasks)
      return ctx->fail(MORAP_INVALID_CONFIG, "build_products: pair " + std::to_string(k) + " out of range");
    const int64_t SQ = static_cast<int64_t>(agents[a].num_states) * tasks[t].num_locations;
    SQmax = std::max(SQmax, SQ);
    Rmax = std::max(Rmax, SQ * maxRows[a]);
    Nmax = std::max(Nmax, SQ * maxEdges[a]);
    SAmax = std::max<int64_t>(SAmax, agents[a].num_states);
    int64_t T = SQ;
    if (maxRows[a] < kRowCap && maxEdges[a] < kNnzCap)
      T = std::min(SQ, 2 + SQ / kBlock + SQ * maxRows[a] / (kRowCap - maxRows[a]) +
                            SQ * maxEdges[a] / (kNnzCap - maxEdges[a]));
    Tmax = std::max(Tmax, T);
  }
  if (Nmax >= (int64_t{1} << 31) - 2 || Rmax >= (int64_t{1} << 31) - 2)
    return ctx->fail(MORAP_SIZE_GUARD, "build_products: a product could exceed 2^31 transitions");

  // agents, tasks, alphabet, pairs and the outputs in one device block
  std::vector<char> blob;
  auto add = [&](const void* src, size_t bytes) {
    const size_t at = blob.size();
    blob.resize(at + align_up(std::max<size_t>(bytes, 1), 256));
    if (bytes && src) std::memcpy(blob.data() + at, src, bytes);
    return at;
  };
  struct AgentOff {
    size_t row, trn, succ, pc, cc, name, lset;
  };
  struct TaskOff {
    size_t delta, flags, letter;
  };
  std::vector<AgentOff> ao(nagents);
  std::vector<TaskOff> tof(ntasks);
  const size_t offAgents = add(nullptr, sizeof(BAgent) * nagents);
  const size_t offTasks = add(nullptr, sizeof(BTask) * ntasks);
  for (int a = 0; a < nagents; ++a) {
    const morap_build_agent& g = agents[a];
    ao[a].row = add(g.row_offset, 4ull * (g.num_states + 1));
    ao[a].trn = add(g.trn_offset, 4ull * (g.num_rows + 1));
    ao[a].succ = add(g.succ, 4ull * g.nnz);
    ao[a].pc = add(g.prob_cand, 4ull * g.nnz);
    ao[a].cc = add(g.cost_cand, 4ull * g.num_rows);
    ao[a].name = add(g.name_id, 4ull * g.num_rows);
    ao[a].lset = add(g.label_set, 4ull * g.num_states);
  }
  for (int t = 0; t < ntasks; ++t) {
    const morap_build_task& d = tasks[t];
    tof[t].delta = add(d.delta, 4ull * d.num_locations * d.num_letters);
    tof[t].flags = add(d.flags, d.num_locations);
    tof[t].letter = add(d.letter_of_set, 4ull * alpha->num_label_sets);
  }
  const size_t offProbs = add(alpha->probs, 8ull * alpha->num_probs);
  const size_t offCosts = add(alpha->costs, 8ull * alpha->num_costs);
  const size_t offPairs = add(pairs, 8ull * npairs);
  const size_t offOffsets = add(nullptr, 8ull * npairs);
  const size_t offNext = add(nullptr, 4);
  const size_t upBytes = blob.size();  // the outputs are not uploaded
  const size_t offOut = add(nullptr, sizeof(BuildOut) * npairs);
  char* dBlob = nullptr;
  CK(cudaMalloc(&dBlob, blob.size()));
  struct Free {
    char* p;
    ~Free() { cudaFree(p); }
  } freeBlob{dBlob};
  auto dptr = [&](size_t off) { return reinterpret_cast<const int32_t*>(dBlob + off); };
  for (int a = 0; a < nagents; ++a) {
    const morap_build_agent& g = agents[a];
    const BAgent b{g.num_states, g.num_rows, g.nnz, g.initial, dptr(ao[a].row), dptr(ao[a].trn), dptr(ao[a].succ),
                   dptr(ao[a].pc), dptr(ao[a].cc), dptr(ao[a].name), dptr(ao[a].lset)};
    std::memcpy(blob.data() + offAgents + sizeof(BAgent) * a, &b, sizeof b);
  }
  for (int t = 0; t < ntasks; ++t) {
    const morap_build_task& d = tasks[t];
    const BTask b{d.num_locations, d.num_letters, d.initial, 0, dptr(tof[t].delta),
                  reinterpret_cast<const uint8_t*>(dBlob + tof[t].flags), dptr(tof[t].letter)};
    std::memcpy(blob.data() + offTasks + sizeof(BTask) * t, &b, sizeof b);
  }
  // write: each product's block at the prefix of the measured sizes
  size_t arenaBytes = 0;
  if (write) {
    std::vector<unsigned long long> offs(npairs);
    for (int k = 0; k < npairs; ++k) {
      if (info[k].status != MORAP_OK || info[k].bytes == 0)
        return ctx->fail(MORAP_INVALID_CONFIG, "build_products: write needs the measure results of every pair");
      offs[k] = arenaBytes;
      arenaBytes += align_up(info[k].bytes, 256);
    }
    std::memcpy(blob.data() + offOffsets, offs.data(), 8ull * npairs);
  }
  CK(cudaMemcpyAsync(dBlob, blob.data(), upBytes, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // the pageable blob is freed on return
  lap("inputs uploaded");

  // per-CTA workspaces: one CTA per SM, fewer when they would not fit in a quarter of free memory
  const size_t wsBytes = align_up(build_ws_layout(nullptr, static_cast<int>(SQmax), static_cast<int>(SQmax),
                                                  static_cast<int>(Rmax), static_cast<int>(Nmax),
                                                  static_cast<int>(SAmax), static_cast<int>(Tmax), nullptr),
                                  256);
  int grid = std::min(npairs, ctx->numSMs * kBuildCtasPerSm);
  if (ctx->buildWsBytes < wsBytes * grid) {
    if (ctx->buildWs) CK(cudaFree(ctx->buildWs));
    ctx->buildWs = nullptr;
    ctx->buildWsBytes = 0;
    size_t freeB = 0, totalB = 0;
    CK(cudaMemGetInfo(&freeB, &totalB));
    grid = static_cast<int>(std::min<size_t>(grid, std::max<size_t>(1, freeB / 4 / wsBytes)));
    CK(cudaMalloc(&ctx->buildWs, wsBytes * grid));
    ctx->buildWsBytes = wsBytes * grid;
  }
  grid = static_cast<int>(std::min<size_t>(grid, ctx->buildWsBytes / wsBytes));
  void* arena = nullptr;
  if (write) {
    const int rc = acquire_block(ctx, arenaBytes, &arena);
    if (rc) return rc;
  }
  CK(cudaMemsetAsync(dBlob + offNext, 0, 4, ctx->stream));
  BuildArgs A{};
  A.agents = reinterpret_cast<const BAgent*>(dBlob + offAgents);
  A.tasks = reinterpret_cast<const BTask*>(dBlob + offTasks);
  A.pairs = dptr(offPairs);
  A.npairs = npairs;
  A.probs = reinterpret_cast<const double*>(dBlob + offProbs);
  A.costs = reinterpret_cast<const double*>(dBlob + offCosts);
  A.nProbs = alpha->num_probs;
  A.nCosts = alpha->num_costs;
  A.probOne = probOne;
  A.internalName = alpha->internal_name;
  A.mode = write ? 1 : 0;
  A.ws = static_cast<char*>(ctx->buildWs);
  A.wsBytes = wsBytes;
  A.SQmax = static_cast<int32_t>(SQmax);
  A.Smax = static_cast<int32_t>(SQmax);
  A.Rmax = static_cast<int32_t>(Rmax);
  A.Nmax = static_cast<int32_t>(Nmax);
  A.SAmax = static_cast<int32_t>(SAmax);
  A.Tmax = static_cast<int32_t>(Tmax);
  A.arena = static_cast<char*>(arena);
  A.offsets = reinterpret_cast<const unsigned long long*>(dBlob + offOffsets);
  A.out = reinterpret_cast<BuildOut*>(dBlob + offOut);
  A.next = reinterpret_cast<int*>(dBlob + offNext);
  k_build_products<<<grid, kBT, 0, ctx->stream>>>(A);
  CK(cudaGetLastError());
  std::vector<BuildOut> out(npairs);
  CK(d2h(ctx, out.data(), dBlob + offOut, sizeof(BuildOut) * npairs));
  CK(cudaStreamSynchronize(ctx->stream));
  lap("kernel done");
  for (int k = 0; k < npairs; ++k) {
    const BuildOut& o = out[k];
    if (write && (o.bytes != info[k].bytes || o.status != MORAP_OK))
      return ctx->fail(MORAP_SOLVER_FAILURE,
                       "build_products: product " + std::to_string(k) + " differs between the measure and write passes");
    info[k] = morap_build_info{o.status, o.S, o.R, o.nnz, o.rewardFinite, o.ntiles, o.hash, o.bytes};
  }
  if (!write) return MORAP_OK;
  std::vector<DevModel> built(npairs);
  std::vector<HostModel> hmods(npairs);
  for (int k = 0; k < npairs; ++k) {
    const BuildOut& o = out[k];
    built[k] = o.dm;
    const double nnzPerRow = o.R ? static_cast<double>(o.nnz) / o.R : 0.0;  // as pack_models
    built[k].bytesPerEval = static_cast<unsigned long long>(o.S * (29.0 + 12.0 * nnzPerRow));
    hmods[k] = HostModel{o.S, o.R, o.nnz, 0, o.ntiles, 2, o.rewardFinite, o.maxRowNnz, o.nOutGrp, o.needB};
  }
  return register_models(ctx, built, hmods, model_ids_out);
}

int morap_cuda_debug_model_digest(morap_ctx* ctx, int id, uint64_t* out) {
  if (!ctx || !out) return MORAP_INVALID_CONFIG;
  if (id < 0 || id >= static_cast<int>(ctx->hm.size())) return ctx->fail(MORAP_INVALID_CONFIG, "unknown model id");
  cudaSetDevice(ctx->device);
  CK(cudaDeviceSynchronize());
  const DevModel& d = ctx->dm[static_cast<size_t>(id)];
  if (!d.compact) return ctx->fail(MORAP_INVALID_CONFIG, "digest: not a compact model");
  const size_t nt = static_cast<size_t>(d.ntiles);
  int32_t nGrp = 0;
  CK(cudaMemcpy(&nGrp, d.outIdx + nt, 4, cudaMemcpyDeviceToHost));
  const std::pair<const void*, size_t> arrays[17] = {{d.rowOffset, 4ull * (d.S + 1)},
                                                     {d.trnOffset, 4ull * (d.R + 1)},
                                                     {d.succ, 4ull * d.nnz},
                                                     {d.done, 1ull * d.S},
                                                     {d.probIdx, 1ull * d.nnz},
                                                     {d.rclass, 2ull * d.R},
                                                     {d.tileStart, 4 * (nt + 1)},
                                                     {d.tiles, sizeof(TileDesc) * (nt + 1)},
                                                     {d.probDict, 8ull * d.nDict},
                                                     {d.classTable, 8ull * d.K * d.nclass},
                                                     {d.stW, 4ull * d.nStW},
                                                     {d.rowW, 4ull * d.nRowW},
                                                     {d.trW, 4ull * d.nTrW},
                                                     {d.tilePos, sizeof(TilePos) * nt},
                                                     {d.outIdx, 4 * (nt + 1)},
                                                     {d.outGrp, 4ull * nGrp},
                                                     {d.outSucc, 4ull * d.nOutSucc}};
  std::vector<unsigned char> v;
  for (int i = 0; i < 17; ++i) {
    v.resize(arrays[i].second);
    if (!v.empty()) CK(cudaMemcpy(v.data(), arrays[i].first, v.size(), cudaMemcpyDeviceToHost));
    uint64_t h = 1469598103934665603ull ^ v.size();
    for (unsigned char c : v) h = (h ^ c) * 1099511628211ull;
    out[i] = h;
  }
  return MORAP_OK;
}

int morap_cuda_num_models(morap_ctx* ctx) { return ctx ? static_cast<int>(ctx->hm.size()) : -1; }

int morap_cuda_model_info(morap_ctx* ctx, int id, int32_t* out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  if (id < 0 || id >= static_cast<int>(ctx->hm.size())) return ctx->fail(MORAP_INVALID_CONFIG, "unknown model id");
  const DevModel& d = ctx->dm[static_cast<size_t>(id)];
  const int32_t v[6] = {d.S, d.R, d.nnz, d.K, d.compact, d.prob ? 0 : 1};
  std::memcpy(out, v, sizeof v);
  return MORAP_OK;
}

int morap_cuda_optimize(morap_ctx* ctx, int njobs, const int32_t* model_ids, const double* weights, int K, double eps,
                        int sweep_cap, double* value_out, int32_t* sweeps_out, double* residual_out,
                        int32_t* status_out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  cudaSetDevice(ctx->device);
  return optimize_impl(ctx, njobs, model_ids, weights, K, nullptr, eps, sweep_cap, value_out, sweeps_out,
                       residual_out, status_out);
}

int morap_cuda_optimize_rho(morap_ctx* ctx, int njobs, const int32_t* model_ids, const double* const* rho, double eps,
                            int sweep_cap, double* value_out, int32_t* sweeps_out, double* residual_out,
                            int32_t* status_out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  if (njobs > 0 && !rho) return ctx->fail(MORAP_INVALID_CONFIG, "null reward list");
  cudaSetDevice(ctx->device);
  return optimize_impl(ctx, njobs, model_ids, nullptr, 0, rho, eps, sweep_cap, value_out, sweeps_out, residual_out,
                       status_out);
}

int morap_cuda_fetch_values(morap_ctx* ctx, int job, double* out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  if (job < 0 || job >= ctx->optJobs) return ctx->fail(MORAP_INVALID_CONFIG, "job out of range");
  cudaSetDevice(ctx->device);
  const HostModel& m = ctx->hm[ctx->optModel[job]];
  if (ctx->optSweeps[job] <= 0) {
    std::fill(out, out + m.S, 0.0);
    return MORAP_OK;
  }
  CK(d2h(ctx, out, ctx->hOptJobs[job].buf[ctx->optSweeps[job] & 1], sizeof(double) * m.S));
  CK(cudaStreamSynchronize(ctx->stream));
  return MORAP_OK;
}

int morap_cuda_fetch_policy(morap_ctx* ctx, int job, int32_t* out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  if (job < 0 || job >= ctx->optJobs) return ctx->fail(MORAP_INVALID_CONFIG, "job out of range");
  if (ctx->optSweeps[job] <= 0) return ctx->fail(ctx->optStatus[job] ? ctx->optStatus[job] : MORAP_INVALID_CONFIG, "job has no policy");
  cudaSetDevice(ctx->device);
  int rc = extract_policies(ctx, {job});
  if (rc) return rc;
  const HostModel& m = ctx->hm[ctx->optModel[job]];
  CK(d2h(ctx, out, ctx->hOptJobs[job].policy, sizeof(int32_t) * m.S));
  CK(cudaStreamSynchronize(ctx->stream));
  return MORAP_OK;
}

int morap_cuda_policy_views(morap_ctx* ctx, int njobs, const int32_t* jobs, const int32_t** rows_out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  if (njobs <= 0) return MORAP_OK;
  std::vector<int32_t> list(jobs, jobs + njobs);
  size_t bytes = 0;
  for (int j : list) {
    if (j < 0 || j >= ctx->optJobs) return ctx->fail(MORAP_INVALID_CONFIG, "job out of range");
    if (ctx->optSweeps[j] <= 0) return ctx->fail(ctx->optStatus[j] ? ctx->optStatus[j] : MORAP_INVALID_CONFIG, "job has no policy");
    bytes += align_up(sizeof(int32_t) * ctx->hm[ctx->optModel[j]].S, 256);
  }
  cudaSetDevice(ctx->device);
  CK(cudaEventSynchronize(ctx->polCopied));  // staged by evaluate_optimized (or a stale prefetch still copying)
  if (list != ctx->polPrefetched) {
    ctx->polPrefetched.clear();
    int rc = extract_policies(ctx, list);
    if (rc) return rc;
    // one pinned staging area, one synchronisation for the whole batch
    if (bytes > ctx->polStageBytes) {
      cudaFreeHost(ctx->polStage);
      ctx->polStage = nullptr;
      ctx->polStageBytes = 0;
      CK(cudaMallocHost(&ctx->polStage, bytes));
      ctx->polStageBytes = bytes;
    }
    ctx->polOff.assign(static_cast<size_t>(njobs), 0);
    size_t o = 0;
    for (int q = 0; q < njobs; ++q) {
      const size_t n = sizeof(int32_t) * ctx->hm[ctx->optModel[list[q]]].S;
      ctx->polOff[q] = o;
      CK(d2h(ctx, static_cast<char*>(ctx->polStage) + o, ctx->hOptJobs[list[q]].policy, n));
      o += align_up(n, 256);
    }
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->polPrefetched = list;
  }
  for (int q = 0; q < njobs; ++q)
    rows_out[q] = reinterpret_cast<const int32_t*>(static_cast<char*>(ctx->polStage) + ctx->polOff[q]);
  return MORAP_OK;
}

int morap_cuda_fetch_policies(morap_ctx* ctx, int njobs, const int32_t* jobs, int32_t* const* rows_out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  if (njobs <= 0) return MORAP_OK;
  std::vector<const int32_t*> views(static_cast<size_t>(njobs));
  const int rc = morap_cuda_policy_views(ctx, njobs, jobs, views.data());
  if (rc) return rc;
  for (int q = 0; q < njobs; ++q)
    std::memcpy(rows_out[q], views[q], sizeof(int32_t) * ctx->hm[ctx->optModel[jobs[q]]].S);
  return MORAP_OK;
}

int morap_cuda_evaluate_optimized(morap_ctx* ctx, int njobs, const int32_t* opt_jobs, int nrhs, const int32_t* objective,
                                  double eps, int sweep_cap, double* value_out, int32_t* sweeps_out,
                                  double* residual_out, int32_t* status_out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  cudaSetDevice(ctx->device);
  if (njobs < 0 || nrhs < 1 || nrhs > MORAP_MAX_RHS) return ctx->fail(MORAP_INVALID_CONFIG, "bad evaluate batch");
  if (!(eps >= 0.0) || sweep_cap < 1) return ctx->fail(MORAP_INVALID_CONFIG, "bad eps / sweep cap");
  ctx->evalJobs = 0;
  ctx->evalSplitG = 1;
  ctx->evalSplitChunk = 0;
  if (njobs == 0) return MORAP_OK;
  std::vector<int32_t> jl(opt_jobs, opt_jobs + njobs);
  for (int j : jl)
    if (j < 0 || j >= ctx->optJobs) return ctx->fail(MORAP_INVALID_CONFIG, "unknown optimize job");
  for (int j : jl)
    if (ctx->optSweeps[j] <= 0 || ctx->optStatus[j] != MORAP_OK)
      return ctx->fail(ctx->optStatus[j] ? ctx->optStatus[j] : MORAP_SOLVER_FAILURE, "optimize job failed");
  const bool trace = ctx->trace;
  const auto tp0 = std::chrono::steady_clock::now();
  int rc = extract_policies(ctx, jl);
  if (rc) return rc;
  // the caller reads these policies next (supportingPoint's schedulers): copy them to the
  // pinned staging area on a side stream while the evaluate sweeps run
  if ((rc = prefetch_policies(ctx, jl))) return rc;
  if (trace) {
    cudaStreamSynchronize(ctx->stream);
    std::fprintf(stderr, "[morap] evaluate_optimized: policies %.3f ms\n",
                 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - tp0).count());
  }
  // more RHS than the chain kernels take (e.g. the 2n objectives of a centralised model):
  // G sub-jobs of <= kEvRhs RHS each on the same policy chain, consecutive, so the outputs
  // keep the caller's layout (every RHS is its own stop test: splitting changes nothing)
  const int G = nrhs > kEvRhs && ctx->useTma ? (nrhs + kEvRhs - 1) / kEvRhs : 1;
  const int chunk = (nrhs + G - 1) / G;
  std::vector<EvalJob> proto(static_cast<size_t>(njobs) * G);
  std::vector<uint32_t> mask(proto.size());
  std::vector<int32_t> st(proto.size() * MORAP_MAX_RHS, MORAP_OK);
  for (int q = 0; q < njobs; ++q) {
    const int j = jl[q];
    const int model = ctx->optModel[j];
    for (int o = 0; o < nrhs; ++o)
      if (objective[o] < 0 || objective[o] >= ctx->hm[model].K)
        return ctx->fail(MORAP_DIMENSION_MISMATCH, "objective index out of range");
    for (int g = 0; g < G; ++g) {
      EvalJob& E = proto[static_cast<size_t>(q) * G + g];
      E = EvalJob{};
      E.model = model;
      E.nrhs = std::min(chunk, nrhs - g * chunk);
      E.policy = ctx->hOptJobs[j].policy;
      for (int o = 0; o < E.nrhs; ++o) {
        E.rho[o] = ctx->dm[model].obj[objective[g * chunk + o]];  // null for lean models (class table used)
        E.objIdx[o] = objective[g * chunk + o];
      }
      mask[static_cast<size_t>(q) * G + g] = (1u << E.nrhs) - 1u;
    }
    if (!ctx->dm[model].obj[0] && !ctx->useTma)
      return ctx->fail(MORAP_INVALID_CONFIG, "lean models are evaluated through policy chains");
  }
  ctx->evalModelRewards = true;  // rewards are the models' own objective vectors
  const int rc2 = evaluate_impl(ctx, static_cast<int>(proto.size()), proto, eps, sweep_cap, value_out, sweeps_out,
                                residual_out, status_out, mask, st);
  ctx->evalSplitG = G;
  ctx->evalSplitChunk = G > 1 ? chunk : 0;
  return rc2;
}

int morap_cuda_evaluate(morap_ctx* ctx, int njobs, const int32_t* model_ids, const int32_t* const* policies,
                        const double* const* rho, double eps, int sweep_cap, double* value_out, int32_t* sweeps_out,
                        double* residual_out, int32_t* status_out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  cudaSetDevice(ctx->device);
  if (njobs < 0 || (njobs > 0 && (!model_ids || !policies || !rho)))
    return ctx->fail(MORAP_INVALID_CONFIG, "bad evaluate batch");
  if (!(eps >= 0.0) || sweep_cap < 1) return ctx->fail(MORAP_INVALID_CONFIG, "bad eps / sweep cap");
  ctx->evalJobs = 0;
  ctx->evalSplitG = 1;
  ctx->evalSplitChunk = 0;
  if (njobs == 0) return MORAP_OK;
  // stage policies + rewards in one device block
  size_t bytes = 0;
  std::vector<size_t> off(njobs);
  for (int j = 0; j < njobs; ++j) {
    if (model_ids[j] < 0 || model_ids[j] >= static_cast<int>(ctx->hm.size()))
      return ctx->fail(MORAP_INVALID_CONFIG, "unknown model id");
    const HostModel& m = ctx->hm[model_ids[j]];
    off[j] = bytes;
    bytes += align_up(4ull * m.S, 256) + align_up(8ull * m.R, 256);
  }
  int rc;
  if ((rc = ensure_arena(ctx, &ctx->evalStage, &ctx->evalStageBytes, bytes))) return rc;
  std::vector<EvalJob> proto(njobs);
  std::vector<uint32_t> mask(njobs, 1u);
  std::vector<int32_t> st(static_cast<size_t>(njobs) * MORAP_MAX_RHS, MORAP_OK);
  std::vector<int32_t> rowsHost;
  for (int j = 0; j < njobs; ++j) {
    const int model = model_ids[j];
    const HostModel& m = ctx->hm[model];
    // checkScheduler (numerics.hpp:51-66) needs rowOffset; validate against host copy
    std::vector<int32_t> ro(m.S + 1);
    CK(d2h(ctx, ro.data(), ctx->dm[model].rowOffset, 4ull * (m.S + 1), true));
    std::vector<uint8_t> dn(m.S);
    CK(d2h(ctx, dn.data(), ctx->dm[model].done, m.S, true));
    bool ok = true;
    for (int s = 0; s < m.S && ok; ++s)
      if (!dn[s] && (policies[j][s] < ro[s] || policies[j][s] >= ro[s + 1])) ok = false;
    char* base = static_cast<char*>(ctx->evalStage) + off[j];
    CK(cudaMemcpyAsync(base, policies[j], 4ull * m.S, cudaMemcpyHostToDevice, ctx->stream));
    char* rb = base + align_up(4ull * m.S, 256);
    if (m.R) CK(cudaMemcpyAsync(rb, rho[j], 8ull * m.R, cudaMemcpyHostToDevice, ctx->stream));
    EvalJob& E = proto[j];
    E = EvalJob{};
    E.model = model;
    E.nrhs = 1;
    E.policy = reinterpret_cast<const int32_t*>(base);
    E.rho[0] = reinterpret_cast<const double*>(rb);
    if (!ok) {
      mask[j] = 0;
      st[static_cast<size_t>(j) * MORAP_MAX_RHS] = MORAP_INVALID_MODEL;
    }
  }
  ctx->evalModelRewards = false;  // explicit reward vectors
  return evaluate_impl(ctx, njobs, proto, eps, sweep_cap, value_out, sweeps_out, residual_out, status_out, mask, st);
}

int morap_cuda_fetch_eval_values(morap_ctx* ctx, int job, int rhs, double* out) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  if (ctx->evalSplitChunk > 0) {  // the caller's (job, rhs) in the split batch
    if (job < 0 || job >= ctx->evalJobs / ctx->evalSplitG || rhs < 0)
      return ctx->fail(MORAP_INVALID_CONFIG, "job out of range");
    job = job * ctx->evalSplitG + rhs / ctx->evalSplitChunk;
    rhs %= ctx->evalSplitChunk;
  }
  if (job < 0 || job >= ctx->evalJobs) return ctx->fail(MORAP_INVALID_CONFIG, "job out of range");
  const EvalJob& J = ctx->hEvalJobs[job];
  if (rhs < 0 || rhs >= J.nrhs) return ctx->fail(MORAP_INVALID_CONFIG, "rhs out of range");
  cudaSetDevice(ctx->device);
  const HostModel& m = ctx->hm[J.model];
  const int sw = ctx->evalSweeps[job * MORAP_MAX_RHS + rhs];
  if (sw <= 0) {
    std::fill(out, out + m.S, 0.0);
    return MORAP_OK;
  }
  CK(d2h(ctx, out, J.buf[rhs][sw & 1], 8ull * m.S));
  CK(cudaStreamSynchronize(ctx->stream));
  return MORAP_OK;
}

int morap_cuda_set_lean(morap_ctx* ctx, int on) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  if (on && !ctx->useCompact) return ctx->fail(MORAP_INVALID_CONFIG, "lean uploads need compact streams");
  ctx->lean = on != 0;
  return MORAP_OK;
}

int morap_cuda_debug_cta_trace(morap_ctx* ctx, int enable, uint64_t* out, int64_t n) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  cudaSetDevice(ctx->device);
  const size_t words = static_cast<size_t>(kTraceSlots) * ctx->cmpBlocks * 4;
  if (enable > 0) {
    if (!ctx->dTrace) CK(cudaMalloc(&ctx->dTrace, words * 8));
    CK(cudaMemset(ctx->dTrace, 0, words * 8));
    unsigned long long* p = static_cast<unsigned long long*>(ctx->dTrace);
    CK(cudaMemcpyToSymbol(g_ctaTrace, &p, sizeof(p)));
  } else if (enable == 0) {
    unsigned long long* p = nullptr;
    CK(cudaMemcpyToSymbol(g_ctaTrace, &p, sizeof(p)));
  }
  if (out && ctx->dTrace) {
    CK(cudaStreamSynchronize(ctx->stream));
    CK(d2h(ctx, out, ctx->dTrace, std::min<size_t>(words, static_cast<size_t>(n)) * 8, true));
  }
  return MORAP_OK;
}

int morap_cuda_set_skip(morap_ctx* ctx, int on) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  ctx->skip = on != 0;
  return MORAP_OK;
}

int morap_cuda_set_profiling(morap_ctx* ctx, int on) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  ctx->profiling = on != 0;
  return MORAP_OK;
}

int morap_cuda_stats(morap_ctx* ctx, double* out, int nout) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  for (int i = 0; i < nout && i < 12; ++i) out[i] = ctx->stats[i];
  return MORAP_OK;
}

int morap_cuda_reset_stats(morap_ctx* ctx) {
  if (!ctx) return MORAP_INVALID_CONFIG;
  for (double& s : ctx->stats) s = 0.0;
  return MORAP_OK;
}

int morap_cuda_device_bytes(morap_ctx* ctx, int64_t* out) {
  if (!ctx || !out) return MORAP_INVALID_CONFIG;
  *out = static_cast<int64_t>(ctx->optArenaBytes + ctx->evalArenaBytes);
  return MORAP_OK;
}

}  // extern "C"
