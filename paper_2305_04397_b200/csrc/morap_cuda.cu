// libmorap_cuda.so -- sm_100a value-iteration backend behind include/morap_cuda.h.
//
// What runs on the GPU (reference functions replaced, /root/reference/proj/include/morap):
//   k_weighted_reward  weightedReward               numerics.hpp:224-234 (per optimize job)
//   k_greedy_sweep     optimalSchedulerOn sweep     numerics.hpp:84-113
//   k_policy           final argmax scheduler       numerics.hpp:96-102,114-115
//   k_eval_sweep       evaluateSchedulerOn sweep    numerics.hpp:138-162 (multi-RHS)
//   k_finalize_*       per-job stop test + compaction of the active set (delta <= eps,
//                      sweep cap -> NonConvergence, numerics.hpp:105-112)
//
// Layout in HBM: every uploaded model keeps the reference CSR verbatim
// (int32 rowOffset/trnOffset/succ, fp64 prob, u8 done, K fp64 objective vectors) in
// pooled device buffers, plus a tile table: state ranges of <= 256 states and <= 1024
// action rows. One optimize job = (model, rho_w fp64[R], x fp64[S] x 2, policy int32[S]).
//
// Execution: jobs advance in lock step, one sweep per k_greedy_sweep launch; the launch
// walks only the tiles of still-active jobs (a compacted job list plus a tile prefix sum
// that k_finalize rebuilds on the device after every sweep), so converged jobs cost
// nothing and there is no per-sweep host synchronisation. The host polls the active
// count once per batch of sweeps.
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

constexpr int kBlock = 256;     // threads per CTA = max states per tile
constexpr int kRowCap = 768;    // max action rows per tile (staged in shared memory)
constexpr int kNnzCap = 1024;   // max transitions per multi-state tile (staged)
constexpr int kFinBlock = 1024; // finalize kernel block
constexpr bool kFusedStates = true;  // TMA sweep: thread-per-state single pass (else 3 phases)
// Diagnostics only (MORAP_DEBUG_DRY=1): consumers skip the arithmetic, so the pipeline's
// pure streaming rate can be measured. Never set in tests or the benchmark.
__device__ int g_dryRun = 0;
// diagnostics (morap_cuda_debug_cta_trace): per compact optimize sweep and CTA, globaltimer
// stamps {start, first stage consumed, all warps done, finalize done (last CTA)}
__device__ unsigned long long* g_ctaTrace = nullptr;
constexpr int kTraceSlots = 128;
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Tile descriptor: first state / row / transition of the tile; `fits` = the tile's
// streams fit one shared-memory stage of the TMA pipeline (every multi-state tile does;
// a single state with more than kRowCap rows or kNnzCap transitions does not).
struct TileDesc {
  int32_t s0, r0, k0, fits;
  int32_t wlo, wn;  // successor window: x[wlo, wlo + wn) is staged with the tile
  int32_t allIn;    // compact: every successor of the tile lies inside the window
  int32_t simple;   // compact: every row of the tile has at most two transitions
};

// Where a tile's slice starts in each compact sweep stream. Every slice starts on a 16-byte
// boundary (the streams are padded per tile), so each lands at offset 0 of its stage region.
struct TilePos {
  int32_t row, trn, succ, pad;  // u32 state words, u32 row words, u32 transition words
};

struct DevModel {
  const int32_t* rowOffset;
  const int32_t* trnOffset;
  const int32_t* succ;
  const double* prob;
  const uint8_t* done;
  const double* obj[MORAP_MAX_OBJECTIVES];
  const TileDesc* tiles;     // ntiles + 1 (sentinel {S, R, nnz, 0})
  const int32_t* tileStart;  // ntiles + 1 state boundaries
  // compact stream: when a model has <= 256 distinct transition
  // probabilities and <= 256 distinct reward tuples, sweeps read a u8 probability index
  // per transition and a u8 reward class per row instead of fp64 prob and rho_w.
  const uint8_t* probIdx;     // nnz
  const double* probDict;     // <= 256 distinct probabilities
  const uint16_t* rclass;     // R (u16: up to kMaxClasses reward tuples)
  const double* classTable;   // nclass x K objective tuples
  // compact sweep streams, tile-major and padded per tile (TilePos): rowOffset[s + 1] -
  // tile.r0 and trnOffset[r + 1] - tile.k0 (u16), succW, and copies of probIdx / rclass / done
  const uint32_t* stW;   // per state: row end | transition end << 10 | done << 21 (tile-relative)
  const uint32_t* rowW;  // per row: tile-relative transition end (11 bits) | reward class << 11
  const uint32_t* trW;   // per transition: window offset (0xFFFF outside) | probability index << 16
  const TilePos* tilePos;     // ntiles
  // frozen-tile skipping: stamp groups (32 states) of the successors outside each tile's
  // window, outGrp[outIdx[t] .. outIdx[t + 1]) (sorted, distinct; a single -1: too many)
  const int32_t* outIdx;      // ntiles + 1
  const int32_t* outGrp;
  int32_t S, R, nnz, initial, ntiles, K, rewardFinite, compact;
  int32_t nclass, pad2;
  unsigned long long bytesPerSweep;  // algorithmic bytes of one greedy sweep
  unsigned long long bytesPerEval;   // per evaluate sweep, one RHS
};

struct OptJob {
  int32_t model;
  int32_t stampOff;  // first stamp of this job in the batch's stamp array (multiple of 4)
  double w[MORAP_MAX_OBJECTIVES];
  double* rho;
  double* classRho;  // compact models: rho_w of each reward class (nclass <= kMaxClasses)
  double* buf[2];
  int32_t* policy;
  int32_t* stamp;  // frozen-tile skipping: last sweep in which a state of group g (32 states) changed
  const int32_t* outGrp;  // the model's out-of-window stamp groups (DevModel::outGrp)
  unsigned long long bytesPerSweep;  // the model's (stats)
  int32_t nnz;
  int32_t outBase;  // this job's slice of the batch's absolute out-group list (k_build_cand)
};

struct EvalJob {
  int32_t model;
  int32_t nrhs;
  const int32_t* policy;
  const double* rho[MORAP_MAX_RHS];
  double* buf[MORAP_MAX_RHS][2];
  // policy chain (compact CSR of the chosen rows, built once per evaluate call)
  int32_t* chainOff;   // S + 1
  int32_t* chainSucc;  // <= nnz
  double* chainProb;   // <= nnz
  double* rhoC[MORAP_MAX_RHS];  // rho_o of each state's chosen row
  int32_t objIdx[MORAP_MAX_RHS];  // objective of each RHS (lean models read the class table)
};

// Device control block for one batch loop.
struct Ctl {
  int32_t nactive;      // jobs in the active list
  int32_t totalTiles;   // tiles of active jobs (tilePrefix[nactive])
  int32_t sweepsDone;   // sweeps completed by every active job
  int32_t nsel;         // tiles selected for the current sweep (k_select); reset by the finalize
  int32_t claimed;      // dynamic tail of the selected tiles: claimed so far; reset by the finalize
  int32_t nactNext;     // k_select mode: jobs k_select let into the coming sweep
  unsigned long long bytes;    // algorithmic bytes of all sweeps so far
  unsigned long long backups;  // nnz backups of all sweeps so far (every tile of every active job)
  unsigned long long execBytes;    // of the tiles actually swept (k_select mode)
  unsigned long long execBackups;
};

// --------------------------------------------------------------------------------------
// device helpers

__device__ __forceinline__ int find_slot(const int32_t* __restrict__ prefix, int n, int t) {
  // largest a with prefix[a] <= t  (prefix[0] = 0, prefix[n] = total)
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ double row_value(const int32_t* __restrict__ trn, const int32_t* __restrict__ succ,
                                            const double* __restrict__ prob, const double* __restrict__ rho,
                                            const double* __restrict__ x, int r) {
  // numerics.hpp:94-95: v = rho[r]; v += prob[k] * x[succ[k]] left to right, no FMA.
  double v = rho[r];
  const int kb = trn[r], ke = trn[r + 1];
  for (int k = kb; k < ke; ++k) v = __dadd_rn(v, __dmul_rn(prob[k], __ldg(x + succ[k])));
  return v;
}

// Model accessors that work for lean compact models too (no fp64 prob / objective arrays
// on the device: the values come from the model's dictionary / class table, bit-identical).
__device__ __forceinline__ double model_prob(const DevModel& M, int k) {
  return M.prob ? M.prob[k] : M.probDict[M.probIdx[k]];
}
__device__ __forceinline__ double model_obj(const DevModel& M, int o, int r) {
  return M.obj[o] ? M.obj[o][r] : M.classTable[M.rclass[r] * M.K + o];
}
// row value of the compact kernel's fallback path: rho_w from the job's class table
__device__ __forceinline__ double row_value_cmp(const DevModel& M, const double* __restrict__ classRho,
                                               const double* __restrict__ x, int r) {
  double v = classRho[M.rclass[r]];
  const int kb = M.trnOffset[r], ke = M.trnOffset[r + 1];
  for (int k = kb; k < ke; ++k) v = __dadd_rn(v, __dmul_rn(M.probDict[M.probIdx[k]], __ldg(x + M.succ[k])));
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int NW>
__device__ __forceinline__ double block_max(double v, double* red) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = lane < NW ? red[lane] : 0.0;
    r = warp_max(r);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// --------------------------------------------------------------------------------------
// K3: rho_w[r] = 0 + w0*obj0[r] + w1*obj1[r] + ...  (numerics.hpp:227-231)

__global__ void __launch_bounds__(kBlock) k_weighted_reward(const DevModel* __restrict__ models,
                                                            const OptJob* __restrict__ jobs,
                                                            const int32_t* __restrict__ list,
                                                            const int32_t* __restrict__ prefix, int nlist,
                                                            int total) {
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int a = find_slot(prefix, nlist + 1, t);
    const OptJob& J = jobs[list[a]];
    const DevModel& M = models[J.model];
    const int lt = t - prefix[a];
    const int s0 = M.tileStart[lt], s1 = M.tileStart[lt + 1];
    const int r0 = M.rowOffset[s0], r1 = M.rowOffset[s1];
    if (J.rho)  // lean compact jobs keep only the class table below
      for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        double acc = 0.0;
        for (int o = 0; o < M.K; ++o) acc = __dadd_rn(acc, __dmul_rn(J.w[o], M.obj[o][r]));
        J.rho[r] = acc;
      }
    if (M.compact && lt == 0) {
      // the same rounded combination for every reward class: rho_w[r] == classRho[rclass[r]]
      for (int c = threadIdx.x; c < M.nclass; c += blockDim.x) {
        double acc = 0.0;
        for (int o = 0; o < M.K; ++o) acc = __dadd_rn(acc, __dmul_rn(J.w[o], M.classTable[c * M.K + o]));
        J.classRho[c] = acc;
      }
    }
  }
}

// classRho of every active compact job (one CTA per job): the same rounded combination as
// weightedReward for each reward class, rho_w[r] == classRho[rclass[r]].
__global__ void __launch_bounds__(kBlock) k_class_rho(const DevModel* __restrict__ models,
                                                      const OptJob* __restrict__ jobs,
                                                      const int32_t* __restrict__ list) {
  const OptJob& J = jobs[list[blockIdx.x]];
  const DevModel& M = models[J.model];
  for (int c = threadIdx.x; c < M.nclass; c += blockDim.x) {
    double acc = 0.0;
    for (int o = 0; o < M.K; ++o) acc = __dadd_rn(acc, __dmul_rn(J.w[o], M.classTable[c * M.K + o]));
    J.classRho[c] = acc;
  }
}

// --------------------------------------------------------------------------------------
// K1: one greedy Jacobi sweep over the tiles of every active optimize job
// (numerics.hpp:86-104). Phase 1: threads own action rows (coalesced trnOffset / rho /
// succ / prob streams), row values land in shared memory. Phase 2: threads own states
// and scan their rows in order for the first strict maximum.
// POLICY = true: recompute the argmax of the final sweep from x_{k-1} and store rows.

template <bool POLICY>
__global__ void __launch_bounds__(kBlock) k_greedy_sweep(const DevModel* __restrict__ models,
                                                         const OptJob* __restrict__ jobs,
                                                         const int32_t* __restrict__ list,
                                                         const int32_t* __restrict__ prefix,
                                                         const Ctl* __restrict__ ctl,
                                                         const int32_t* __restrict__ jobSweeps,
                                                         unsigned long long* __restrict__ deltaBits) {
  __shared__ int32_t sRow[kBlock + 1];
  __shared__ double sVal[kRowCap];
  __shared__ double sRed[kBlock / 32];

  const int nact = ctl->nactive;
  const int total = ctl->totalTiles;
  if (total <= 0) return;
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per;
  const int t1 = min(total, t0 + per);
  if (t0 >= t1) return;
  int a = find_slot(prefix, nact + 1, t0);
  const int k = ctl->sweepsDone;

  for (int t = t0; t < t1; ++t) {
    while (t >= prefix[a + 1]) ++a;
    const int job = list[a];
    const OptJob& J = jobs[job];
    const DevModel& M = models[J.model];
    const int lt = t - prefix[a];
    const int s0 = M.tileStart[lt];
    const int ns = M.tileStart[lt + 1] - s0;
    const int32_t* __restrict__ trn = M.trnOffset;
    const int32_t* __restrict__ succ = M.succ;
    const double* __restrict__ prob = M.prob;
    const double* __restrict__ rho = J.rho;
    int parity = k & 1;
    if (POLICY) parity = (jobSweeps[job] - 1) & 1;
    const double* __restrict__ x = J.buf[parity];
    double* __restrict__ y = J.buf[parity ^ 1];

    for (int i = threadIdx.x; i <= ns; i += kBlock) sRow[i] = M.rowOffset[s0 + i];
    __syncthreads();
    const int r0 = sRow[0];
    const int nr = sRow[ns] - r0;
    const int nstage = min(nr, kRowCap);
    for (int i = threadIdx.x; i < nstage; i += kBlock) sVal[i] = row_value(trn, succ, prob, rho, x, r0 + i);
    __syncthreads();

    double d = 0.0;
    if (threadIdx.x < ns) {
      const int s = s0 + threadIdx.x;
      const int rb = sRow[threadIdx.x] - r0, re = sRow[threadIdx.x + 1] - r0;
      if (M.done[s]) {
        if (POLICY) J.policy[s] = r0 + rb;  // numerics.hpp:114-115
      } else {
        double best = 0.0;
        int bestRow = -1;
        for (int q = rb; q < re; ++q) {
          const double v = q < kRowCap ? sVal[q] : row_value(trn, succ, prob, rho, x, r0 + q);
          if (bestRow < 0 || v > best) {
            best = v;
            bestRow = q;
          }
        }
        if (POLICY) {
          J.policy[s] = r0 + bestRow;
        } else {
          y[s] = best;
          d = fabs(__dsub_rn(best, x[s]));
        }
      }
    }
    if (!POLICY) {
      d = block_max<kBlock / 32>(d, sRed);
      if (threadIdx.x == 0 && d > 0.0) atomicMax(deltaBits + job, (unsigned long long)__double_as_longlong(d));
    } else {
      __syncthreads();
    }
  }
}

// --------------------------------------------------------------------------------------
// K1 (TMA pipeline): the same sweep with every tile's five CSR streams (rowOffset,
// trnOffset, rho, succ, prob) and the done bytes brought into shared memory by 1-D bulk
// async copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier, double-buffered:
// while the CTA computes tile i from stage i&1, the copies of the next tile are in
// flight. Streaming copies carry an L2 evict-first policy so the x vectors (gathered
// through L2) stay resident. Phases per tile:
//   1a  t_k = prob[k] * x[succ[k]]          thread per transition (independent gathers)
//   1b  v_r = rho[r] + t_k + t_k' + ...      thread per row, left to right (in place)
//   2   first strict max over the state's rows, y, |y - x| -> block max -> atomicMax
// 1a/1b is the same rounded arithmetic as row_value (product rounded, then the sum),
// so results stay bitwise identical. Tiles that do not fit a stage take the global path.

constexpr int kStRowInts = 264;    // >= kBlock + 1 + 3 (front misalignment), multiple of 4
constexpr int kStTrnInts = kRowCap + 8;    // >= kRowCap + 1 + 3, multiple of 4
constexpr int kStRhoDbls = kRowCap + 2;    // >= kRowCap + 1, even
constexpr int kStSuccInts = kNnzCap + 4;   // >= kNnzCap + 3
constexpr int kStProbDbls = kNnzCap + 2;   // >= kNnzCap + 1
constexpr int kStDoneBytes = 272;  // >= kBlock + 15
constexpr int kStXDbls = 258;      // >= kBlock + 1 (own states' x for the residual)
constexpr int kOffRow = 0;
constexpr int kOffTrn = kOffRow + 4 * kStRowInts;
constexpr int kOffRho = kOffTrn + 4 * kStTrnInts;
constexpr int kOffSucc = kOffRho + 8 * kStRhoDbls;
constexpr int kOffProb = kOffSucc + 4 * kStSuccInts;
constexpr int kOffDone = kOffProb + 8 * kStProbDbls;
constexpr int kOffX = kOffDone + kStDoneBytes;
constexpr int kOffIdx = kOffX + 8 * kStXDbls;  // compact models: u8 probability index per transition
constexpr int kOffCls = kOffIdx + kNnzCap + 16;  // compact models: u16 reward class per row
#ifndef MORAP_XWIN
#define MORAP_XWIN 992
#endif
constexpr int kXWin = MORAP_XWIN;                        // successor window of x staged per tile
constexpr int kOffXw = kOffCls + 2 * kRowCap + 16;
constexpr int kStageBytes = kOffXw + 8 * (kXWin + 2);
static_assert(kStageBytes % 16 == 0 && kOffTrn % 16 == 0 && kOffRho % 16 == 0 && kOffSucc % 16 == 0 &&
                  kOffProb % 16 == 0 && kOffDone % 16 == 0 && kOffX % 16 == 0 && kOffIdx % 16 == 0 &&
                  kOffXw % 16 == 0 &&
                  kOffCls % 16 == 0,
              "stage regions must be 16-byte aligned");
#ifndef MORAP_STAGES
#define MORAP_STAGES 2
#endif
constexpr int kStages = MORAP_STAGES;  // TMA pipeline depth of the greedy sweep
constexpr int kTmaSmemBytes = kStages * kStageBytes;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Same, but a waiting warp is suspended up to `kSuspendNs` per try instead of re-issuing
// the test in a tight loop (the spin took ~20% of the compact sweep's issue slots).
#ifndef MORAP_SUSPEND_NS
#define MORAP_SUSPEND_NS 20000
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity), "n"(MORAP_SUSPEND_NS)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

// Copy elements [b, e) of `base` (element size es) with 16-byte aligned source and size;
// returns the element offset of `b` inside the staged copy.
__device__ __forceinline__ int stage_range(unsigned char* dst, const void* base, long long b, long long e, int es,
                                           uint64_t* bar, uint64_t pol, uint32_t& tx) {
  const long long lo = (b * es) & ~15ll;
  const long long hi = (e * es + 15) & ~15ll;
  if (hi > lo) {
    bulk_g2s(dst, static_cast<const unsigned char*>(base) + lo, static_cast<uint32_t>(hi - lo), bar, pol);
    tx += static_cast<uint32_t>(hi - lo);
  }
  return static_cast<int>((b * es - lo) / es);
}

// What the producer warp resolved for one staged tile (consumers never walk the
// prefix / job / model / tile tables themselves).
struct StageInfo {
  int t;  // global tile index, -1 = end of this CTA's range
  int job, fits, compact;
  int s0, r0, k0, ns, nr, nz;
  int offRow, offTrn, offRho, offSucc, offProb, offDone, offX, offIdx, offCls, offXw;
  int wlo, wn;
  const double* dict;      // compact: probability dictionary
  const double* classRho;  // compact: rho_w per reward class
  const double* x;
  double* y;
  int32_t* policy;
  const TileDesc* tiles;  // fallback path only
  const DevModel* model;
  const double* rho;
};

constexpr int kConsumers = kBlock;           // 8 compute warps
constexpr int kTmaThreads = kBlock + 32;     // + 1 producer warp

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// block max over the 256 consumer threads (named barrier 1)
__device__ __forceinline__ double consumer_max(double v, double* red) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  consumer_sync();
  double r = 0.0;
  if (threadIdx.x < 32) r = warp_max(lane < kConsumers / 32 ? red[lane] : 0.0);
  consumer_sync();
  return r;
}

// row value from the staged products: rho + t_k + t_k' ... (left to right)
__device__ __forceinline__ double staged_row(const double* rhoS, const int32_t* trnS, const double* prodS, int i,
                                             int k0) {
  double acc = rhoS[i];
  const int kb = trnS[i] - k0, ke = trnS[i + 1] - k0;
  const int n = ke - kb;
  if (n == 1) return __dadd_rn(acc, prodS[kb]);
  if (n == 2) return __dadd_rn(__dadd_rn(acc, prodS[kb]), prodS[kb + 1]);
  for (int q = kb; q < ke; ++q) acc = __dadd_rn(acc, prodS[q]);
  return acc;
}

template <bool POLICY>
__global__ void __launch_bounds__(kTmaThreads, kStages >= 3 ? 2 : 3) k_greedy_sweep_tma(const DevModel* __restrict__ models,
                                                                     const OptJob* __restrict__ jobs,
                                                                     const int32_t* __restrict__ list,
                                                                     const int32_t* __restrict__ prefix,
                                                                     const Ctl* __restrict__ ctl,
                                                                     const int32_t* __restrict__ jobSweeps,
                                                                     unsigned long long* __restrict__ deltaBits) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ StageInfo info[kStages];
  __shared__ double sRed[kConsumers / 32];

  const int nact = ctl->nactive;
  const int total = ctl->totalTiles;
  if (total <= 0) return;
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per;
  const int t1 = min(total, t0 + per);
  if (t0 >= t1) return;
  const int k = ctl->sweepsDone;
  const int tid = threadIdx.x;

  if (tid == 0) {
    for (int q = 0; q < kStages; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (tid >= kConsumers) {
    // ---------------- producer warp: resolve tiles, stage them with bulk copies ----------
    // Every lane resolves the tile (broadcast loads), lane i issues stream i's bulk copy,
    // so the eight copies of a tile go out in parallel instead of one after another.
    const int lane = tid & 31;
    const uint64_t pol = evict_first_policy(), polKeep = evict_last_policy();
    int ai = find_slot(prefix, nact + 1, t0);
    int use = 0;
    auto acquire = [&](int b) {
      if (use >= kStages) mbar_wait(&empty[b], ((use / kStages) - 1) & 1);
    };
    for (int ti = t0; ti < t1; ++ti, ++use) {
      while (ti >= prefix[ai + 1]) ++ai;
      const int job = list[ai];
      const OptJob& J = jobs[job];
      const DevModel* M = &models[J.model];
      const int lt = ti - prefix[ai];
      const TileDesc d = M->tiles[lt], e = M->tiles[lt + 1];
      const int parity = POLICY ? ((jobSweeps[job] - 1) & 1) : (k & 1);
      const int b = use % kStages;
      const double* xcur = J.buf[parity];
      const bool cp = M->compact != 0 && J.classRho != nullptr;  // explicit-rho jobs stream fp64 rho
      // this lane's stream: 0 rowOffset, 1 trnOffset, 2 succ, 3 rho|class, 4 prob|index, 5 done,
      // 6 own x, 7 successor window of x
      const void* src = nullptr;
      long long lo = 0, hi = 0;
      int es = 1, dstOff = 0;
      uint64_t lp = pol;
      switch (lane) {
        case 0: src = M->rowOffset; lo = d.s0; hi = e.s0 + 1; es = 4; dstOff = kOffRow; break;
        case 1: src = M->trnOffset; lo = d.r0; hi = e.r0 + 1; es = 4; dstOff = kOffTrn; break;
        case 2: src = M->succ; lo = d.k0; hi = e.k0; es = 4; dstOff = kOffSucc; break;
        case 3:
          if (cp) { src = M->rclass; es = 2; dstOff = kOffCls; }
          else { src = J.rho; es = 8; dstOff = kOffRho; }
          lo = d.r0; hi = e.r0;
          break;
        case 4:
          if (cp) { src = M->probIdx; es = 1; dstOff = kOffIdx; }
          else { src = M->prob; es = 8; dstOff = kOffProb; }
          lo = d.k0; hi = e.k0;
          break;
        case 5: src = M->done; lo = d.s0; hi = e.s0; es = 1; dstOff = kOffDone; break;
        case 6:
          if (!POLICY) { src = xcur; lo = d.s0; hi = e.s0; es = 8; dstOff = kOffX; lp = polKeep; }
          break;
        case 7: src = xcur; lo = d.wlo; hi = d.wlo + d.wn; es = 8; dstOff = kOffXw; lp = polKeep; break;
        default: break;
      }
      const long long a0 = (lo * es) & ~15ll, z0 = (hi * es + 15) & ~15ll;
      const uint32_t bytes = (src && d.fits && z0 > a0) ? static_cast<uint32_t>(z0 - a0) : 0u;
      const int off = src ? static_cast<int>((lo * es - a0) / es) : 0;
      const uint32_t txBytes = __reduce_add_sync(0xffffffffu, bytes);
      const int o0 = __shfl_sync(0xffffffffu, off, 0), o1 = __shfl_sync(0xffffffffu, off, 1),
                o2 = __shfl_sync(0xffffffffu, off, 2), o3 = __shfl_sync(0xffffffffu, off, 3),
                o4 = __shfl_sync(0xffffffffu, off, 4), o5 = __shfl_sync(0xffffffffu, off, 5),
                o6 = __shfl_sync(0xffffffffu, off, 6), o7 = __shfl_sync(0xffffffffu, off, 7);
      acquire(b);
      uint64_t* bar = &full[b];
      if (lane == 0) {
        StageInfo v;
        v.t = ti;
        v.job = job;
        v.fits = d.fits;
        v.compact = cp;
        v.s0 = d.s0;
        v.r0 = d.r0;
        v.k0 = d.k0;
        v.ns = e.s0 - d.s0;
        v.nr = e.r0 - d.r0;
        v.nz = e.k0 - d.k0;
        v.offRow = o0;
        v.offTrn = o1;
        v.offSucc = o2;
        v.offRho = cp ? 0 : o3;
        v.offCls = cp ? o3 : 0;
        v.offProb = cp ? 0 : o4;
        v.offIdx = cp ? o4 : 0;
        v.offDone = o5;
        v.offX = o6;
        v.offXw = o7;
        v.wlo = d.wlo;
        v.wn = d.wn;
        v.dict = M->probDict;
        v.classRho = J.classRho;
        v.x = xcur;
        v.y = J.buf[parity ^ 1];
        v.policy = J.policy;
        v.tiles = M->tiles;
        v.model = M;
        v.rho = J.rho;
        info[b] = v;
        if (d.fits) mbar_expect_tx(bar, txBytes);  // arrive (release: info[b] visible to waiters)
        else mbar_arrive(bar);                     // no copies: consumers take the global path
      }
      __syncwarp();
      if (bytes) bulk_g2s(smem + b * kStageBytes + dstOff, static_cast<const unsigned char*>(src) + a0, bytes, bar, lp);
    }
    if (lane == 0) {
      const int b = use % kStages;
      acquire(b);
      info[b].t = -1;
      mbar_arrive(&full[b]);
    }
    return;
  }

  // ---------------- consumer warps ---------------------------------------------------------
  for (int use = 0;; ++use) {
    const int b = use % kStages;
    mbar_wait(&full[b], (use / kStages) & 1);
    const StageInfo v = info[b];
    if (v.t < 0) break;
    double dl = 0.0;
    if (v.fits && g_dryRun) {
      // diagnostics: staged but not computed
    } else if (v.fits) {
      unsigned char* st = smem + b * kStageBytes;
      const int32_t* rowS = reinterpret_cast<const int32_t*>(st + kOffRow) + v.offRow;
      const int32_t* trnS = reinterpret_cast<const int32_t*>(st + kOffTrn) + v.offTrn;
      double* rhoS = reinterpret_cast<double*>(st + kOffRho) + v.offRho;  // compact: offRho = 0
      const int32_t* succS = reinterpret_cast<const int32_t*>(st + kOffSucc) + v.offSucc;
      double* prodS = reinterpret_cast<double*>(st + kOffProb) + v.offProb;  // compact: offProb = 0
      const uint8_t* doneS = st + kOffDone + v.offDone;
      const double* xS = reinterpret_cast<const double*>(st + kOffX) + v.offX;
      const double* __restrict__ x = v.x;
      if (kFusedStates) {
        // thread per state, one pass: a state's rows -- and so its transitions -- are
        // contiguous, so the thread first forms all its rounded products t_k =
        // prob_k * x[succ_k] (independent gathers, written to its own slice of the stage),
        // then accumulates each row left to right from rho and keeps the first strict max
        // (numerics.hpp:86-103). No barrier between the phases: nothing is shared.
        if (tid < v.ns) {
          const int s = v.s0 + tid;
          const int rb = rowS[tid] - v.r0, re = rowS[tid + 1] - v.r0;
          if (doneS[tid]) {
            if (POLICY) v.policy[s] = v.r0 + rb;  // numerics.hpp:114-115
          } else {
            const int qb = trnS[rb] - v.k0, qe = trnS[re] - v.k0;
            const double* xwS = reinterpret_cast<const double*>(st + kOffXw) + v.offXw;
            auto xAt = [&](int sIdx) {  // staged window, else global (rare long-range successor)
              const unsigned off = static_cast<unsigned>(sIdx - v.wlo);
              return off < static_cast<unsigned>(v.wn) ? xwS[off] : __ldg(x + sIdx);
            };
            if (v.compact) {
              const uint8_t* idxS = st + kOffIdx + v.offIdx;
#pragma unroll 4
              for (int q = qb; q < qe; ++q) prodS[q] = __dmul_rn(__ldg(v.dict + idxS[q]), xAt(succS[q]));
            } else {
#pragma unroll 4
              for (int q = qb; q < qe; ++q) prodS[q] = __dmul_rn(prodS[q], xAt(succS[q]));
            }
            const uint16_t* clsS = reinterpret_cast<const uint16_t*>(st + kOffCls) + v.offCls;
            double best = 0.0;
            int bestRow = -1;
            int kb = qb;
            for (int r = rb; r < re; ++r) {
              const int ke = trnS[r + 1] - v.k0;
              double acc = v.compact ? __ldg(v.classRho + clsS[r]) : rhoS[r];
              for (int q = kb; q < ke; ++q) acc = __dadd_rn(acc, prodS[q]);
              kb = ke;
              if (bestRow < 0 || acc > best) {
                best = acc;
                bestRow = r;
              }
            }
            if (POLICY) {
              v.policy[s] = v.r0 + bestRow;
            } else {
              v.y[s] = best;
              dl = fabs(__dsub_rn(best, xS[tid]));
            }
          }
        }
      } else if (v.compact) {
        // compact stream: prob from the model's dictionary, rho_w from the job's class table
        // (the same fp64 values, so the same rounded products and sums)
        const uint8_t* idxS = st + kOffIdx + v.offIdx;
        const uint16_t* clsS = reinterpret_cast<const uint16_t*>(st + kOffCls) + v.offCls;
#pragma unroll 4
        for (int i = tid; i < v.nz; i += kConsumers)
          prodS[i] = __dmul_rn(__ldg(v.dict + idxS[i]), __ldg(x + succS[i]));
        consumer_sync();
        for (int i = tid; i < v.nr; i += kConsumers) {
          const int kb = trnS[i] - v.k0, ke = trnS[i + 1] - v.k0;
          double acc = __ldg(v.classRho + clsS[i]);
          for (int q = kb; q < ke; ++q) acc = __dadd_rn(acc, prodS[q]);
          rhoS[i] = acc;
        }
        consumer_sync();
      } else {
        // 1a: t_k = prob[k] * x[succ[k]] for every transition (independent gathers)
#pragma unroll 4
        for (int i = tid; i < v.nz; i += kConsumers) prodS[i] = __dmul_rn(prodS[i], __ldg(x + succS[i]));
        consumer_sync();
        // 1b: row values, left to right from rho (numerics.hpp:94-95), written over rho
        for (int i = tid; i < v.nr; i += kConsumers) rhoS[i] = staged_row(rhoS, trnS, prodS, i, v.k0);
        consumer_sync();
      }
      // 2: first strict maximum over the state's rows (numerics.hpp:96-103)
      if (!kFusedStates && tid < v.ns) {
        const int s = v.s0 + tid;
        const int rb = rowS[tid] - v.r0, re = rowS[tid + 1] - v.r0;
        if (doneS[tid]) {
          if (POLICY) v.policy[s] = v.r0 + rb;  // numerics.hpp:114-115
        } else {
          double best = rhoS[rb];
          int bestRow = rb;
          for (int q = rb + 1; q < re; ++q) {
            const double val = rhoS[q];
            if (val > best) {
              best = val;
              bestRow = q;
            }
          }
          if (POLICY) {
            v.policy[s] = v.r0 + bestRow;
          } else {
            v.y[s] = best;
            dl = fabs(__dsub_rn(best, xS[tid]));
          }
        }
      }
    } else {
      // oversized single-state tile: rows straight from global memory (its stage slot
      // carries no copies, so it holds the row offsets and staged row values instead)
      const DevModel& M = *v.model;
      const double* __restrict__ x = v.x;
      int32_t* sRow = reinterpret_cast<int32_t*>(smem + b * kStageBytes + kOffRow);
      double* sVal = reinterpret_cast<double*>(smem + b * kStageBytes + kOffRho);
      for (int i = tid; i <= v.ns; i += kConsumers) sRow[i] = M.rowOffset[v.s0 + i];
      consumer_sync();
      const int r0 = sRow[0];
      const int nr = sRow[v.ns] - r0;
      const int nstage = min(nr, kRowCap);
      for (int i = tid; i < nstage; i += kConsumers) sVal[i] = row_value(M.trnOffset, M.succ, M.prob, v.rho, x, r0 + i);
      consumer_sync();
      if (tid < v.ns) {
        const int s = v.s0 + tid;
        const int rb = sRow[tid] - r0, re = sRow[tid + 1] - r0;
        if (M.done[s]) {
          if (POLICY) v.policy[s] = r0 + rb;
        } else {
          double best = 0.0;
          int bestRow = -1;
          for (int q = rb; q < re; ++q) {
            const double val = q < kRowCap ? sVal[q] : row_value(M.trnOffset, M.succ, M.prob, v.rho, x, r0 + q);
            if (bestRow < 0 || val > best) {
              best = val;
              bestRow = q;
            }
          }
          if (POLICY) {
            v.policy[s] = r0 + bestRow;
          } else {
            v.y[s] = best;
            dl = fabs(__dsub_rn(best, x[s]));
          }
        }
      }
    }
    if (!POLICY) {
      dl = consumer_max(dl, sRed);  // both named barriers: every consumer is done with stage b
      if (tid == 0 && dl > 0.0) atomicMax(deltaBits + v.job, (unsigned long long)__double_as_longlong(dl));
    } else {
      consumer_sync();
    }
    if (tid == 0) mbar_arrive(&empty[b]);
  }
}

// --------------------------------------------------------------------------------------
// K1 on compact streams, deep pipeline. When every job of the batch runs on a compact
// model (u8 probability index + u8 reward class) a stage shrinks to ~20 KB:
// rowOffset, trnOffset, succ, index, class, done, own x and the successor window of x.
// That buys kCmpStages = 5 stages per CTA at 2 CTAs per SM, so ~8 stages (~165 KB) are in
// flight per SM -- what Little's law asks for at ~4 us of copy latency -- instead of 3.
// Arithmetic per state as in k_greedy_sweep_tma's single pass: row value =
// classRho[class] + dict[idx_k] * x[succ_k] + ..., left to right, first strict max.

#ifndef MORAP_CMP_STAGES
#define MORAP_CMP_STAGES 3
#endif
#ifndef MORAP_CMP_CTAS
#define MORAP_CMP_CTAS 4
#endif
constexpr int kCmpStages = MORAP_CMP_STAGES;
// stage: u16 tile-relative row ends per state and transition ends per row, u16 window
// offsets, u8 probability index, u8 reward class, done, own x, successor window of x
constexpr int kCOffRow = 0;                               // u32 state word: row end | transition end << 10 | done << 21
constexpr int kCOffTrn = kCOffRow + 4 * (kBlock + 4);     // u32 row word: transition end | class << 11
constexpr int kCOffSucc = kCOffTrn + 4 * (kRowCap + 4);   // u32 transition word: window offset | index << 16
constexpr int kCOffX = kCOffSucc + 4 * (kNnzCap + 4);
constexpr int kCOffXw = kCOffX + 8 * kStXDbls;
constexpr int kCStageBytes = kCOffXw + 8 * (kXWin + 2);
static_assert(kCOffTrn % 16 == 0 && kCOffSucc % 16 == 0 && kCOffX % 16 == 0 &&
                  kCOffXw % 16 == 0 && kCStageBytes % 16 == 0,
              "compact stage regions must be 16-byte aligned");
constexpr int kCFbRows = kXWin + 2 < kRowCap ? kXWin + 2 : kRowCap;  // fallback row values in the window region
constexpr int kCmpSmemBytes = kCmpStages * kCStageBytes;
// MORAP_CMP_CTAS CTAs per SM must fit the 228 KB of shared memory (1 KB reserved per CTA,
// ~2.5 KB of static shared memory): one CTA less costs ~5% (measured)
static_assert(MORAP_CMP_CTAS * (kCmpSmemBytes + 2560 + 1024) <= 228 * 1024, "compact sweep stages too large");

// Arguments of the finalize step fused into the compact sweep (count == nullptr: none).
struct FinArgs {
  unsigned* count;  // CTAs finished in this launch; reset by the last one
  const int32_t* jobModel;
  double eps;
  int cap;
  int32_t* sweeps;
  double* residual;
  int32_t* status;
};

// exclusive scan of (a, b) over the whole block (any multiple of 32 threads <= 1024)
__device__ __forceinline__ void block_scan2n(int& a, int& b, int* sa, int* sb, int& totA, int& totB) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int xa = a, xb = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
    if (lane >= o) {
      xa += ya;
      xb += yb;
    }
  }
  if (lane == 31) {
    sa[wid] = xa;
    sb[wid] = xb;
  }
  __syncthreads();
  if (wid == 0) {
    int va = lane < nw ? sa[lane] : 0, vb = lane < nw ? sb[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ya = __shfl_up_sync(0xffffffffu, va, o), yb = __shfl_up_sync(0xffffffffu, vb, o);
      if (lane >= o) {
        va += ya;
        vb += yb;
      }
    }
    sa[lane] = va;
    sb[lane] = vb;
  }
  __syncthreads();
  const int offA = wid ? sa[wid - 1] : 0, offB = wid ? sb[wid - 1] : 0;
  totA = sa[nw - 1];
  totB = sb[nw - 1];
  a = offA + xa - a;
  b = offB + xb - b;
  __syncthreads();
}

// Per-job stop test after an optimize sweep (numerics.hpp:105-112) and compaction of the
// active list / tile prefix, by one block (k_finalize's body for the optimize kind).
__device__ void finalize_opt(const DevModel* __restrict__ models, const int32_t* __restrict__ jobModel,
                             int32_t* list, int32_t* prefix, Ctl* ctl, unsigned long long* deltaBits, double eps,
                             int cap, int32_t* sweeps, double* residual, int32_t* status) {
  __shared__ int sa[32], sb[32];
  __shared__ unsigned long long sBytes[32], sBk[32];
  const int nact = __ldcg(&ctl->nactive);
  if (nact == 0) return;
  const int k = __ldcg(&ctl->sweepsDone) + 1;  // sweeps completed including the one just run
  int outBase = 0, tileBase = 0;
  unsigned long long bytes = 0, backups = 0;
  for (int base = 0; base < nact; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int keep = 0, nt = 0, job = -1;
    if (i < nact) {
      job = __ldcg(list + i);
      const DevModel& M = models[jobModel[job]];
      const double d = __longlong_as_double(static_cast<long long>(__ldcg(deltaBits + job)));
      deltaBits[job] = 0ull;
      sweeps[job] = k;
      residual[job] = d;
      bytes += M.bytesPerSweep;
      backups += static_cast<unsigned long long>(M.nnz);
      if (d <= eps) status[job] = MORAP_OK;
      else if (k >= cap) status[job] = MORAP_NON_CONVERGENCE;
      else keep = 1;
      if (keep) nt = M.ntiles;
    }
    int pa = keep, pb = nt, ta, tb;
    block_scan2n(pa, pb, sa, sb, ta, tb);
    if (keep) {
      list[outBase + pa] = job;
      prefix[outBase + pa] = tileBase + pb;
    }
    outBase += ta;
    tileBase += tb;
    __syncthreads();
  }
  unsigned long long vb = bytes, vk = backups;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vb += __shfl_xor_sync(0xffffffffu, vb, o);
    vk += __shfl_xor_sync(0xffffffffu, vk, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sBytes[threadIdx.x >> 5] = vb;
    sBk[threadIdx.x >> 5] = vk;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tbytes = 0, tk = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      tbytes += sBytes[w];
      tk += sBk[w];
    }
    prefix[outBase] = tileBase;
    ctl->nactive = outBase;
    ctl->totalTiles = tileBase;
    ctl->sweepsDone = k;
    ctl->nsel = 0;
    ctl->claimed = 0;
    ctl->bytes += tbytes;
    ctl->backups += tk;
  }
}

// Frozen-tile selection (exact work skipping). A tile's new values are a function of x over
// its successor window only (allIn tiles), so when no state of the window and none of the
// tile's own states changed bitwise in the previous sweep, this sweep would reproduce the
// previous values bit for bit -- and the y buffer (two sweeps old) already holds them; the
// tile's residual contribution is exactly 0 and its policy is extracted after convergence
// anyway. Such tiles are left out of the sweep. stamp[g] = the last sweep in which a state
// of group g (32 states) of the job changed (written by the sweep's compute warps; 0 =
// never). Values, residuals, sweep counts and policies are identical to sweeping every tile.
//
// The candidates of an optimize batch -- every tile of every initially active job, with
// the stamp groups it depends on -- are listed once per batch (k_build_cand); per sweep,
// k_select keeps the candidates whose job is still active (alive[job] == sweeps done: the
// finalize stamps every job it keeps, -1 the ones it drops) and whose groups changed in the
// previous sweep, and
// compacts them into `sel` (in order within each block, one atomic per block).
constexpr int kSelThreads = 256;
#ifndef MORAP_TAIL_PCT
#define MORAP_TAIL_PCT 25
#endif
#ifndef MORAP_CLAIM
#define MORAP_CLAIM 2
#endif
constexpr int kTailPct = MORAP_TAIL_PCT;  // share of the selected tiles handed out dynamically
constexpr int kClaim = MORAP_CLAIM;       // tiles per claim

// cand[prefix[slot] + lt] = {job, lt | (n window loads << 20) | (n own loads << 24) | (n out
// groups << 27), first stamp of the successor window, first stamp of the tile's own states}
// as absolute indices into the batch's stamp array; candOut[...] = offset of the tile's
// out-of-window stamps (absolute) in candOutG.
// Window / own groups are rounded down to multiples of 4 (16-byte loads of 4 stamps); the
// two ranges are kept apart because a window can lie far from the tile's own states
// (centralised models). Oversized tiles and tiles with more than kMaxOutGroups
// out-of-window groups are never skipped: window group -1.
constexpr int kCandLtBits = 20;  // tiles per model < 2^20 (skipping is off for larger models)
constexpr int kMaxOutGroups = 16;  // out-of-window stamp groups a skippable tile may depend on
// the packed candidate word holds the window's 16-byte stamp loads in 4 bits, the tile's own
// in 3 and the out-of-window group count in 5: the -D knobs must keep them in range
static_assert((kXWin + 31) / 32 / 4 + 2 <= 15, "successor-window stamp loads overflow 4 bits");
static_assert((kBlock / 32) / 4 + 2 <= 7, "own-state stamp loads overflow 3 bits");
static_assert(kMaxOutGroups < 32 && kCandLtBits + 7 + 5 <= 32, "candidate word layout");
__global__ void __launch_bounds__(kSelThreads) k_build_cand(const DevModel* __restrict__ models,
                                                            const OptJob* __restrict__ jobs,
                                                            const int32_t* __restrict__ list,
                                                            const int32_t* __restrict__ prefix,
                                                            int4* __restrict__ cand, int32_t* __restrict__ candOut,
                                                            int32_t* __restrict__ candOutG, int slotBase) {
  const int slot = slotBase + blockIdx.y;
  const int job = list[slot];
  const int base = prefix[slot], nt = prefix[slot + 1] - base;
  const int lt = blockIdx.x * kSelThreads + threadIdx.x;
  if (lt >= nt) return;
  const OptJob& J = jobs[job];
  const DevModel& M = models[J.model];
  const int4* tp = reinterpret_cast<const int4*>(M.tiles + lt);
  const int4 d0 = tp[0], d1 = tp[1], e0 = tp[2];  // (s0 r0 k0 fits) (wlo wn allIn simple) (next s0 ...)
  int gw = -1, go = 0, oOff = 0;
  unsigned packed = static_cast<unsigned>(lt);
  const int ob = M.outIdx[lt], on = M.outIdx[lt + 1] - ob;
  const bool outOk = on <= kMaxOutGroups && (on == 0 || M.outGrp[ob] >= 0);
  if (d0.w && outOk) {
    gw = d1.y > 0 ? (d1.x >> 5) & ~3 : 0;  // no successors at all: own states only
    const int nw = d1.y > 0 ? (((d1.x + d1.y - 1) >> 5) - gw) / 4 + 1 : 0;  // <= 9 for a 992-state window
    go = (d0.x >> 5) & ~3;
    const int no = (((e0.x - 1) >> 5) - go) / 4 + 1;         // <= 3 for 256 states
    packed |= (static_cast<unsigned>(nw) << kCandLtBits) | (static_cast<unsigned>(no) << (kCandLtBits + 4)) |
              (static_cast<unsigned>(on) << (kCandLtBits + 7));
    gw += J.stampOff;  // absolute stamp indices (multiples of 4)
    go += J.stampOff;
    oOff = J.outBase + ob;
    for (int q = 0; q < on; ++q) candOutG[oOff + q] = J.stampOff + M.outGrp[ob + q];
  }
  cand[base + lt] = make_int4(job, static_cast<int>(packed), gw, go);
  candOut[base + lt] = oOff;
}

// k_select also carries the stop test of the sweep just completed (numerics.hpp:105-112),
// distributed: every candidate thread decides for its own job from that job's residual
// (the same inputs give the same decision in every thread), and the thread of the job's
// first tile records it (sweeps, residual, status, act = 0 once stopped), clears the
// job's residual slot for the coming sweep and counts the job in. Residual slots alternate
// by sweep parity: deltaBits[2 * job + (sweep & 1)]. The sweep kernel then only bumps the
// sweep count (last-CTA ticket) -- no serial finalize between sweeps.
__global__ void __launch_bounds__(kSelThreads) k_select(const DevModel* __restrict__ models,
                                                        const OptJob* __restrict__ jobs, int32_t* act,
                                                        const int4* __restrict__ cand,
                                                        const int32_t* __restrict__ candOut,
                                                        const int32_t* __restrict__ candOutG,
                                                        const int32_t* __restrict__ stampAll, int ncand, Ctl* ctl,
                                                        int2* __restrict__ sel, unsigned long long* deltaBits,
                                                        double eps, int cap, int32_t* sweeps, double* residual,
                                                        int32_t* status) {
  __shared__ unsigned long long sB[kSelThreads / 32], sK[kSelThreads / 32];
  const int k = ctl->sweepsDone;
  if (ctl->nactive == 0) return;
  const int per = ((ncand + gridDim.x - 1) / gridDim.x + kSelThreads - 1) / kSelThreads * kSelThreads;
  const int t0 = blockIdx.x * per, t1 = min(ncand, t0 + per);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long ranBytes = 0, ranNnz = 0;  // jobs that ran sweep k (reference-layout stats)
  for (int base = t0; base < t1; base += kSelThreads) {
    const int t = base + threadIdx.x;
    int keep = 0;
    int4 c = make_int4(0, 0, 0, 0);
    if (t < t1) {
      c = __ldg(cand + t);
      const int oo = __ldg(candOut + t);
      const int job = c.x;
      const bool first = (c.y & ((1 << kCandLtBits) - 1)) == 0;
      bool run = __ldcg(act + job) != 0;
      if (run && k > 0) {  // stop test of sweep k
        const double d = __longlong_as_double(static_cast<long long>(__ldcg(deltaBits + 2 * job + (k & 1))));
        const bool stop = d <= eps || k >= cap;
        if (first) {
          sweeps[job] = k;
          residual[job] = d;
          if (stop) {
            status[job] = d <= eps ? MORAP_OK : MORAP_NON_CONVERGENCE;
            act[job] = 0;
          }
          ranBytes += jobs[job].bytesPerSweep;
          ranNnz += static_cast<unsigned long long>(jobs[job].nnz);
        }
        run = !stop;
      }
      if (run && first) {
        deltaBits[2 * job + ((k + 1) & 1)] = 0ull;
        atomicAdd(&ctl->nactNext, 1);
      }
      if (run) {
        keep = 1;
        if (k > 0 && c.z >= 0) {
          const int4* stamp = reinterpret_cast<const int4*>(stampAll);
          const unsigned u = static_cast<unsigned>(c.y);
          const int nw = (u >> kCandLtBits) & 15, no = (u >> (kCandLtBits + 4)) & 7, nout = u >> (kCandLtBits + 7);
          int m = 0;
          for (int q = 0; q < nout; ++q)  // successors outside the window: their groups one by one
            m = max(m, __ldcg(stampAll + __ldg(candOutG + oo + q)));
          for (int q = 0; q < nw; ++q) {  // successor window
            const int4 v = __ldcg(stamp + (c.z >> 2) + q);
            m = max(m, max(max(v.x, v.y), max(v.z, v.w)));
          }
          for (int q = 0; q < no; ++q) {  // own states
            const int4 v = __ldcg(stamp + (c.w >> 2) + q);
            m = max(m, max(max(v.x, v.y), max(v.z, v.w)));
          }
          keep = m >= k;  // something it depends on changed in the previous sweep
        }
      }
      c.y &= (1 << kCandLtBits) - 1;
    }
    // compaction per warp: one atomic per warp with a kept tile, order kept within the warp
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    int at = 0;
    if (lane == 0 && bal) at = atomicAdd(&ctl->nsel, __popc(bal));
    at = __shfl_sync(0xffffffffu, at, 0);
    if (keep) sel[at + __popc(bal & ((1u << lane) - 1u))] = make_int2(c.x, c.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ranBytes += __shfl_xor_sync(0xffffffffu, ranBytes, o);
    ranNnz += __shfl_xor_sync(0xffffffffu, ranNnz, o);
  }
  if (lane == 0) {
    sB[wid] = ranBytes;
    sK[wid] = ranNnz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tb = 0, tk = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) {
      tb += sB[w];
      tk += sK[w];
    }
    if (tb) atomicAdd(&ctl->bytes, tb);
    if (tk) atomicAdd(&ctl->backups, tk);
  }
}

// Stage record the producer publishes per tile (seven 16-byte words: one vector store each).
struct alignas(16) CmpInfo {
  int t, job, fits, allIn;
  int simple, s0, r0, k0;
  int ns, offX;
  int32_t* stamp;  // frozen-tile stamps of the job (nullptr: no skipping)
  const double* dict;
  const double* classRho;
  const double* x;
  double* y;
  int32_t* policy;
  const DevModel* model;
  const int32_t* succG;  // absolute successors (out-of-window transitions)
  const double* rho;
};

// One tile of a compact optimize sweep (numerics.hpp:84-113), thread per state: the tile's
// streams are staged at `st`; returns |y - x| of this thread's state (0 for done states and
// idle threads). POLICY: record the argmax row instead of writing y. `k` is the sweep being
// run (stamps of changed states become k + 1, frozen-tile skipping).
template <bool POLICY>
__device__ __forceinline__ double cmp_tile(const CmpInfo& v, unsigned char* st, int tid, int k) {
  double dl = 0.0;
  const double* __restrict__ x = v.x;
  if (v.fits && g_dryRun) {
    // diagnostics: stream only
  } else if (v.fits) {
    // Tile-relative u16 row ends per state: state i owns rows [rowE[i-1], rowE[i]) (0 for
    // i = 0). One u32 word per row: transition end (tile-relative, bits 0-10) and reward
    // class (bits 11-31); one u32 word per transition: window offset (low 16 bits, 0xFFFF
    // outside the window) and probability index (bits 16-23) -- one shared-memory load
    // each instead of two (the compute warps are bound by shared-memory wavefronts).
    // Padded per-tile streams: every slice starts at offset 0 of its region.
    // one u32 word per state: row end (bits 0-9), transition end (bits 10-20), done (bit 21)
    const uint32_t* stW = reinterpret_cast<const uint32_t*>(st + kCOffRow);
    const uint32_t* rowW = reinterpret_cast<const uint32_t*>(st + kCOffTrn);
    const uint32_t* trW = reinterpret_cast<const uint32_t*>(st + kCOffSucc);
    const double* xS = reinterpret_cast<const double*>(st + kCOffX) + v.offX;
    const double* xwS = reinterpret_cast<const double*>(st + kCOffXw);  // even wlo: no front offset
    if (tid < v.ns) {
      const int s = v.s0 + tid;
      const uint32_t w0 = tid ? stW[tid - 1] : 0u, w1 = stW[tid];
      const int rb = static_cast<int>(w0 & 0x3FFu), re = static_cast<int>(w1 & 0x3FFu);
      if (w1 >> 21) {  // done state
        if (POLICY) v.policy[s] = v.r0 + rb;  // numerics.hpp:114-115
      } else {
        double best = 0.0;
        int bestRow = -1;
        int kb = static_cast<int>((w0 >> 10) & 0x7FFu);
        const double* __restrict__ dict = v.dict;
        const double* __restrict__ crho = v.classRho;
        auto term = [&](uint32_t w) { return __dmul_rn(__ldg(dict + (w >> 16)), xwS[w & 0xFFFFu]); };
        if (v.allIn && v.simple && re > rb) {
          // every successor in the window, at most two transitions per row: straight-line
          // rows, the first one peeled so the max needs no "no row yet" test
          auto row = [&](int r, int& k) {
            const uint32_t rw = rowW[r];
            const int ke = static_cast<int>(rw & 0x7FFu);
            double acc = __ldg(crho + (rw >> 11));
            if (k < ke) acc = __dadd_rn(acc, term(trW[k]));
            if (k + 1 < ke) acc = __dadd_rn(acc, term(trW[k + 1]));
            k = ke;
            return acc;
          };
          best = row(rb, kb);
          bestRow = rb;
#pragma unroll 1
          for (int r = rb + 1; r < re; ++r) {
            const double acc = row(r, kb);
            if (acc > best) {
              best = acc;
              bestRow = r;
            }
          }
        } else if (v.allIn) {  // every successor inside the staged window: no out-of-window test
#pragma unroll 1
          for (int r = rb; r < re; ++r) {
            const uint32_t rw = rowW[r];
            const int ke = static_cast<int>(rw & 0x7FFu);
            double acc = __ldg(crho + (rw >> 11));
#pragma unroll 1
            for (int q = kb; q < ke; ++q) acc = __dadd_rn(acc, term(trW[q]));
            kb = ke;
            if (bestRow < 0 || acc > best) {
              best = acc;
              bestRow = r;
            }
          }
        } else {
          auto xAt = [&](int q, uint32_t w) {  // window offset staged; absolute successor only outside it
            const unsigned o = w & 0xFFFFu;
            return o != 0xFFFFu ? xwS[o] : __ldg(x + __ldg(v.succG + v.k0 + q));
          };
          for (int r = rb; r < re; ++r) {
            const uint32_t rw = rowW[r];
            const int ke = static_cast<int>(rw & 0x7FFu);
            double acc = __ldg(crho + (rw >> 11));
            for (int q = kb; q < ke; ++q) {
              const uint32_t w = trW[q];
              acc = __dadd_rn(acc, __dmul_rn(__ldg(dict + (w >> 16)), xAt(q, w)));
            }
            kb = ke;
            if (bestRow < 0 || acc > best) {
              best = acc;
              bestRow = r;
            }
          }
        }
        if (POLICY) {
          v.policy[s] = v.r0 + bestRow;
        } else {
          const double xo = xS[tid];
          v.y[s] = best;
          dl = fabs(__dsub_rn(best, xo));
          // bitwise change (not |y - x| > 0: -0.0 and +0.0 differ for the skip invariant)
          if (v.stamp && __double_as_longlong(best) != __double_as_longlong(xo)) v.stamp[s >> 5] = k + 1;
        }
      }
    }
  } else {
    // oversized single-state tile from global memory (stage slot reused as scratch)
    const DevModel& M = *v.model;
    int32_t* sRow = reinterpret_cast<int32_t*>(st + kCOffRow);
    double* sVal = reinterpret_cast<double*>(st + kCOffXw);
    for (int i = tid; i <= v.ns; i += kConsumers) sRow[i] = M.rowOffset[v.s0 + i];
    consumer_sync();
    const int r0 = sRow[0];
    const int nr = sRow[v.ns] - r0;
    const int nstage = min(nr, kCFbRows);
    for (int i = tid; i < nstage; i += kConsumers) sVal[i] = row_value_cmp(M, v.classRho, x, r0 + i);
    consumer_sync();
    if (tid < v.ns) {
      const int s = v.s0 + tid;
      const int rb = sRow[tid] - r0, re = sRow[tid + 1] - r0;
      if (M.done[s]) {
        if (POLICY) v.policy[s] = r0 + rb;
      } else {
        double best = 0.0;
        int bestRow = -1;
        for (int q = rb; q < re; ++q) {
          const double val = q < kCFbRows ? sVal[q] : row_value_cmp(M, v.classRho, x, r0 + q);
          if (bestRow < 0 || val > best) {
            best = val;
            bestRow = q;
          }
        }
        if (POLICY) {
          v.policy[s] = r0 + bestRow;
        } else {
          const double xo = x[s];
          v.y[s] = best;
          dl = fabs(__dsub_rn(best, xo));
          if (v.stamp && __double_as_longlong(best) != __double_as_longlong(xo)) v.stamp[s >> 5] = k + 1;
        }
      }
    }
  }
  return dl;
}

template <bool POLICY>
__global__ void __launch_bounds__(kTmaThreads, MORAP_CMP_CTAS) k_greedy_sweep_cmp(const DevModel* __restrict__ models,
                                                                     const OptJob* __restrict__ jobs,
                                                                     const int32_t* __restrict__ list,
                                                                     const int32_t* __restrict__ prefix,
                                                                     const Ctl* __restrict__ ctl,
                                                                     const int32_t* __restrict__ jobSweeps,
                                                                     unsigned long long* __restrict__ deltaBits,
                                                                     const int2* __restrict__ sel, FinArgs fin) {
  // sel != nullptr: sweep only the (job, tile) pairs k_select kept (frozen-tile skipping);
  // otherwise every tile of every active job (prefix / list)
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kCmpStages], empty[kCmpStages];
  __shared__ CmpInfo info[kCmpStages];
  __shared__ double sRed[kConsumers / 32];
  __shared__ int32_t sPos[32][4];  // producer: TilePos of the current batch of 32 tiles

  const int nact = ctl->nactive;
  const int total = sel ? ctl->nsel : ctl->totalTiles;
  // sel mode: the first (100 - kTailPct)% of the tiles are split evenly over the CTAs, the
  // rest is claimed kClaim tiles at a time by whichever CTAs finish first (tiles differ in
  // work, and a static split alone leaves a ~25% tail)
  const int staticN = sel ? total - static_cast<int>(static_cast<long long>(total) * kTailPct / 100) : total;
  const int per = (staticN + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per;
  const int t1 = min(staticN, t0 + per);
  const int k = ctl->sweepsDone;
  const int tid = threadIdx.x;
  unsigned long long* trace =
      !POLICY && g_ctaTrace ? g_ctaTrace + (static_cast<size_t>(k % kTraceSlots) * gridDim.x + blockIdx.x) * 4 : nullptr;
  if (trace && tid == 0) trace[0] = global_ns();
  if (t0 < t1 || staticN < total) {  // this CTA has tiles (the fused finalize below runs in every CTA)
  if (tid == 0) {
    for (int q = 0; q < kCmpStages; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kConsumers / 32);  // every consumer warp releases a stage on its own
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (tid >= kConsumers) {
    // Producer warp. Tile metadata is resolved 32 tiles at a time (lane l walks the
    // prefix / list / job / model / tile tables for tile tb + l, so the chain of dependent
    // loads is paid once per 32 tiles instead of once per tile), and each lane keeps the
    // base pointer of "its" stream for the current job, reloaded only when the job
    // changes. Per tile: broadcasts, one elected bookkeeping write, lane i issues the
    // bulk copy of stream i.
    const int lane = tid & 31;
    const uint64_t pol = evict_first_policy(), polKeep = evict_last_policy();
    int ai = sel ? 0 : find_slot(prefix, nact + 1, t0);
    int use = 0;
    int curJob = -1;
    const unsigned char* myBase = nullptr;  // stream base of this lane for curJob
    // per-lane stream constants: element size (log2) and stage region
    const int laneSh = lane == 6 || lane == 7 ? 3 : 2;
    const int laneDst = lane == 0 ? kCOffRow : lane == 1 ? kCOffTrn : lane == 2 ? kCOffSucc : lane == 6 ? kCOffX
                      : kCOffXw;
    const DevModel* curM = nullptr;
    const OptJob* curJ = nullptr;
    int parity = k & 1;
    uint32_t exBytes = 0, exNnz = 0;  // sel mode: what this CTA swept (DESIGN.md §4 bytes)
    for (int tb = t0, tEnd = t1;;) {
      if (tb >= tEnd) {  // static range done: claim from the dynamic tail
        if (staticN >= total) break;
        int c = 0;
        if (lane == 0) c = atomicAdd(&const_cast<Ctl*>(ctl)->claimed, kClaim);
        tb = staticN + __shfl_sync(0xffffffffu, c, 0);
        if (tb >= total) break;
        tEnd = min(total, tb + kClaim);
      }
      const int nb = min(32, tEnd - tb);
      // ---- resolve tiles tb .. tb+nb-1, one per lane ---------------------------------
      const int tl = tb + lane;
      int mJob = 0, mS0 = 0, mR0 = 0, mK0 = 0, mFits = 0, mWlo = 0, mWn = 0, mAll = 0, mSimple = 0, eS0 = 0,
          eR0 = 0, eK0 = 0;
      __syncwarp();  // the previous batch is done with sPos
      if (lane < nb) {
        int lt;
        if (sel) {
          const int2 e = sel[tl];
          mJob = e.x;
          lt = e.y;
        } else {
          int a = ai;
          while (tl >= prefix[a + 1]) ++a;
          mJob = list[a];
          lt = tl - prefix[a];
        }
        const DevModel* M = &models[jobs[mJob].model];
        const int4* tp = reinterpret_cast<const int4*>(M->tiles + lt);
        const int4 d0 = tp[0], d1 = tp[1], e0 = tp[2];
        const int4 p0 = *reinterpret_cast<const int4*>(M->tilePos + lt);
        mS0 = d0.x; mR0 = d0.y; mK0 = d0.z; mFits = d0.w;
        mWlo = d1.x; mWn = d1.y; mAll = d1.z; mSimple = d1.w;
        eS0 = e0.x; eR0 = e0.y; eK0 = e0.z;
        sPos[lane][0] = p0.x; sPos[lane][1] = p0.y; sPos[lane][2] = p0.z;
      }
      __syncwarp();
      if (!sel) {  // advance ai to the slot of the last tile of the batch
        const int last = tb + nb - 1;
        while (last >= prefix[ai + 1]) ++ai;
      }
      for (int q = 0; q < nb; ++q, ++use) {
        const int ti = tb + q;
        const int job = __shfl_sync(0xffffffffu, mJob, q);
        const int s0 = __shfl_sync(0xffffffffu, mS0, q), r0 = __shfl_sync(0xffffffffu, mR0, q);
        const int k0 = __shfl_sync(0xffffffffu, mK0, q), fits = __shfl_sync(0xffffffffu, mFits, q);
        const int wlo = __shfl_sync(0xffffffffu, mWlo, q), wn = __shfl_sync(0xffffffffu, mWn, q);
        const int allIn = __shfl_sync(0xffffffffu, mAll, q);
        const int simple = __shfl_sync(0xffffffffu, mSimple, q);
        const int s1 = __shfl_sync(0xffffffffu, eS0, q), r1 = __shfl_sync(0xffffffffu, eR0, q);
        const int k1 = __shfl_sync(0xffffffffu, eK0, q);
        if (sel) {
          exBytes += 4u * (k1 - k0) + 4u * (r1 - r0) + 20u * (s1 - s0);
          exNnz += static_cast<uint32_t>(k1 - k0);
        }
        if (job != curJob) {  // uniform: reload this lane's stream base for the new job
          curJob = job;
          curJ = &jobs[job];
          curM = &models[curJ->model];
          if (POLICY) parity = (jobSweeps[job] - 1) & 1;
          const void* bp = nullptr;
          switch (lane) {
            case 0: bp = curM->stW; break;
            case 1: bp = curM->rowW; break;
            case 2: bp = curM->trW; break;
            case 6: bp = POLICY ? nullptr : curJ->buf[parity]; break;
            case 7: bp = curJ->buf[parity]; break;
            default: break;
          }
          myBase = static_cast<const unsigned char*>(bp);
        }
        const int b = use % kCmpStages;
        // stream of this lane: [lo, hi) in elements of 1 << sh bytes, selected without
        // branching (lanes 0-2: tile-major padded streams, slice start from TilePos;
        // lane 6: own x; lane 7: the successor window)
        const int pos = lane < 3 ? sPos[q][lane] : 0;
        const int len = lane == 0 ? s1 - s0 : (lane == 1 ? r1 - r0 : k1 - k0);
        long long lo = lane < 6 ? pos : (lane == 6 ? s0 : wlo);
        long long hi = lane < 6 ? pos + len : (lane == 6 ? s1 : wlo + wn);
        if (lane > 7 || (lane >= 3 && lane <= 5)) lo = hi = 0;  // lanes 3-5: no stream
        const int sh = laneSh, dstOff = laneDst;
        const uint64_t lp = lane >= 6 ? polKeep : pol;
        const long long a0 = (lo << sh) & ~15ll, z0 = ((hi << sh) + 15) & ~15ll;
        const uint32_t bytes =
            (myBase && fits && z0 > a0) ? static_cast<uint32_t>(z0 - a0) : 0u;
        const int off = static_cast<int>(((lo << sh) - a0) >> sh);
        const uint32_t txBytes = __reduce_add_sync(0xffffffffu, bytes);
        if (use >= kCmpStages) mbar_wait_sleep(&empty[b], ((use / kCmpStages) - 1) & 1);
        // bookkeeping for the consumers: lane i < 8 writes its stream offset, lane 0 the rest
        const int offX = __shfl_sync(0xffffffffu, off, 6);  // own x: front offset of lane 6's copy
        if (lane == 0) {
          CmpInfo rec;
          rec.t = ti;
          rec.job = job;
          rec.fits = fits;
          rec.allIn = allIn;
          rec.simple = simple;
          rec.s0 = s0;
          rec.r0 = r0;
          rec.k0 = k0;
          rec.ns = s1 - s0;
          rec.offX = offX;
          rec.stamp = POLICY ? nullptr : curJ->stamp;
          rec.dict = curM->probDict;
          rec.classRho = curJ->classRho;
          rec.x = curJ->buf[parity];
          rec.y = curJ->buf[parity ^ 1];
          rec.policy = curJ->policy;
          rec.model = curM;
          rec.succG = curM->succ;
          rec.rho = curJ->rho;
          info[b] = rec;
        }
        __syncwarp();
        uint64_t* bar = &full[b];
        if (lane == 0) {
          if (fits) mbar_expect_tx(bar, txBytes);
          else mbar_arrive(bar);
        }
        __syncwarp();
        if (bytes) bulk_g2s(smem + b * kCStageBytes + dstOff, myBase + a0, bytes, bar, lp);
      }
      tb += nb;
    }
    if (sel && lane == 0 && exNnz) {
      atomicAdd(&const_cast<Ctl*>(ctl)->execBytes, static_cast<unsigned long long>(exBytes));
      atomicAdd(&const_cast<Ctl*>(ctl)->execBackups, static_cast<unsigned long long>(exNnz));
    }
    if (lane == 0) {
      const int b = use % kCmpStages;
      if (use >= kCmpStages) mbar_wait_sleep(&empty[b], ((use / kCmpStages) - 1) & 1);
      info[b].t = -1;
      mbar_arrive(&full[b]);
    }
  } else {  // compute warps

  // The residual max is carried per thread across the consecutive tiles of one job and
  // reduced over the CTA only when the job changes (a CTA's tiles are contiguous in the
  // active-tile order, so that is a handful of times per sweep instead of once per tile).
  double runMax = 0.0;
  int runJob = -1;
  const int lane = tid & 31;
  for (int use = 0;; ++use) {
    const int b = use % kCmpStages;
    mbar_wait_sleep(&full[b], (use / kCmpStages) & 1);
    const CmpInfo v = info[b];
    if (trace && use == 0 && tid == 0) trace[1] = global_ns();
    if (v.t < 0) break;
    if (!POLICY && v.job != runJob) {  // uniform over the consumers
      if (runJob >= 0) {
        runMax = consumer_max(runMax, sRed);
        if (tid == 0 && runMax > 0.0)
          atomicMax(deltaBits + (sel ? 2 * runJob + ((k + 1) & 1) : runJob),
                    (unsigned long long)__double_as_longlong(runMax));
      }
      runMax = 0.0;
      runJob = v.job;
    }
    const double dl = cmp_tile<POLICY>(v, smem + b * kCStageBytes, tid, k);
    runMax = fmax(runMax, dl);
    __syncwarp();  // this warp is done with stage b (warps drift apart up to the pipeline depth)
    if (lane == 0) mbar_arrive(&empty[b]);
  }
  if (!POLICY && runJob >= 0) {  // residual of the last job of this CTA's range
    runMax = consumer_max(runMax, sRed);
    if (tid == 0 && runMax > 0.0)
      atomicMax(deltaBits + (sel ? 2 * runJob + ((k + 1) & 1) : runJob),
                (unsigned long long)__double_as_longlong(runMax));
  }
  }  // compute warps
  }  // CTA has tiles
  if (!POLICY && fin.count) {
    // fused k_finalize: the last CTA to finish runs the per-job stop test and rebuilds the
    // active list / tile prefix (every other CTA has read them and published its residuals)
    __shared__ int sLast;
    __syncthreads();
    if (tid == 0) {
      if (trace) trace[2] = global_ns();
      __threadfence();
      sLast = atomicAdd(fin.count, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (sLast) {
      __threadfence();
      if (sel) {  // k_select mode: the stop test runs in the next k_select; count the sweep
        if (tid == 0) {
          Ctl* c = const_cast<Ctl*>(ctl);
          const int ran = c->nactNext;
          if (ran > 0) c->sweepsDone = k + 1;
          c->nactive = ran;
          c->nactNext = 0;
          c->nsel = 0;
          c->claimed = 0;
        }
      } else {
        finalize_opt(models, fin.jobModel, const_cast<int32_t*>(list), const_cast<int32_t*>(prefix),
                     const_cast<Ctl*>(ctl), deltaBits, fin.eps, fin.cap, fin.sweeps, fin.residual, fin.status);
      }
      if (tid == 0) {
        *fin.count = 0u;
        if (trace) trace[3] = global_ns();
      }
    }
  }
}

// --------------------------------------------------------------------------------------
// Policy chain: a fixed deterministic scheduler turns the product into a Markov chain
// with one row per state. Before the evaluate sweeps start, the chosen row of every state
// is copied into a compact CSR (chainOff / chainSucc / chainProb) together with that row's
// reward for each RHS (rhoC_o), so a sweep streams ~70 B per state instead of chasing
// policy -> trnOffset -> succ/prob per state. Three small passes over the tiles of the
// evaluate jobs: count, per-job scan of the tile counts, fill.

__device__ __forceinline__ void block_scan2(int& a, int& b, int* sa, int* sb, int& totA, int& totB);

__device__ __forceinline__ int chosen_nnz(const DevModel& M, const EvalJob& J, int s) {
  if (M.done[s]) return 0;
  const int r = J.policy[s];
  return M.trnOffset[r + 1] - M.trnOffset[r];
}

__device__ __forceinline__ int block_exclusive_scan(int v, int* scratch, int& total) {
  // kBlock threads; scratch >= kBlock / 32 ints
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < kBlock / 32 ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kBlock / 32) scratch[lane] = w;
  }
  __syncthreads();
  total = scratch[kBlock / 32 - 1];
  const int base = wid ? scratch[wid - 1] : 0;
  __syncthreads();
  return base + x - v;
}

__global__ void __launch_bounds__(kBlock) k_chain_count(const DevModel* __restrict__ models,
                                                        const EvalJob* __restrict__ jobs,
                                                        const int32_t* __restrict__ list,
                                                        const int32_t* __restrict__ prefix, int nlist, int total,
                                                        int32_t* __restrict__ tileCount) {
  __shared__ int scratch[kBlock / 32];
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int a = find_slot(prefix, nlist + 1, t);
    const EvalJob& J = jobs[list[a]];
    const DevModel& M = models[J.model];
    const int lt = t - prefix[a];
    const int s0 = M.tileStart[lt], ns = M.tileStart[lt + 1] - s0;
    const int c = threadIdx.x < ns ? chosen_nnz(M, J, s0 + threadIdx.x) : 0;
    int tot;
    block_exclusive_scan(c, scratch, tot);
    if (threadIdx.x == 0) tileCount[t] = tot;
  }
}

// one CTA per job: exclusive scan of its tile counts (in place), chainOff[S] = total
__global__ void __launch_bounds__(1024) k_chain_scan(const DevModel* __restrict__ models,
                                                     const EvalJob* __restrict__ jobs,
                                                     const int32_t* __restrict__ list,
                                                     const int32_t* __restrict__ prefix,
                                                     int32_t* __restrict__ tileCount) {
  __shared__ int sa[32], sb[32];
  const int a = blockIdx.x;
  const int b0 = prefix[a], b1 = prefix[a + 1];
  int carry = 0;
  for (int base = b0; base < b1; base += 1024) {
    const int i = base + threadIdx.x;
    int v = i < b1 ? tileCount[i] : 0, dummy = 0, tot, tot2;
    block_scan2(v, dummy, sa, sb, tot, tot2);
    if (i < b1) tileCount[i] = carry + v;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const EvalJob& J = jobs[list[a]];
    J.chainOff[models[J.model].S] = carry;
  }
}

__global__ void __launch_bounds__(kBlock) k_chain_fill(const DevModel* __restrict__ models,
                                                       const EvalJob* __restrict__ jobs,
                                                       const int32_t* __restrict__ list,
                                                       const int32_t* __restrict__ prefix, int nlist, int total,
                                                       const int32_t* __restrict__ tileBase) {
  __shared__ int scratch[kBlock / 32];
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int a = find_slot(prefix, nlist + 1, t);
    const EvalJob& J = jobs[list[a]];
    const DevModel& M = models[J.model];
    const int lt = t - prefix[a];
    const int s0 = M.tileStart[lt], ns = M.tileStart[lt + 1] - s0;
    const int s = s0 + threadIdx.x;
    const int c = threadIdx.x < ns ? chosen_nnz(M, J, s) : 0;
    int tot;
    const int off = tileBase[t] + block_exclusive_scan(c, scratch, tot);
    if (threadIdx.x < ns) {
      J.chainOff[s] = off;
      if (c > 0) {
        const int r = J.policy[s];
        const int kb = M.trnOffset[r];
        for (int q = 0; q < c; ++q) {
          J.chainSucc[off + q] = M.succ[kb + q];
          J.chainProb[off + q] = model_prob(M, kb + q);
        }
        for (int o = 0; o < J.nrhs; ++o) J.rhoC[o][s] = J.rho[o] ? J.rho[o][r] : model_obj(M, J.objIdx[o], r);
      } else {
        for (int o = 0; o < J.nrhs; ++o) J.rhoC[o][s] = 0.0;
      }
    }
  }
}

// --------------------------------------------------------------------------------------
// K2 (TMA pipeline): fused multi-RHS sweep over the policy chain. Same producer /
// consumer structure as k_greedy_sweep_tma; a stage holds chainOff, the chain's
// succ/prob, done, and rhoC_o / x_o of the tile's states for every still-active RHS.
// y_o(s) = 0 + 1.0 * (rhoC_o[s] + sum_k P_k x_o[succ_k])   (numerics.hpp:145-151)

constexpr int kEvRhs = 4;        // RHS handled by the pipelined kernel (more -> k_eval_sweep)
constexpr int kEvChainCap = 1024;
constexpr int kEvOffInts = kStRowInts;
constexpr int kEvSuccInts = kEvChainCap + 4;
constexpr int kEvProbDbls = kEvChainCap + 2;
constexpr int kEvVecDbls = 258;  // >= kBlock + 1
constexpr int kEvOffOff = 0;
constexpr int kEvOffSucc = kEvOffOff + 4 * kEvOffInts;
constexpr int kEvOffProb = kEvOffSucc + 4 * kEvSuccInts;
constexpr int kEvOffDone = kEvOffProb + 8 * kEvProbDbls;
constexpr int kEvOffRho = kEvOffDone + kStDoneBytes;
constexpr int kEvOffX = kEvOffRho + 8 * kEvVecDbls * kEvRhs;
constexpr int kEvStageBytes = kEvOffX + 8 * kEvVecDbls * kEvRhs;
constexpr int kEvSmemBytes = 2 * kEvStageBytes;
static_assert(kEvOffSucc % 16 == 0 && kEvOffProb % 16 == 0 && kEvOffDone % 16 == 0 && kEvOffRho % 16 == 0 &&
                  kEvOffX % 16 == 0 && kEvStageBytes % 16 == 0,
              "eval stage regions must be 16-byte aligned");

struct EvStageInfo {
  int t, job, fits, mask;
  int s0, ns, c0, nc;
  int offOff, offSucc, offProb, offDone;
  int offRho[kEvRhs], offX[kEvRhs];
  const EvalJob* J;
  const DevModel* model;
  int parity;
};

__global__ void __launch_bounds__(kTmaThreads, 3) k_eval_sweep_tma(const DevModel* __restrict__ models,
                                                                   const EvalJob* __restrict__ jobs,
                                                                   const int32_t* __restrict__ list,
                                                                   const int32_t* __restrict__ prefix,
                                                                   const Ctl* __restrict__ ctl,
                                                                   const uint32_t* __restrict__ rhsMask,
                                                                   unsigned long long* __restrict__ deltaBits) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[2], empty[2];
  __shared__ EvStageInfo info[2];
  __shared__ double sRed[kConsumers / 32];

  const int nact = ctl->nactive;
  const int total = ctl->totalTiles;
  if (total <= 0) return;
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per;
  const int t1 = min(total, t0 + per);
  if (t0 >= t1) return;
  const int parity = ctl->sweepsDone & 1;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], 1);
    mbar_init(&empty[1], 1);
    mbar_fence_init();
  }
  __syncthreads();

  if (tid >= kConsumers) {
    if (tid != kConsumers) return;
    const uint64_t pol = evict_first_policy(), polKeep = evict_last_policy();
    int ai = find_slot(prefix, nact + 1, t0);
    int use = 0;
    auto acquire = [&](int b) {
      if (use >= 2) mbar_wait(&empty[b], ((use >> 1) - 1) & 1);
    };
    auto span = [](long long lo, long long hi, int es) {
      const long long a0 = (lo * es) & ~15ll, z = (hi * es + 15) & ~15ll;
      return static_cast<uint32_t>(z - a0);
    };
    for (int ti = t0; ti < t1; ++ti, ++use) {
      while (ti >= prefix[ai + 1]) ++ai;
      const int job = list[ai];
      const EvalJob& J = jobs[job];
      const DevModel* M = &models[J.model];
      const int lt = ti - prefix[ai];
      const int s0 = M->tileStart[lt], ns = M->tileStart[lt + 1] - s0;
      const int c0 = J.chainOff[s0], c1 = J.chainOff[s0 + ns];
      const int b = use & 1;
      acquire(b);
      EvStageInfo v;
      v.t = ti;
      v.job = job;
      v.mask = static_cast<int>(rhsMask[job]);
      v.s0 = s0;
      v.ns = ns;
      v.c0 = c0;
      v.nc = c1 - c0;
      v.J = &J;
      v.model = M;
      v.parity = parity;
      v.fits = J.nrhs <= kEvRhs && c1 - c0 <= kEvChainCap;
      uint64_t* bar = &full[b];
      if (!v.fits) {
        info[b] = v;
        mbar_arrive(bar);
        continue;
      }
      uint32_t txBytes = span(s0, s0 + ns + 1, 4) + span(c0, c1, 4) + span(c0, c1, 8) + span(s0, s0 + ns, 1);
      for (int o = 0; o < J.nrhs; ++o)
        if (v.mask >> o & 1) txBytes += 2 * span(s0, s0 + ns, 8);
      unsigned char* st = smem + b * kEvStageBytes;
      uint32_t tx = 0;
      v.offOff = stage_range(st + kEvOffOff, J.chainOff, s0, s0 + ns + 1, 4, bar, pol, tx);
      v.offSucc = stage_range(st + kEvOffSucc, J.chainSucc, c0, c1, 4, bar, pol, tx);
      v.offProb = stage_range(st + kEvOffProb, J.chainProb, c0, c1, 8, bar, pol, tx);
      v.offDone = stage_range(st + kEvOffDone, M->done, s0, s0 + ns, 1, bar, pol, tx);
      for (int o = 0; o < kEvRhs; ++o) {
        v.offRho[o] = v.offX[o] = 0;
        if (o < J.nrhs && (v.mask >> o & 1)) {
          v.offRho[o] = stage_range(st + kEvOffRho + o * 8 * kEvVecDbls, J.rhoC[o], s0, s0 + ns, 8, bar, pol, tx);
          v.offX[o] = stage_range(st + kEvOffX + o * 8 * kEvVecDbls, J.buf[o][parity], s0, s0 + ns, 8, bar, polKeep, tx);
        }
      }
      info[b] = v;
      mbar_expect_tx(bar, txBytes);
    }
    const int b = use & 1;
    acquire(b);
    info[b].t = -1;
    mbar_arrive(&full[b]);
    return;
  }

  for (int use = 0;; ++use) {
    const int b = use & 1;
    mbar_wait(&full[b], (use >> 1) & 1);
    const EvStageInfo v = info[b];
    if (v.t < 0) break;
    const EvalJob& J = *v.J;
    const int nrhs = J.nrhs;
    double d[kEvRhs];
#pragma unroll
    for (int o = 0; o < kEvRhs; ++o) d[o] = 0.0;
    if (v.fits) {
      unsigned char* st = smem + b * kEvStageBytes;
      const int32_t* offS = reinterpret_cast<const int32_t*>(st + kEvOffOff) + v.offOff;
      const int32_t* succS = reinterpret_cast<const int32_t*>(st + kEvOffSucc) + v.offSucc;
      const double* probS = reinterpret_cast<const double*>(st + kEvOffProb) + v.offProb;
      const uint8_t* doneS = st + kEvOffDone + v.offDone;
      if (tid < v.ns && !doneS[tid]) {
        const int s = v.s0 + tid;
        const int cb = offS[tid] - v.c0, ce = offS[tid + 1] - v.c0;
#pragma unroll
        for (int o = 0; o < kEvRhs; ++o) {
          if (o >= nrhs || !(v.mask >> o & 1)) continue;
          const double* rhoS = reinterpret_cast<const double*>(st + kEvOffRho + o * 8 * kEvVecDbls) + v.offRho[o];
          const double* xS = reinterpret_cast<const double*>(st + kEvOffX + o * 8 * kEvVecDbls) + v.offX[o];
          const double* __restrict__ x = J.buf[o][v.parity];
          double acc = rhoS[tid];
          for (int q = cb; q < ce; ++q) acc = __dadd_rn(acc, __dmul_rn(probS[q], __ldg(x + succS[q])));
          const double val = __dadd_rn(0.0, __dmul_rn(1.0, acc));
          J.buf[o][v.parity ^ 1][s] = val;
          d[o] = fabs(__dsub_rn(val, xS[tid]));
        }
      }
    } else {
      // chain too long for a stage (or more than kEvRhs RHS): straight from global memory
      const DevModel& M = *v.model;
      if (tid < v.ns) {
        const int s = v.s0 + tid;
        if (!M.done[s]) {
          const int cb = J.chainOff[s], ce = J.chainOff[s + 1];
          for (int o = 0; o < nrhs && o < kEvRhs; ++o) {
            if (!(v.mask >> o & 1)) continue;
            const double* __restrict__ x = J.buf[o][v.parity];
            double acc = J.rhoC[o][s];
            for (int q = cb; q < ce; ++q) acc = __dadd_rn(acc, __dmul_rn(J.chainProb[q], __ldg(x + J.chainSucc[q])));
            const double val = __dadd_rn(0.0, __dmul_rn(1.0, acc));
            J.buf[o][v.parity ^ 1][s] = val;
            d[o] = fabs(__dsub_rn(val, x[s]));
          }
        }
      }
    }
#pragma unroll
    for (int o = 0; o < kEvRhs; ++o) {
      if (o < nrhs && (v.mask >> o & 1)) {  // uniform over the consumers
        const double m = consumer_max(d[o], sRed);
        if (tid == 0 && m > 0.0) atomicMax(deltaBits + v.job * MORAP_MAX_RHS + o, (unsigned long long)__double_as_longlong(m));
      }
    }
    consumer_sync();
    if (tid == 0) mbar_arrive(&empty[b]);
  }
}

// --------------------------------------------------------------------------------------
// K2 (persistent): the whole evaluate batch in ONE cooperative launch. Evaluate batches are
// small (n chains of the assigned pairs, L2-resident), so per-sweep launches, the finalize
// kernel and host polls dominated them. Here every CTA owns a contiguous range of the
// batch's states; after each sweep the CTAs meet at a grid barrier, every CTA reads the
// per-(job, RHS) residuals and takes the same stop decisions (delta <= eps, sweep cap),
// CTA 0 records them. Residual slots rotate over three buffers so clearing one never races
// with the sweep writing another. x is read with ld.global.cg (L2): it was written by other
// SMs in the previous sweep of the same launch.

constexpr int kPersistJobs = 16;   // per-CTA residual accumulators (jobs touched by one CTA)
constexpr int kPersistMaxJobs = 1024;

__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vg = gen;
    const unsigned g = *vg;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vg == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

struct PersistArgs {
  const DevModel* models;
  const EvalJob* jobs;
  const long long* statePrefix;  // njobs + 1
  int njobs;
  double eps;
  int cap;
  uint32_t* mask;                 // per job, RHS still running
  unsigned long long* slots;      // 3 x njobs x MORAP_MAX_RHS residual bits
  int32_t* sweeps;
  double* residual;
  int32_t* status;
  Ctl* ctl;
  unsigned* barCount;
  unsigned* barGen;
  int cacheStates;  // > 0: every CTA keeps its states' chains (<= 2 transitions) in shared memory
};

#ifndef MORAP_PERSIST_THREADS
#define MORAP_PERSIST_THREADS 1024
#endif
#ifndef MORAP_PERSIST_MINB
#define MORAP_PERSIST_MINB (1024 / MORAP_PERSIST_THREADS)  // 64 registers: 1024 threads per SM
#endif
constexpr int kPersistThreads = MORAP_PERSIST_THREADS;
constexpr int kPersistCacheBytes = 200 * 1024;  // shared-memory chain cache per CTA (at most)
// Only reached with <= kEvRhs RHS per job (the policy-chain path), so the per-thread
// residual accumulators are kEvRhs wide; done states carry an empty chain and rhoC = 0,
// so they compute y = 0 + 1.0 * 0 = +0.0, the pinned value, without a branch.
__global__ void __launch_bounds__(kPersistThreads, MORAP_PERSIST_MINB) k_eval_persistent(PersistArgs A) {
  __shared__ uint32_t sMask[kPersistMaxJobs];
  __shared__ unsigned long long sDelta[kPersistJobs * MORAP_MAX_RHS];
  __shared__ int sActive;
  const int tid = threadIdx.x;
  const long long total = A.statePrefix[A.njobs];
  const long long per = (total + gridDim.x - 1) / gridDim.x;
  const long long i0 = static_cast<long long>(blockIdx.x) * per;
  const long long i1 = min(total, i0 + per);
  for (int j = tid; j < A.njobs; j += blockDim.x) sMask[j] = A.mask[j];
  // first job touched by this CTA
  int jBase = 0;
  if (i0 < total) {
    int lo = 0, hi = A.njobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (A.statePrefix[mid] <= i0) lo = mid; else hi = mid - 1;
    }
    jBase = lo;
  }
  // The CTA owns the same states in every sweep: with cacheStates its chains (count,
  // successors, probabilities) are read once into shared memory, so a sweep's dependent
  // chain is one L2 gather of x instead of chainOff -> chainSucc -> x.
  extern __shared__ __align__(16) unsigned char esm[];
  const int C = A.cacheStates;
  uint8_t* sN = esm;
  int32_t* sSucc = reinterpret_cast<int32_t*>(esm + ((C + 15) & ~15));
  double* sProb = reinterpret_cast<double*>(esm + ((C + 15) & ~15) + 8 * static_cast<size_t>(C));
  if (C > 0) {
    int jl = jBase;
    for (long long i = i0 + tid; i < i1; i += blockDim.x) {
      while (i >= A.statePrefix[jl + 1]) ++jl;
      const EvalJob& J = A.jobs[jl];
      const int sl = static_cast<int>(i - A.statePrefix[jl]);
      const int li = static_cast<int>(i - i0);
      const int cbl = __ldg(J.chainOff + sl), nl = __ldg(J.chainOff + sl + 1) - cbl;
      sN[li] = static_cast<uint8_t>(nl);
      sSucc[2 * li] = nl > 0 ? __ldg(J.chainSucc + cbl) : 0;
      sSucc[2 * li + 1] = nl > 1 ? __ldg(J.chainSucc + cbl + 1) : 0;
      sProb[2 * li] = nl > 0 ? __ldg(J.chainProb + cbl) : 0.0;
      sProb[2 * li + 1] = nl > 1 ? __ldg(J.chainProb + cbl + 1) : 0.0;
    }
  }
  __syncthreads();
  unsigned long long bytesAcc = 0, backupsAcc = 0;
  for (int k = 0;; ++k) {
    const int parity = k & 1;
    // diagnostics (morap_cuda_debug_cta_trace): {start, states done, barrier passed, decided}
    unsigned long long* trace = g_ctaTrace ? g_ctaTrace + (static_cast<size_t>(k % kTraceSlots) * gridDim.x + blockIdx.x) * 4
                                           : nullptr;
    if (trace && tid == 0) trace[0] = global_ns();
    unsigned long long* slot = A.slots + static_cast<size_t>(k % 3) * A.njobs * MORAP_MAX_RHS;
    for (int q = tid; q < kPersistJobs * MORAP_MAX_RHS; q += blockDim.x) sDelta[q] = 0ull;
    __syncthreads();
    int j = jBase;
    // per-thread running residual of the current job, flushed when the job changes
    double run[kEvRhs];
#pragma unroll
    for (int o = 0; o < kEvRhs; ++o) run[o] = 0.0;
    int runJob = -1;
    auto flush = [&]() {
      if (runJob < 0) return;
      const int rel = runJob - jBase;
#pragma unroll
      for (int o = 0; o < kEvRhs; ++o) {
        if (run[o] > 0.0) {
          const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(run[o]));
          if (rel < kPersistJobs) atomicMax(&sDelta[rel * MORAP_MAX_RHS + o], bits);
          else atomicMax(&slot[runJob * MORAP_MAX_RHS + o], bits);
        }
        run[o] = 0.0;
      }
    };
    // two states per thread per step, their loads issued together (the chain is
    // chainOff -> chainSucc -> x: three dependent L2 round trips per state)
    const long long bd = blockDim.x;
    for (long long ib = i0 + tid; ib < i1; ib += 2 * bd) {
      int jj[2], sv[2], cb[2], n[2];
      uint32_t mk[2];
      int sc0[2], sc1[2];
      double p0[2], p1[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const long long i = ib + u * bd;
        mk[u] = 0u;
        jj[u] = j;
        sv[u] = 0;
        if (i < i1) {
          while (i >= A.statePrefix[j + 1]) ++j;
          jj[u] = j;
          mk[u] = sMask[j];
          sv[u] = static_cast<int>(i - A.statePrefix[j]);
        }
      }
      if (C > 0) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          cb[u] = 0;
          n[u] = 0;
          sc0[u] = sc1[u] = 0;
          p0[u] = p1[u] = 0.0;
          if (mk[u]) {
            const int li = static_cast<int>(ib + u * bd - i0);
            n[u] = sN[li];
            sc0[u] = sSucc[2 * li];
            sc1[u] = sSucc[2 * li + 1];
            p0[u] = sProb[2 * li];
            p1[u] = sProb[2 * li + 1];
          }
        }
      } else {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        cb[u] = 0;
        n[u] = 0;
        if (mk[u]) {
          const EvalJob& J = A.jobs[jj[u]];
          cb[u] = __ldg(J.chainOff + sv[u]);
          n[u] = __ldg(J.chainOff + sv[u] + 1) - cb[u];
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        sc0[u] = sc1[u] = 0;
        p0[u] = p1[u] = 0.0;
        if (mk[u]) {
          const EvalJob& J = A.jobs[jj[u]];
          if (n[u] > 0) {
            sc0[u] = __ldg(J.chainSucc + cb[u]);
            p0[u] = __ldg(J.chainProb + cb[u]);
          }
          if (n[u] > 1) {
            sc1[u] = __ldg(J.chainSucc + cb[u] + 1);
            p1[u] = __ldg(J.chainProb + cb[u] + 1);
          }
        }
      }
      }  // chains from global memory
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!mk[u]) continue;
        if (jj[u] != runJob) {
          flush();
          runJob = jj[u];
        }
        const EvalJob& J = A.jobs[jj[u]];
        const int st = sv[u];
#pragma unroll
        for (int o = 0; o < kEvRhs; ++o) {
          if (o >= J.nrhs || !(mk[u] >> o & 1u)) continue;
          const double* x = J.buf[o][parity];
          double acc = __ldg(J.rhoC[o] + st);
          const double x0 = n[u] > 0 ? __ldcg(x + sc0[u]) : 0.0;
          const double x1 = n[u] > 1 ? __ldcg(x + sc1[u]) : 0.0;
          const double xs = __ldcg(x + st);
          if (n[u] > 0) acc = __dadd_rn(acc, __dmul_rn(p0[u], x0));
          if (n[u] > 1) acc = __dadd_rn(acc, __dmul_rn(p1[u], x1));
          for (int q = cb[u] + 2; q < cb[u] + n[u]; ++q)
            acc = __dadd_rn(acc, __dmul_rn(__ldg(J.chainProb + q), __ldcg(x + __ldg(J.chainSucc + q))));
          const double v = __dadd_rn(0.0, __dmul_rn(1.0, acc));
          J.buf[o][parity ^ 1][st] = v;
          run[o] = fmax(run[o], fabs(__dsub_rn(v, xs)));
        }
      }
    }
    flush();
    __syncthreads();
    if (trace && tid == 0) trace[1] = global_ns();
    for (int q = tid; q < kPersistJobs * MORAP_MAX_RHS; q += blockDim.x) {
      const int jj = jBase + q / MORAP_MAX_RHS;
      if (sDelta[q] && jj < A.njobs) atomicMax(&slot[jj * MORAP_MAX_RHS + (q % MORAP_MAX_RHS)], sDelta[q]);
    }
    grid_barrier(A.barCount, A.barGen, gridDim.x);
    if (trace && tid == 0) trace[2] = global_ns();
    // every CTA takes the same decisions (numerics.hpp:105-112)
    if (tid == 0) sActive = 0;
    __syncthreads();
    unsigned long long* nextClear = A.slots + static_cast<size_t>((k + 2) % 3) * A.njobs * MORAP_MAX_RHS;
    for (int jj = tid; jj < A.njobs; jj += blockDim.x) {
      uint32_t mk = sMask[jj];
      const EvalJob& J = A.jobs[jj];
      for (int o = 0; o < J.nrhs; ++o) {
        if (!(mk >> o & 1u)) continue;
        const unsigned long long bits = __ldcg(slot + jj * MORAP_MAX_RHS + o);
        const double d = __longlong_as_double(static_cast<long long>(bits));
        int st = -1;
        if (d <= A.eps) st = MORAP_OK;
        else if (k + 1 >= A.cap) st = MORAP_NON_CONVERGENCE;
        if (blockIdx.x == 0) {
          A.sweeps[jj * MORAP_MAX_RHS + o] = k + 1;
          A.residual[jj * MORAP_MAX_RHS + o] = d;
          if (st >= 0) A.status[jj * MORAP_MAX_RHS + o] = st;
          bytesAcc += A.models[J.model].bytesPerEval;
          backupsAcc += static_cast<unsigned long long>(A.models[J.model].S);
        }
        if (st >= 0) mk &= ~(1u << o);
      }
      sMask[jj] = mk;
      if (mk) sActive = 1;  // benign race: every writer stores 1
      if (blockIdx.x == 0)
        for (int o = 0; o < MORAP_MAX_RHS; ++o) nextClear[jj * MORAP_MAX_RHS + o] = 0ull;
    }
    __syncthreads();
    if (trace && tid == 0) trace[3] = global_ns();
    if (!sActive) {
      if (blockIdx.x == 0) {
        if (tid == 0) A.ctl->sweepsDone = k + 1;
        for (int jj = tid; jj < A.njobs; jj += blockDim.x) A.mask[jj] = 0u;
        atomicAdd(&A.ctl->bytes, bytesAcc);
        atomicAdd(&A.ctl->backups, backupsAcc);
      }
      return;
    }
    // the next sweep writes slot (k+1)%3, cleared one round ago; (k+2)%3 is cleared by CTA 0
    // above and is next written two barriers from now
  }
}

#include "eval_interleaved.cuh"

// --------------------------------------------------------------------------------------
// K2: fused multi-RHS fixed-scheduler sweep (numerics.hpp:140-153 with a deterministic
// scheduler): y_o(s) = 0 + 1.0 * (rho_o[r] + sum_k P_k x_o[succ_k]), r = policy[s].
// Each RHS o is skipped once converged (its own stop test), so every RHS reproduces a
// separate evaluateSchedulerOn run exactly.

__global__ void __launch_bounds__(kBlock) k_eval_sweep(const DevModel* __restrict__ models,
                                                       const EvalJob* __restrict__ jobs,
                                                       const int32_t* __restrict__ list,
                                                       const int32_t* __restrict__ prefix,
                                                       const Ctl* __restrict__ ctl,
                                                       const uint32_t* __restrict__ rhsMask,
                                                       unsigned long long* __restrict__ deltaBits) {
  __shared__ double sRed[kBlock / 32];
  const int nact = ctl->nactive;
  const int total = ctl->totalTiles;
  if (total <= 0) return;
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per;
  const int t1 = min(total, t0 + per);
  if (t0 >= t1) return;
  int a = find_slot(prefix, nact + 1, t0);
  const int parity = ctl->sweepsDone & 1;

  for (int t = t0; t < t1; ++t) {
    while (t >= prefix[a + 1]) ++a;
    const int job = list[a];
    const EvalJob& J = jobs[job];
    const DevModel& M = models[J.model];
    const int lt = t - prefix[a];
    const int s0 = M.tileStart[lt];
    const int ns = M.tileStart[lt + 1] - s0;
    const uint32_t mask = rhsMask[job];
    const int nrhs = J.nrhs;

    double d[MORAP_MAX_RHS];
#pragma unroll
    for (int o = 0; o < MORAP_MAX_RHS; ++o) d[o] = 0.0;
    if (threadIdx.x < ns) {
      const int s = s0 + threadIdx.x;
      if (!M.done[s]) {
        const int r = J.policy[s];
        const int kb = M.trnOffset[r], ke = M.trnOffset[r + 1];
        double acc[MORAP_MAX_RHS];
#pragma unroll
        for (int o = 0; o < MORAP_MAX_RHS; ++o)
          if (o < nrhs && (mask >> o & 1u)) acc[o] = J.rho[o][r];
        for (int kk = kb; kk < ke; ++kk) {
          const double p = M.prob[kk];
          const int c = M.succ[kk];
#pragma unroll
          for (int o = 0; o < MORAP_MAX_RHS; ++o)
            if (o < nrhs && (mask >> o & 1u)) acc[o] = __dadd_rn(acc[o], __dmul_rn(p, __ldg(J.buf[o][parity] + c)));
        }
#pragma unroll
        for (int o = 0; o < MORAP_MAX_RHS; ++o)
          if (o < nrhs && (mask >> o & 1u)) {
            const double v = __dadd_rn(0.0, __dmul_rn(1.0, acc[o]));
            J.buf[o][parity ^ 1][s] = v;
            d[o] = fabs(__dsub_rn(v, J.buf[o][parity][s]));
          }
      }
    }
#pragma unroll
    for (int o = 0; o < MORAP_MAX_RHS; ++o) {
      if (o < nrhs && (mask >> o & 1u)) {  // block-uniform condition
        const double m = block_max<kBlock / 32>(d[o], sRed);
        if (threadIdx.x == 0 && m > 0.0)
          atomicMax(deltaBits + job * MORAP_MAX_RHS + o, (unsigned long long)__double_as_longlong(m));
      }
    }
  }
}

// --------------------------------------------------------------------------------------
// Finalize: stop test per job/RHS (numerics.hpp:105-112), then compact the active list
// and rebuild the tile prefix for the next sweep. One CTA; jobs in chunks of 1024.

__device__ __forceinline__ void block_scan2(int& a, int& b, int* sa, int* sb, int& totA, int& totB) {
  // exclusive scan of (a, b) over the block (kFinBlock threads)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int xa = a, xb = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
    if (lane >= o) { xa += ya; xb += yb; }
  }
  if (lane == 31) { sa[wid] = xa; sb[wid] = xb; }
  __syncthreads();
  if (wid == 0) {
    int va = sa[lane], vb = sb[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int ya = __shfl_up_sync(0xffffffffu, va, o), yb = __shfl_up_sync(0xffffffffu, vb, o);
      if (lane >= o) { va += ya; vb += yb; }
    }
    sa[lane] = va;
    sb[lane] = vb;
  }
  __syncthreads();
  const int offA = wid ? sa[wid - 1] : 0, offB = wid ? sb[wid - 1] : 0;
  totA = sa[31];
  totB = sb[31];
  a = offA + xa - a;
  b = offB + xb - b;
  __syncthreads();
}

template <bool EVAL>
__global__ void __launch_bounds__(kFinBlock) k_finalize(const DevModel* __restrict__ models,
                                                        const int32_t* __restrict__ jobModel,
                                                        int32_t* __restrict__ list, int32_t* __restrict__ prefix,
                                                        Ctl* __restrict__ ctl, unsigned long long* __restrict__ deltaBits,
                                                        uint32_t* __restrict__ rhsMask, const int32_t* __restrict__ nrhsOf,
                                                        double eps, int cap, int32_t* __restrict__ sweeps,
                                                        double* __restrict__ residual, int32_t* __restrict__ status) {
  __shared__ int sa[32], sb[32];
  __shared__ unsigned long long sBytes[kFinBlock / 32], sBk[kFinBlock / 32];
  const int nact = ctl->nactive;
  if (nact == 0) return;  // batch already finished: keep the sweep count exact
  const int k = ctl->sweepsDone + 1;  // sweeps completed including the one just run
  int outBase = 0, tileBase = 0;
  unsigned long long bytes = 0, backups = 0;
  for (int base = 0; base < nact; base += kFinBlock) {
    const int i = base + threadIdx.x;
    int keep = 0, nt = 0, job = -1;
    if (i < nact) {
      job = list[i];
      const DevModel& M = models[jobModel[job]];
      if (!EVAL) {
        const double d = __longlong_as_double((long long)deltaBits[job]);
        deltaBits[job] = 0ull;
        sweeps[job] = k;
        residual[job] = d;
        bytes += M.bytesPerSweep;
        backups += (unsigned long long)M.nnz;
        if (d <= eps) status[job] = MORAP_OK;
        else if (k >= cap) status[job] = MORAP_NON_CONVERGENCE;
        else keep = 1;
      } else {
        uint32_t mask = rhsMask[job];
        const int nr = nrhsOf[job];
        for (int o = 0; o < nr; ++o) {
          if (!(mask >> o & 1u)) continue;
          const int slot = job * MORAP_MAX_RHS + o;
          const double d = __longlong_as_double((long long)deltaBits[slot]);
          deltaBits[slot] = 0ull;
          sweeps[slot] = k;
          residual[slot] = d;
          bytes += M.bytesPerEval;
          backups += (unsigned long long)M.S;  // one policy row per state (approx. nnz of chosen rows)
          if (d <= eps) { status[slot] = MORAP_OK; mask &= ~(1u << o); }
          else if (k >= cap) { status[slot] = MORAP_NON_CONVERGENCE; mask &= ~(1u << o); }
        }
        rhsMask[job] = mask;
        keep = mask != 0;
      }
      if (keep) nt = M.ntiles;
    }
    int pa = keep, pb = nt, ta, tb;
    block_scan2(pa, pb, sa, sb, ta, tb);
    if (keep) {
      list[outBase + pa] = job;
      prefix[outBase + pa] = tileBase + pb;
    }
    outBase += ta;
    tileBase += tb;
    __syncthreads();
  }
  // algorithmic-byte accounting for the sweep just run
  unsigned long long vb = bytes, vk = backups;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vb += __shfl_xor_sync(0xffffffffu, vb, o);
    vk += __shfl_xor_sync(0xffffffffu, vk, o);
  }
  if ((threadIdx.x & 31) == 0) { sBytes[threadIdx.x >> 5] = vb; sBk[threadIdx.x >> 5] = vk; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tb = 0, tk = 0;
    for (int w = 0; w < kFinBlock / 32; ++w) { tb += sBytes[w]; tk += sBk[w]; }
    prefix[outBase] = tileBase;
    ctl->nactive = outBase;
    ctl->totalTiles = tileBase;
    ctl->sweepsDone = k;
    ctl->bytes += tb;
    ctl->backups += tk;
  }
}

// --------------------------------------------------------------------------------------
// value at the initial state of every job's final buffer (OptimizeResult::value,
// numerics.hpp:120) gathered into one array -> one D2H copy per batch

__global__ void k_gather_opt(const DevModel* __restrict__ models, const OptJob* __restrict__ jobs, int njobs,
                             const int32_t* __restrict__ sweeps, double* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < njobs; j += gridDim.x * blockDim.x) {
    const int sw = sweeps[j];
    out[j] = sw > 0 ? jobs[j].buf[sw & 1][models[jobs[j].model].initial] : 0.0;
  }
}

__global__ void k_gather_eval(const DevModel* __restrict__ models, const EvalJob* __restrict__ jobs, int njobs,
                              const int32_t* __restrict__ sweeps, double* __restrict__ out) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < njobs * MORAP_MAX_RHS; q += gridDim.x * blockDim.x) {
    const int j = q / MORAP_MAX_RHS, o = q % MORAP_MAX_RHS;
    const int sw = sweeps[q];
    out[q] = (o < jobs[j].nrhs && sw > 0) ? jobs[j].buf[o][sw & 1][models[jobs[j].model].initial] : 0.0;
  }
}

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
  int sweepBlocks = 0;  // persistent grid of the greedy sweep kernel
  int evalBlocks = 0;   // persistent grid of the evaluate sweep kernel
  int tmaBlocks = 0;    // persistent grid of the TMA-pipelined sweep kernel
  int evalTmaBlocks = 0;
  bool useTma = true;
  bool evalTma = false;  // current evaluate batch runs the pipelined chain kernel
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;           // policy prefetch copies (overlap the evaluate sweeps)
  cudaEvent_t polReady = nullptr, polCopied = nullptr;
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
  double* dGather = nullptr;
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
  bool timeSweepOnly = std::getenv("MORAP_TIME_SELECT") == nullptr;
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
  unsigned* dBar = nullptr;   // grid-barrier counter + generation
  unsigned* dFinCount = nullptr;  // CTAs done in the current compact sweep (fused finalize)
  void* persistArena = nullptr;
  size_t persistArenaBytes = 0;
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
  CK(cudaMalloc(&ctx->dGather, cap * MORAP_MAX_RHS * sizeof(double)));
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

// Tile table: consecutive states, <= kBlock states and <= kRowCap rows (a state with
// more rows than kRowCap gets a tile of its own; its overflow rows are computed from
// global memory in phase 2).
// The x window staged with a tile: the kXWin consecutive states covering the most of the
// tile's transitions (two pointers over the sorted successors). On warehouse products
// successors of a 256-state tile sit within ~1000 states of each other (BFS numbering),
// so >99% of the gathers are served from shared memory; the rest read global memory.
void successor_window(const morap_csr_view& v, int k0, int k1, int32_t& wlo, int32_t& wn) {
  wn = std::min(kXWin, v.num_states);
  if (k1 <= k0) {
    wlo = 0;
    wn = 0;
    return;
  }
  // histogram of successors in 64-state bins over [min, max], then the best run of
  // (kXWin / 64 - 1) bins -- O(transitions) per tile, within one bin of the optimum
  int lo = v.succ[k0], hi = lo;
  for (int k = k0 + 1; k < k1; ++k) {
    lo = std::min(lo, v.succ[k]);
    hi = std::max(hi, v.succ[k]);
  }
  // windows start at an even state, so the 16-byte aligned window copy lands at offset 0
  if (hi - lo < wn) {  // the whole successor range fits: stage just that range
    wlo = lo & ~1;
    wn = hi - wlo + 1;
    return;
  }
  constexpr int kBin = 64;
  const int nb = (hi - lo) / kBin + 1;
  std::vector<int> h(static_cast<size_t>(nb), 0);
  for (int k = k0; k < k1; ++k) ++h[(v.succ[k] - lo) / kBin];
  const int span = std::max(1, wn / kBin - 1);
  int run = 0, best = -1, bestBin = 0;
  for (int i = 0; i < nb; ++i) {
    run += h[i];
    if (i >= span) run -= h[i - span];
    if (run > best) {
      best = run;
      bestBin = std::max(0, i - span + 1);
    }
  }
  wlo = std::max(0, std::min(lo + bestBin * kBin, v.num_states - wn)) & ~1;
}

void make_tiles(const morap_csr_view& v, std::vector<int32_t>& out, std::vector<TileDesc>& desc) {
  const int32_t* ro = v.row_offset;
  const int32_t* to = v.trn_offset;
  out.clear();
  desc.clear();
  int s = 0;
  out.push_back(0);
  while (s < v.num_states) {
    int e = s + 1;
    while (e < v.num_states && e - s < kBlock && ro[e + 1] - ro[s] <= kRowCap && to[ro[e + 1]] - to[ro[s]] <= kNnzCap)
      ++e;
    const int rows = ro[e] - ro[s], nz = to[ro[e]] - to[ro[s]];
    TileDesc td{s, ro[s], to[ro[s]], rows <= kRowCap && nz <= kNnzCap ? 1 : 0, 0, 0, 0, 0};
    successor_window(v, to[ro[s]], to[ro[e]], td.wlo, td.wn);
    desc.push_back(td);
    out.push_back(e);
    s = e;
  }
  desc.push_back(TileDesc{v.num_states, v.num_rows, v.nnz, 0, 0, 0, 0, 0});
}

// Compact stream of one model: u8 index into a dictionary of the distinct transition
// probabilities and u8 class of each row's objective tuple. Keys are the exact fp64 bit
// patterns, so the device reads back the very same values. ok = false when either
// alphabet exceeds 256 entries (the model then streams the plain fp64 arrays).
struct CompactStream {
  bool ok = false;
  std::vector<uint8_t> idx;    // per transition: probability index (<= 256 distinct)
  std::vector<uint16_t> cls;   // per row: reward class (<= kMaxClasses distinct tuples)
  std::vector<double> dict, table;
  size_t nStW = 0, nRowW = 0, nTrW = 0;        // packed state / row / transition words, padded per tile
                                               // (written straight into the upload staging: fill_streams)
  std::vector<TilePos> pos;
  std::vector<int32_t> outIdx, outGrp;        // out-of-window stamp groups per tile (DevModel)
};

// The sweep streams of a compact model, tile-major: each tile's slice of every stream
// starts on a 16-byte boundary (padded), so one bulk copy per stream lands at offset 0 of
// its stage region. u16 window offsets succW = succ - wlo inside the tile's x window
// (0xFFFF outside), u16 ends relative to the tile, allIn / simple flags per tile.
// layout_streams: slice positions, stream sizes, the per-tile flags and out-of-window
// stamp groups; fill_streams (at packing time) writes the words into the staging buffer.
void layout_streams(const morap_csr_view& v, std::vector<TileDesc>& desc, CompactStream& c) {
  const size_t nt = desc.size() - 1;
  c.pos.assign(nt, TilePos{});
  auto up16 = [](size_t n, size_t es) { return (n * es + 15) / 16 * 16 / es; };  // elements, padded
  size_t nRow = 0, nTrn = 0, nSucc = 0;
  for (size_t t = 0; t < nt; ++t) {
    const TileDesc &d = desc[t], &e = desc[t + 1];
    const bool f = d.fits != 0;  // oversized tiles are swept from the global arrays
    const size_t ns = f ? e.s0 - d.s0 : 0, nr = f ? e.r0 - d.r0 : 0, nz = f ? e.k0 - d.k0 : 0;
    TilePos& p = c.pos[t];
    p.row = static_cast<int32_t>(nRow);
    p.trn = static_cast<int32_t>(nTrn);
    p.succ = static_cast<int32_t>(nSucc);
    nRow += up16(ns, 4);
    nTrn += up16(nr, 4);
    nSucc += up16(nz, 4);
  }
  c.nStW = nRow;
  c.nRowW = nTrn;
  c.nTrW = nSucc;
  c.outIdx.assign(nt + 1, 0);
  c.outGrp.clear();
  for (size_t t = 0; t < nt; ++t) {
    TileDesc& d = desc[t];
    const TileDesc& e = desc[t + 1];
    int simple = 1;
    for (int r = d.r0; r < e.r0; ++r) simple &= v.trn_offset[r + 1] - v.trn_offset[r] <= 2 ? 1 : 0;
    d.simple = simple;
    if (!d.fits) {
      d.allIn = 0;
      c.outGrp.push_back(-1);  // swept from the global arrays: never skipped
      c.outIdx[t + 1] = static_cast<int32_t>(c.outGrp.size());
      continue;
    }
    int allIn = 1;
    for (int k = d.k0; k < e.k0; ++k) allIn &= static_cast<unsigned>(v.succ[k] - d.wlo) < static_cast<unsigned>(d.wn);
    d.allIn = allIn;
    if (!allIn) {  // stamp groups of the out-of-window successors (sorted, distinct, <= kMaxOutGroups)
      const size_t at = c.outGrp.size();
      for (int k = d.k0; k < e.k0; ++k)
        if (static_cast<unsigned>(v.succ[k] - d.wlo) >= static_cast<unsigned>(d.wn)) c.outGrp.push_back(v.succ[k] >> 5);
      std::sort(c.outGrp.begin() + at, c.outGrp.end());
      c.outGrp.erase(std::unique(c.outGrp.begin() + at, c.outGrp.end()), c.outGrp.end());
      if (c.outGrp.size() - at > static_cast<size_t>(kMaxOutGroups)) {
        c.outGrp.resize(at);
        c.outGrp.push_back(-1);
      }
    }
    c.outIdx[t + 1] = static_cast<int32_t>(c.outGrp.size());
  }
}

void fill_streams(const morap_csr_view& v, const std::vector<TileDesc>& desc, const CompactStream& c, uint32_t* stW,
                  uint32_t* rowW, uint32_t* trW) {
  const size_t nt = desc.size() - 1;
  for (size_t t = 0; t < nt; ++t) {
    const TileDesc &d = desc[t], &e = desc[t + 1];
    const TilePos& p = c.pos[t];
    const size_t endRow = t + 1 < nt ? static_cast<size_t>(c.pos[t + 1].row) : c.nStW;
    const size_t endTrn = t + 1 < nt ? static_cast<size_t>(c.pos[t + 1].trn) : c.nRowW;
    const size_t endSucc = t + 1 < nt ? static_cast<size_t>(c.pos[t + 1].succ) : c.nTrW;
    size_t a = p.row, b = p.trn, z = p.succ;
    if (d.fits) {
      for (int q = d.s0; q < e.s0; ++q)  // fitting tiles: row end <= 768 (10 bits), transition end <= 1024 (11)
        stW[a++] = static_cast<uint32_t>(v.row_offset[q + 1] - d.r0) |
                   (static_cast<uint32_t>(v.trn_offset[v.row_offset[q + 1]] - d.k0) << 10) | (v.done[q] ? 1u << 21 : 0u);
      for (int r = d.r0; r < e.r0; ++r)
        rowW[b++] = static_cast<uint32_t>(v.trn_offset[r + 1] - d.k0) | (static_cast<uint32_t>(c.cls[r]) << 11);
      for (int k = d.k0; k < e.k0; ++k) {
        const unsigned o = static_cast<unsigned>(v.succ[k] - d.wlo);
        trW[z++] = (o < static_cast<unsigned>(d.wn) ? o : 0xFFFFu) | (static_cast<uint32_t>(c.idx[k]) << 16);
      }
    }
    for (; a < endRow; ++a) stW[a] = 0u;  // padding (never read)
    for (; b < endTrn; ++b) rowW[b] = 0u;
    for (; z < endSucc; ++z) trW[z] = 0xFFFFu;
  }
}

// Open-addressing table of up to `cap` keys of up to 8 words for build_compact (grows by
// doubling; ids in insertion order).
constexpr int kMaxClasses = 65535;  // reward tuples of a compact model (u16 class index)
struct SmallIds {
  int words = 1, count = 0, cap = 256, slots = 1024;
  std::vector<uint64_t> keys;
  std::vector<int32_t> ids;
  SmallIds(int w, int maxKeys) : words(w), cap(maxKeys), keys(static_cast<size_t>(slots) * w), ids(slots, -1) {}
  int slotOf(const uint64_t* k) const {
    // FNV over whole words, then the TOP bits: the low product bits only see the low key
    // bits, which are all zero for short-mantissa doubles (-1, 0.125, ...)
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < words; ++i) h = (h ^ k[i]) * 1099511628211ull;
    h ^= h >> 29;
    h *= 0xbf58476d1ce4e5b9ull;
    h ^= h >> 32;
    return static_cast<int>(h & static_cast<uint64_t>(slots - 1));
  }
  void grow() {
    std::vector<uint64_t> ok = std::move(keys);
    std::vector<int32_t> oi = std::move(ids);
    const int old = slots;
    slots *= 2;
    keys.assign(static_cast<size_t>(slots) * words, 0);
    ids.assign(slots, -1);
    for (int q = 0; q < old; ++q) {
      if (oi[q] < 0) continue;
      int at = slotOf(&ok[static_cast<size_t>(q) * words]);
      while (ids[at] >= 0) at = (at + 1) & (slots - 1);
      std::memcpy(&keys[static_cast<size_t>(at) * words], &ok[static_cast<size_t>(q) * words], 8ull * words);
      ids[at] = oi[q];
    }
  }
  // id of `k` (inserted if new); -1 when more than `cap` keys would be needed
  int find(const uint64_t* k) {
    for (int slot = slotOf(k);; slot = (slot + 1) & (slots - 1)) {
      if (ids[slot] < 0) {
        if (count == cap) return -1;
        if (2 * (count + 1) > slots) {  // keep the load factor <= 1/2
          grow();
          return find(k);
        }
        std::memcpy(&keys[static_cast<size_t>(slot) * words], k, 8ull * words);
        ids[slot] = count;
        return count++;
      }
      if (std::memcmp(&keys[static_cast<size_t>(slot) * words], k, 8ull * words) == 0) return ids[slot];
    }
  }
};

void build_compact(const morap_csr_view& v, CompactStream& c) {
  c = CompactStream{};
  const int K = v.num_objectives;
  if (K < 1) return;
  c.idx.resize(static_cast<size_t>(v.nnz));
  SmallIds probs(1, 256);
  // the first few distinct values are matched by an unrolled compare against a sentinel-padded
  // list (warehouse products have three probabilities; ~0 is a NaN payload, never a valid
  // probability's bits), so the common case has no data-dependent branch; the rest go
  // through the hash table
  constexpr int kScan = 8;
  uint64_t seen[kScan];
  for (int q = 0; q < kScan; ++q) seen[q] = ~0ull;
  int nseen = 0;
  auto scalarProb = [&](int k) {  // false: more than 256 distinct probabilities
    uint64_t b;
    std::memcpy(&b, &v.prob[k], 8);
    int id = -1;
#pragma unroll
    for (int q = 0; q < kScan; ++q) id = seen[q] == b ? q : id;
    if (id < 0) {
      id = probs.find(&b);
      if (id < 0) return false;
      if (id == static_cast<int>(c.dict.size())) {
        c.dict.push_back(v.prob[k]);
        if (nseen < kScan && id == nseen) seen[nseen++] = b;
      }
    }
    c.idx[k] = static_cast<uint8_t>(id);
    return true;
  };
  // AVX2: four probabilities per step against the known values (lane id = position + 1, 0 =
  // unknown); a step with an unknown value goes through the scalar path, which learns it
  int k = 0;
  while (k < v.nnz && nseen == 0)
    if (!scalarProb(k++)) return;
  for (int known = 0; k + 4 <= v.nnz;) {
    __m256i sv[kScan], iv[kScan];
    known = nseen;
    for (int q = 0; q < known; ++q) {
      sv[q] = _mm256_set1_epi64x(static_cast<long long>(seen[q]));
      iv[q] = _mm256_set1_epi64x(q + 1);
    }
    for (; k + 4 <= v.nnz; k += 4) {
      const __m256i x = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(v.prob + k));
      __m256i id = _mm256_setzero_si256();
      for (int q = 0; q < known; ++q) id = _mm256_or_si256(id, _mm256_and_si256(_mm256_cmpeq_epi64(x, sv[q]), iv[q]));
      if (_mm256_movemask_pd(_mm256_castsi256_pd(_mm256_cmpeq_epi64(id, _mm256_setzero_si256())))) break;
      alignas(32) uint64_t t[4];
      _mm256_store_si256(reinterpret_cast<__m256i*>(t), id);
      const uint32_t w = static_cast<uint32_t>(t[0] - 1) | static_cast<uint32_t>(t[1] - 1) << 8 |
                         static_cast<uint32_t>(t[2] - 1) << 16 | static_cast<uint32_t>(t[3] - 1) << 24;
      std::memcpy(&c.idx[k], &w, 4);
    }
    if (k + 4 > v.nnz) break;
    for (int e = k + 4; k < e; ++k)  // a step with an unknown value: scalar (learns it)
      if (!scalarProb(k)) return;
  }
  for (; k < v.nnz; ++k)
    if (!scalarProb(k)) return;
  c.cls.resize(static_cast<size_t>(v.num_rows));
  SmallIds classes(K, kMaxClasses);
  uint64_t key[MORAP_MAX_OBJECTIVES];
  uint64_t prev[MORAP_MAX_OBJECTIVES];
  int prevId = -1;
  int r0 = 0;
  if (K == 2) {
    // the common two-objective case: unrolled compare against up to kScan known tuples
    // (sentinel-padded: ~0 is a NaN payload, never a reward's bits), no data-dependent branch
    uint64_t ta[kScan], tb[kScan];
    for (int q = 0; q < kScan; ++q) ta[q] = tb[q] = ~0ull;
    int nt = 0;
    // AVX2 steps of four rows once a tuple is known (a step with an unknown tuple drops to
    // the scalar loop below for one step, which learns it)
    for (;;) {
      if (nt > 0) {
        __m256i va[kScan], vb[kScan], iv[kScan];
        for (int q = 0; q < nt; ++q) {
          va[q] = _mm256_set1_epi64x(static_cast<long long>(ta[q]));
          vb[q] = _mm256_set1_epi64x(static_cast<long long>(tb[q]));
          iv[q] = _mm256_set1_epi64x(q + 1);
        }
        for (; r0 + 4 <= v.num_rows; r0 += 4) {
          const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(v.rewards[0] + r0));
          const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(v.rewards[1] + r0));
          __m256i id = _mm256_setzero_si256();
          for (int q = 0; q < nt; ++q)
            id = _mm256_or_si256(id, _mm256_and_si256(_mm256_and_si256(_mm256_cmpeq_epi64(a, va[q]),
                                                                        _mm256_cmpeq_epi64(b, vb[q])), iv[q]));
          if (_mm256_movemask_pd(_mm256_castsi256_pd(_mm256_cmpeq_epi64(id, _mm256_setzero_si256())))) break;
          alignas(32) uint64_t t[4];
          _mm256_store_si256(reinterpret_cast<__m256i*>(t), id);
          const uint64_t w = (t[0] - 1) | (t[1] - 1) << 16 | (t[2] - 1) << 32 | (t[3] - 1) << 48;
          std::memcpy(&c.cls[r0], &w, 8);
        }
      }
      if (r0 >= v.num_rows) break;
      const int stepEnd = std::min(v.num_rows, r0 + 4);  // scalar: this step (or the tail)
      bool more = false;
      for (; r0 < stepEnd; ++r0) {
        uint64_t a, b;
        std::memcpy(&a, &v.rewards[0][r0], 8);
        std::memcpy(&b, &v.rewards[1][r0], 8);
        int id = -1;
#pragma unroll
        for (int q = 0; q < kScan; ++q) id = (ta[q] == a) & (tb[q] == b) ? q : id;
        if (id < 0) {
          if (nt == kScan) {
            more = true;  // more tuples: finish in the general loop below
            break;
          }
          key[0] = a;
          key[1] = b;
          id = classes.find(key);
          if (id < 0) return;
          c.table.push_back(v.rewards[0][r0]);
          c.table.push_back(v.rewards[1][r0]);
          ta[nt] = a;
          tb[nt] = b;
          ++nt;
        }
        c.cls[r0] = static_cast<uint16_t>(id);
      }
      if (more || r0 >= v.num_rows) break;
    }
  }
  for (int r = r0; r < v.num_rows; ++r) {
    bool same = prevId >= 0;
    for (int o = 0; o < K; ++o) {
      std::memcpy(&key[o], &v.rewards[o][r], 8);
      same = same && key[o] == prev[o];
    }
    if (same) {  // runs of equal rows
      c.cls[r] = static_cast<uint16_t>(prevId);
      continue;
    }
    int id = -1;
    const int ncls = static_cast<int>(c.table.size()) / K;
    for (int q = 0; q < ncls && q < kScan && id < 0; ++q) {  // small alphabets: linear scan of the table
      bool eq = true;
      for (int o = 0; o < K && eq; ++o) {
        uint64_t tb;
        std::memcpy(&tb, &c.table[static_cast<size_t>(q) * K + o], 8);
        eq = tb == key[o];
      }
      if (eq) id = q;
    }
    if (id < 0) id = classes.find(key);
    if (id < 0) return;
    for (int o = 0; o < K; ++o) prev[o] = key[o];
    prevId = id;
    if (id == static_cast<int>(c.table.size()) / K)
      for (int o = 0; o < K; ++o) c.table.push_back(v.rewards[o][r]);
    c.cls[r] = static_cast<uint16_t>(id);
  }
  if (c.table.empty()) c.table.assign(static_cast<size_t>(K), 0.0);
  c.ok = true;
}

template <class F>
void parallel_for(int n, F&& fn) {
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int T = std::min(n, hw);
  if (T <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&] {
      for (int i; (i = next.fetch_add(1)) < n;) fn(i);
    });
  for (auto& th : pool) th.join();
}

int validate_view(morap_ctx* ctx, const morap_csr_view& v, int idx) {
  auto bad = [&](const std::string& why) {
    return ctx->fail(MORAP_INVALID_MODEL, "model " + std::to_string(idx) + ": " + why);
  };
  if (v.num_states <= 0) return bad("model has no states");
  if (v.num_rows < 0 || v.nnz < 0) return bad("negative sizes");
  if (v.initial < 0 || v.initial >= v.num_states) return bad("initial state out of range");
  if (v.num_objectives < 0 || v.num_objectives > MORAP_MAX_OBJECTIVES) return bad("too many objectives");
  if (!v.row_offset || !v.trn_offset || !v.done || (v.nnz && (!v.succ || !v.prob))) return bad("null array");
  if (v.row_offset[0] != 0 || v.row_offset[v.num_states] != v.num_rows) return bad("rowOffset does not span the rows");
  // branch-free reductions (vectorised), the message picked afterwards
  int ok = 1;
  for (int s = 0; s < v.num_states; ++s) ok &= v.row_offset[s + 1] >= v.row_offset[s] ? 1 : 0;
  if (!ok) return bad("rowOffset not monotone");
  if (v.trn_offset[0] != 0 || v.trn_offset[v.num_rows] != v.nnz) return bad("trnOffset does not span nnz");
  for (int r = 0; r < v.num_rows; ++r) ok &= v.trn_offset[r + 1] >= v.trn_offset[r] ? 1 : 0;
  if (!ok) return bad("trnOffset not monotone");
  const unsigned S = static_cast<unsigned>(v.num_states);
  for (int k = 0; k < v.nnz; ++k) ok &= static_cast<unsigned>(v.succ[k]) < S ? 1 : 0;
  if (!ok) return bad("successor out of range");
  for (int o = 0; o < v.num_objectives; ++o)
    if (!v.rewards || !v.rewards[o]) return bad("null reward vector");
  return MORAP_OK;
}

int upload_models_table(morap_ctx* ctx) {
  if (ctx->dm.size() > ctx->dModelsCap) {
    cudaFree(ctx->dModels);
    size_t cap = std::max<size_t>(ctx->dm.size() * 2, 16);
    CK(cudaMalloc(&ctx->dModels, cap * sizeof(DevModel)));
    ctx->dModelsCap = cap;
  }
  CK(cudaMemcpyAsync(ctx->dModels, ctx->dm.data(), ctx->dm.size() * sizeof(DevModel), cudaMemcpyHostToDevice,
                     ctx->stream));
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
    } else if (kind == 0 && ctx->useTma) {
      k_greedy_sweep_tma<false><<<ctx->tmaBlocks, kTmaThreads, kTmaSmemBytes, ctx->stream>>>(
          ctx->dModels, ctx->dOptJobs, ctx->dList, ctx->dPrefix, ctx->dCtl, nullptr, ctx->dDelta);
    } else if (kind == 0) {
      k_greedy_sweep<false><<<ctx->sweepBlocks, kBlock, 0, ctx->stream>>>(ctx->dModels, ctx->dOptJobs, ctx->dList,
                                                                          ctx->dPrefix, ctx->dCtl, nullptr, ctx->dDelta);
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
  if (!active.empty()) CK(cudaMemcpyAsync(ctx->dList, active.data(), active.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->dPrefix, prefix.data(), prefix.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->dJobModel, jobModel.data(), jobModel.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
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
  CK(cudaMemcpyAsync(ctx->dOptJobs, ctx->hOptJobs.data(), njobs * sizeof(OptJob), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->dStatus, statusInit.data(), njobs * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->dSweeps, zeroI.data(), njobs * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(ctx->dDelta, 0, 2 * njobs * sizeof(unsigned long long), ctx->stream));  // two parities
  CK(cudaMemsetAsync(ctx->dResidual, 0, njobs * sizeof(double), ctx->stream));
  if ((rc = init_ctl(ctx, active, ctx->optModel))) return rc;
  if (ctx->optSkip && !active.empty()) {
    std::vector<int32_t> alive(njobs, 0);  // act: 1 while the job iterates
    for (int j : active) alive[j] = 1;
    CK(cudaMemcpyAsync(ctx->dAlive, alive.data(), njobs * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));  // `alive` is a local
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

  // results: one gather kernel + one copy per array, one synchronisation
  ctx->optSweeps.assign(njobs, 0);
  ctx->optStatus.assign(njobs, 0);
  std::vector<double> resid(njobs), vals(njobs);
  k_gather_opt<<<(njobs + 255) / 256, 256, 0, ctx->stream>>>(ctx->dModels, ctx->dOptJobs, njobs, ctx->dSweeps,
                                                             ctx->dGather);
  CK(cudaGetLastError());
  CK(d2h(ctx, ctx->optSweeps.data(), ctx->dSweeps, njobs * 4));
  CK(d2h(ctx, ctx->optStatus.data(), ctx->dStatus, njobs * 4));
  CK(d2h(ctx, resid.data(), ctx->dResidual, njobs * 8));
  CK(d2h(ctx, vals.data(), ctx->dGather, njobs * 8));
  CK(d2h(ctx, ctx->hCtl, ctx->dCtl, sizeof(Ctl)));
  CK(cudaStreamSynchronize(ctx->stream));
  double backups = 0;
  for (int j = 0; j < njobs; ++j) {
    value_out[j] = vals[j];
    if (sweeps_out) sweeps_out[j] = ctx->optSweeps[j];
    if (residual_out) residual_out[j] = resid[j];
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
  std::vector<int32_t> jobs;
  for (int j : jobsIn)
    if (!ctx->optPolicyReady[j] && ctx->optSweeps[j] > 0) jobs.push_back(j);
  if (jobs.empty()) return MORAP_OK;
  int rc;
  if ((rc = init_ctl(ctx, jobs, ctx->optModel))) return rc;
  CK(cudaMemcpyAsync(ctx->dSweeps, ctx->optSweeps.data(), ctx->optSweeps.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->useTma && ctx->optCompact)
    k_greedy_sweep_cmp<true><<<ctx->cmpBlocks, kTmaThreads, kCmpSmemBytes, ctx->stream>>>(
        ctx->dModels, ctx->dOptJobs, ctx->dList, ctx->dPrefix, ctx->dCtl, ctx->dSweeps, nullptr, nullptr, FinArgs{});
  else if (ctx->useTma)
    k_greedy_sweep_tma<true><<<ctx->tmaBlocks, kTmaThreads, kTmaSmemBytes, ctx->stream>>>(
        ctx->dModels, ctx->dOptJobs, ctx->dList, ctx->dPrefix, ctx->dCtl, ctx->dSweeps, nullptr);
  else
    k_greedy_sweep<true><<<ctx->sweepBlocks, kBlock, 0, ctx->stream>>>(ctx->dModels, ctx->dOptJobs, ctx->dList,
                                                                       ctx->dPrefix, ctx->dCtl, ctx->dSweeps, nullptr);
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
  CK(cudaMemcpyAsync(dPrefix, prefix.data(), 8ull * (njobs + 1), cudaMemcpyHostToDevice, ctx->stream));
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
  const long long per = (prefix[njobs] + ctx->persistBlocks - 1) / ctx->persistBlocks;
  bool narrow = true;
  for (int j = 0; j < njobs && narrow; ++j) narrow = ctx->hm[ctx->hEvalJobs[j].model].maxRowNnz <= 2;
  const size_t cacheBytes = static_cast<size_t>((per + 15) & ~15ll) + 24ull * static_cast<size_t>(per) + 16;
  a.cacheStates = (narrow && ctx->usePersistCache && cacheBytes <= kPersistCacheBytes) ? static_cast<int>(per) : 0;
  // interleaved RHS (k_eval_interleaved) whenever the chains are cached: every job <= 4 RHS here
  InterArgs ia{a, nullptr, nullptr, R};
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
  CK(cudaMemcpyAsync(ctx->dEvalJobsRaw, ctx->hEvalJobs.data(), njobs * sizeof(EvalJob), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->dMask, maskInit.data(), njobs * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->dNrhs, nrhs.data(), njobs * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->dStatus, statusInit.data(), njobs * MORAP_MAX_RHS * 4, cudaMemcpyHostToDevice, ctx->stream));
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
  if (tmaOk && !active.empty()) {
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
    if (tmaOk && ctx->usePersistent && njobs <= kPersistMaxJobs) {
      if ((rc = run_eval_persistent(ctx, njobs, eps, cap))) return rc;
    } else if ((rc = run_loop(ctx, 1, eps, cap))) {
      return rc;
    }
  }

  lap("sweeps");
  ctx->evalSweeps.assign(static_cast<size_t>(njobs) * MORAP_MAX_RHS, 0);
  std::vector<int32_t> st(static_cast<size_t>(njobs) * MORAP_MAX_RHS);
  std::vector<double> res(static_cast<size_t>(njobs) * MORAP_MAX_RHS);
  CK(d2h(ctx, ctx->evalSweeps.data(), ctx->dSweeps, njobs * MORAP_MAX_RHS * 4));
  CK(d2h(ctx, st.data(), ctx->dStatus, njobs * MORAP_MAX_RHS * 4));
  CK(d2h(ctx, res.data(), ctx->dResidual, njobs * MORAP_MAX_RHS * 8));
  std::vector<double> vals(static_cast<size_t>(njobs) * MORAP_MAX_RHS, 0.0);
  k_gather_eval<<<(njobs * MORAP_MAX_RHS + 255) / 256, 256, 0, ctx->stream>>>(
      ctx->dModels, (const EvalJob*)ctx->dEvalJobsRaw, njobs, ctx->dSweeps, ctx->dGather);
  CK(cudaGetLastError());
  CK(d2h(ctx, vals.data(), ctx->dGather, njobs * MORAP_MAX_RHS * 8));
  CK(d2h(ctx, ctx->hCtl, ctx->dCtl, sizeof(Ctl)));
  CK(cudaStreamSynchronize(ctx->stream));
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
  std::vector<size_t> off;  // byte offset of each model in the block
  std::vector<char> lean;   // stored without fp64 prob / objectives
  size_t bytes = 0;
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
  // every array of the batch in one block
  size_t bytes = 0;
  auto& off = P.off;
  off.assign(nmodels, 0);
  P.lean.assign(nmodels, 0);
  for (int m = 0; m < nmodels; ++m) {
    const morap_csr_view& v = models[m];
    off[m] = bytes;
    const bool lean = ctx->lean && compact[m].ok && ctx->useTma;
    P.lean[m] = lean;
    bytes += align_up(4ull * (v.num_states + 1), 256) + align_up(4ull * (v.num_rows + 1), 256) +
             align_up(4ull * v.nnz, 256) + (lean ? 0 : align_up(8ull * v.nnz, 256)) + align_up(1ull * v.num_states, 256) +
             (lean ? 0 : static_cast<size_t>(v.num_objectives) * align_up(8ull * v.num_rows, 256)) +
             align_up(4ull * tiles[m].size(), 256) + align_up(sizeof(TileDesc) * descs[m].size(), 256);
    if (compact[m].ok)
      bytes += align_up(v.nnz, 256) + align_up(8ull * compact[m].dict.size(), 256) + align_up(2ull * v.num_rows, 256) +
               align_up(8ull * compact[m].table.size(), 256) + align_up(4ull * compact[m].nTrW, 256) +
               align_up(4ull * compact[m].nStW, 256) + align_up(4ull * compact[m].nRowW, 256) + align_up(sizeof(TilePos) * compact[m].pos.size(), 256) +
               align_up(4ull * compact[m].outIdx.size(), 256) + align_up(4ull * compact[m].outGrp.size(), 256);
  }
  P.bytes = bytes;
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
  const auto& off = P.off;
  void* dev = devBase;
  parallel_for(nmodels, [&](int m) {
    const morap_csr_view& v = models[m];
    char* h = host + off[m];
    char* d = static_cast<char*>(dev) + off[m];
    DevModel dmod{};
    auto put = [&](const void* src, size_t n) {  // src == nullptr: reserve (filled by the caller)
      if (n && src) std::memcpy(h, src, n);
      char* at = d;
      const size_t a = align_up(n, 256);
      h += a;
      d += a;
      return at;
    };
    dmod.rowOffset = reinterpret_cast<const int32_t*>(put(v.row_offset, 4ull * (v.num_states + 1)));
    dmod.trnOffset = reinterpret_cast<const int32_t*>(put(v.trn_offset, 4ull * (v.num_rows + 1)));
    dmod.succ = reinterpret_cast<const int32_t*>(put(v.succ, 4ull * v.nnz));
    const bool lean = P.lean[m];  // fp64 prob / objectives live in the tables
    if (!lean) dmod.prob = reinterpret_cast<const double*>(put(v.prob, 8ull * v.nnz));
    dmod.done = reinterpret_cast<const uint8_t*>(put(v.done, v.num_states));
    if (!lean)
      for (int o = 0; o < v.num_objectives; ++o)
        dmod.obj[o] = reinterpret_cast<const double*>(put(v.rewards[o], 8ull * v.num_rows));
    dmod.tileStart = reinterpret_cast<const int32_t*>(put(tiles[m].data(), 4ull * tiles[m].size()));
    dmod.tiles = reinterpret_cast<const TileDesc*>(put(descs[m].data(), sizeof(TileDesc) * descs[m].size()));
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
      dmod.probIdx = reinterpret_cast<const uint8_t*>(put(c.idx.data(), c.idx.size()));
      dmod.probDict = reinterpret_cast<const double*>(put(c.dict.data(), 8ull * c.dict.size()));
      dmod.rclass = reinterpret_cast<const uint16_t*>(put(c.cls.data(), 2ull * c.cls.size()));
      dmod.classTable = reinterpret_cast<const double*>(put(c.table.data(), 8ull * c.table.size()));
      dmod.nclass = static_cast<int32_t>(c.table.size() / std::max(1, v.num_objectives));
      uint32_t* hs = reinterpret_cast<uint32_t*>(h);
      dmod.stW = reinterpret_cast<const uint32_t*>(put(nullptr, 4ull * c.nStW));
      uint32_t* hr = reinterpret_cast<uint32_t*>(h);
      dmod.rowW = reinterpret_cast<const uint32_t*>(put(nullptr, 4ull * c.nRowW));
      uint32_t* ht = reinterpret_cast<uint32_t*>(h);
      dmod.trW = reinterpret_cast<const uint32_t*>(put(nullptr, 4ull * c.nTrW));
      fill_streams(v, descs[m], c, hs, hr, ht);  // straight into the staging buffer
      dmod.tilePos = reinterpret_cast<const TilePos*>(put(c.pos.data(), sizeof(TilePos) * c.pos.size()));
      dmod.outIdx = reinterpret_cast<const int32_t*>(put(c.outIdx.data(), 4ull * c.outIdx.size()));
      dmod.outGrp = reinterpret_cast<const int32_t*>(put(c.outGrp.data(), 4ull * c.outGrp.size()));
      // compact stream: one 4-byte word per transition (window offset | index) and per row
      // (transition end | class) and per state (row end | transition end | done) + x 8 + y 8
      dmod.bytesPerSweep = 4ull * v.nnz + 4ull * v.num_rows + 20ull * v.num_states;
    }
    // evaluate, one RHS over the policy chain: chainOff 4 + done 1 + rhoC 8 + x 8 + y 8 per
    // state + 12 per chosen transition (mean nnz per row)
    const double nnzPerRow = v.num_rows ? static_cast<double>(v.nnz) / v.num_rows : 0.0;
    dmod.bytesPerEval = static_cast<unsigned long long>(v.num_states * (29.0 + 12.0 * nnzPerRow));
    built[m] = dmod;
    // this model's block goes out as soon as it is packed (copies overlap the packing)
    const size_t len = static_cast<size_t>(h - (host + off[m]));
    uploadBytes += static_cast<long long>(len);
    if (!copy) return;
    cudaSetDevice(ctx->device);  // packing runs on pool threads
    if (cudaMemcpyAsync(static_cast<char*>(dev) + off[m], host + off[m], len, cudaMemcpyHostToDevice, ctx->stream) !=
        cudaSuccess)
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
                       static_cast<int32_t>(P.compact[m].outGrp.size())};
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
  return d;
}

}  // namespace

struct morap_image {
  int device = 0;
  size_t bytes = 0;
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
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_greedy_sweep<false>, kBlock, 0);
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
  if (const char* pc = std::getenv("MORAP_PERSIST_CTAS")) persistPerSm = std::max(1, std::min(occP, std::atoi(pc)));
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
  const char* sel = std::getenv("MORAP_SWEEP_KERNEL");  // "global" selects the non-TMA sweep (A/B)
  ctx->useTma = !(sel && std::string(sel) == "global") && occT > 0;
  const char* gsel = std::getenv("MORAP_GRAPHS");  // "0" launches sweeps one by one (A/B)
  ctx->useGraphs = !(gsel && std::string(gsel) == "0");
  if (const char* dry = std::getenv("MORAP_DEBUG_DRY")) {
    const int on = std::atoi(dry);
    cudaMemcpyToSymbol(g_dryRun, &on, sizeof(int));
  }
  const char* csel = std::getenv("MORAP_COMPACT");  // "0" keeps the plain fp64 streams (A/B)
  ctx->useCompact = !(csel && std::string(csel) == "0");
  const char* ksel = std::getenv("MORAP_SKIP");  // "0" sweeps every tile every sweep (A/B)
  ctx->skip = !(ksel && std::string(ksel) == "0");
  ctx->selBlocks = ctx->numSMs * 4;
  if (cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking) != cudaSuccess) { delete ctx; return MORAP_CUDA_ERROR; }
  if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->polReady, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->polCopied, cudaEventDisableTiming) != cudaSuccess) {
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
  cudaFree(ctx->evalStage);
  cudaFreeHost(ctx->stage);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
  }
  if (ctx->polReady) cudaEventDestroy(ctx->polReady);
  if (ctx->polCopied) cudaEventDestroy(ctx->polCopied);
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
  if ((rc = prepare_models(ctx, nmodels, models, P))) return rc;
  void* dev = nullptr;
  if ((rc = acquire_block(ctx, P.bytes, &dev))) return rc;
  if (P.bytes > ctx->stageBytes) {  // pinned staging, grow-only (reused by later uploads)
    cudaFreeHost(ctx->stage);
    ctx->stage = nullptr;
    ctx->stageBytes = 0;
    CK(cudaMallocHost(&ctx->stage, P.bytes));
    ctx->stageBytes = P.bytes;
  }
  std::vector<DevModel> built(nmodels);
  std::atomic<bool> copyFailed{false};
  std::atomic<long long> uploadBytes{0};
  pack_models(ctx, nmodels, models, P, static_cast<char*>(ctx->stage), static_cast<char*>(dev), true, built, copyFailed,
              uploadBytes);
  ctx->stats[9] += static_cast<double>(uploadBytes.load());
  cudaError_t e = copyFailed ? cudaErrorUnknown : cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return ctx->cudaFail(e, "upload copy", __LINE__);
  return register_models(ctx, built, host_models(built, P), ids_out);
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
  CK(cudaMemcpyAsync(dev, img->host, img->bytes, cudaMemcpyHostToDevice, ctx->stream));
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
