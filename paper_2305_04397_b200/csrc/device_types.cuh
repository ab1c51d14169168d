// Device data layout and shared device helpers.
// Included by morap_cuda.cu inside its anonymous namespace (one translation unit: the
// kernels, their launch code and the C ABI share these definitions).

constexpr int kBlock = 256;     // threads per CTA = max states per tile
constexpr int kRowCap = 768;    // max action rows per tile (staged in shared memory)
constexpr int kNnzCap = 1024;   // max transitions per multi-state tile (staged)
constexpr int kFinBlock = 1024; // finalize kernel block
constexpr bool kFusedStates = true;  // TMA sweep: thread-per-state single pass (else 3 phases)
// Diagnostics (dev probes scripts/probe_cta_trace.py / probe_eval_trace.py):
//   MORAP_DEBUG_DRY=1  consumers skip the arithmetic, so the pipeline's pure streaming rate
//                      can be measured -- honoured only by -DMORAP_DIAGNOSTICS builds
//                      (MORAP_BUILD_DIAGNOSTICS=1 python -m paper_2305_04397_b200.build);
//   morap_cuda_debug_cta_trace  per sweep and CTA, globaltimer stamps {start, first stage
//                      consumed, all warps done, finalize done}.
// The two diagnostics globals are compiled in always (0 / null unless set): ptxas allocates
// the compact sweep kernel without spills only with the trace stamps present (without them:
// 104 B of spills and a ~4% slower sweep, C2 A/B). Only the dry-run switch (MORAP_DEBUG_DRY)
// is limited to diagnostics builds; traces are armed by morap_cuda_debug_cta_trace.
__device__ int g_dryRun = 0;
__device__ unsigned long long* g_ctaTrace = nullptr;
#define MORAP_DRY_RUN() (g_dryRun != 0)
#define MORAP_CTA_TRACE() (g_ctaTrace)
constexpr int kTraceSlots = 128;
// Device bounds checks, compiled in only with -DMORAP_CHECKED (MORAP_BUILD_CHECKED=1): every
// staged bulk copy against its shared-memory region and its source array, every gather
// index against its array. A failed check traps (the launch fails with an error); the GPU
// test suite runs under this build (compute-sanitizer is not available on this pool).
#ifdef MORAP_CHECKED
#define MORAP_CHECK(cond)                                                                  \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("MORAP_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             blockIdx.x, threadIdx.x);                                                     \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define MORAP_CHECK(cond) ((void)0)
#endif
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
  const uint32_t* trW;   // per transition: window offset | probability index << 16 (outside the
                         // window: bit 15 + index j into outSucc in bits 0-14, 24-31)
  const int32_t* outSucc;  // successors of the out-of-window transitions, in transition order
  const TilePos* tilePos;     // ntiles
  // frozen-tile skipping: stamp groups (32 states) of the successors outside each tile's
  // window, outGrp[outIdx[t] .. outIdx[t + 1]) (sorted, distinct; a single -1: too many)
  const int32_t* outIdx;      // ntiles + 1
  const int32_t* outGrp;
  int32_t S, R, nnz, initial, ntiles, K, rewardFinite, compact;
  int32_t nclass, nOutSucc;  // reward classes; out-of-window transitions (outSucc entries)
  int32_t nDict, nStW, nRowW, nTrW;  // probability dictionary entries; stream words (padded)
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

// Software grid barrier of the persistent (cooperative) kernels: every CTA of the grid is
// resident; fences order the sweep's global writes before the next phase reads them.
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
