// Optimize kernels: weighted rewards (K3), the fp64 TMA sweep and the compact sweep with frozen-tile selection (K1).
// Included by morap_cuda.cu inside its anonymous namespace (one translation unit: the
// kernels, their launch code and the C ABI share these definitions).

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
    if (v.fits && MORAP_DRY_RUN()) {
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
// Latest stamp among the groups candidate c depends on: its successor window, its own states
// and up to kMaxOutGroups out-of-window groups (the lists k_build_cand packed). Every load is
// predicated inside fully unrolled loops so a thread has them all in flight at once (the
// data-dependent loops left up to ~30 dependent L2 round trips on the selection's tail).
__device__ __forceinline__ int cand_stamp_max(const int4 c, int oo, const int32_t* __restrict__ stampAll,
                                              const int32_t* __restrict__ candOutG) {
  const int4* stamp = reinterpret_cast<const int4*>(stampAll);
  const unsigned u = static_cast<unsigned>(c.y);
  const int nw = (u >> kCandLtBits) & 15, no = (u >> (kCandLtBits + 4)) & 7, nout = u >> (kCandLtBits + 7);
  int m = 0;
#pragma unroll
  for (int h = 0; h < kMaxOutGroups; h += 8) {  // successors outside the window, 8 groups at a time
    int g[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) g[q] = h + q < nout ? __ldg(candOutG + oo + h + q) : -1;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (g[q] >= 0) m = max(m, __ldcg(stampAll + g[q]));
  }
#pragma unroll
  for (int q = 0; q < 15; ++q)  // successor window (<= 15 loads of 4 stamps)
    if (q < nw) {
      const int4 v = __ldcg(stamp + (c.z >> 2) + q);
      m = max(m, max(max(v.x, v.y), max(v.z, v.w)));
    }
#pragma unroll
  for (int q = 0; q < 7; ++q)  // own states (<= 7 loads of 4 stamps)
    if (q < no) {
      const int4 v = __ldcg(stamp + (c.w >> 2) + q);
      m = max(m, max(max(v.x, v.y), max(v.z, v.w)));
    }
  return m;
}

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
  __shared__ int sCnt[kSelThreads / 32], sOff[kSelThreads / 32], sBase;
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
          keep = cand_stamp_max(c, oo, stampAll, candOutG) >= k;  // a dependency changed in the previous sweep
        }
      }
      c.y &= (1 << kCandLtBits) - 1;
    }
    // compaction per CTA: one atomic per CTA with a kept tile (same-address atomics from every
    // warp of the grid serialise in L2), order kept within the CTA
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) sCnt[wid] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < kSelThreads / 32; ++w) {
        sOff[w] = tot;
        tot += sCnt[w];
      }
      sBase = tot ? atomicAdd(&ctl->nsel, tot) : 0;
    }
    __syncthreads();
    if (keep) sel[sBase + sOff[wid] + __popc(bal & ((1u << lane) - 1u))] = make_int2(c.x, c.y);
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
  const int32_t* succG;  // the model's out-of-window successors (DevModel::outSucc)
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
  if (v.fits && MORAP_DRY_RUN()) {
    // diagnostics: stream only
  } else if (v.fits) {
    // Tile-relative u16 row ends per state: state i owns rows [rowE[i-1], rowE[i]) (0 for
    // i = 0). One u32 word per row: transition end (tile-relative, bits 0-10) and reward
    // class (bits 11-31); one u32 word per transition: window offset (low 16 bits, bit 15 set
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
        auto term = [&](uint32_t w) {
          MORAP_CHECK((w & 0xFFFFu) < static_cast<uint32_t>(kXWin + 2));
          return __dmul_rn(__ldg(dict + (w >> 16)), xwS[w & 0xFFFFu]);
        };
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
            const unsigned j = (o & 0x7FFFu) | ((w >> 24) << 15);  // out-of-window: outSucc index
            MORAP_CHECK(o & 0x8000u ? __ldg(v.succG + j) < v.model->S : o < static_cast<unsigned>(kXWin + 2));
            return o < 0x8000u ? xwS[o] : __ldg(x + __ldg(v.succG + j));
          };
          for (int r = rb; r < re; ++r) {
            const uint32_t rw = rowW[r];
            const int ke = static_cast<int>(rw & 0x7FFu);
            double acc = __ldg(crho + (rw >> 11));
            for (int q = kb; q < ke; ++q) {
              const uint32_t w = trW[q];
              acc = __dadd_rn(acc, __dmul_rn(__ldg(dict + ((w >> 16) & 0xFFu)), xAt(q, w)));
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
      !POLICY && MORAP_CTA_TRACE() ? MORAP_CTA_TRACE() + (static_cast<size_t>(k % kTraceSlots) * gridDim.x + blockIdx.x) * 4
                                  : nullptr;
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
          rec.succG = curM->outSucc;  // out-of-window successors of the model
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
        MORAP_CHECK(bytes <= static_cast<uint32_t>(lane == 0   ? kCOffTrn - kCOffRow
                                                   : lane == 1 ? kCOffSucc - kCOffTrn
                                                   : lane == 2 ? kCOffX - kCOffSucc
                                                   : lane == 6 ? kCOffXw - kCOffX
                                                               : kCStageBytes - kCOffXw));
        MORAP_CHECK(!bytes || lane < 6 || (lo >= 0 && hi <= curM->S));
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

