// Evaluate kernels: policy chains, the chain sweeps (K2: TMA, persistent, interleaved, plain), the finalize step and result gathers.
// Included by morap_cuda.cu inside its anonymous namespace (one translation unit: the
// kernels, their launch code and the C ABI share these definitions).

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
    unsigned long long* trace = MORAP_CTA_TRACE() ? MORAP_CTA_TRACE() + (static_cast<size_t>(k % kTraceSlots) * gridDim.x + blockIdx.x) * 4
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

// Results of a batch packed for ONE device-to-host copy: value (initial state of the final
// buffer), residual, sweeps, status of m entries -> out[0..m), out[m..2m), then 2 x m int32.
__device__ __forceinline__ void pack_result(double* out, int m, int q, double value, double residual, int sweeps,
                                            int status) {
  out[q] = value;
  out[m + q] = residual;
  int32_t* o = reinterpret_cast<int32_t*>(out + 2 * static_cast<size_t>(m));
  o[q] = sweeps;
  o[m + q] = status;
}

__global__ void k_gather_opt(const DevModel* __restrict__ models, const OptJob* __restrict__ jobs, int njobs,
                             const int32_t* __restrict__ sweeps, const int32_t* __restrict__ status,
                             const double* __restrict__ residual, double* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < njobs; j += gridDim.x * blockDim.x) {
    const int sw = sweeps[j];
    pack_result(out, njobs, j, sw > 0 ? jobs[j].buf[sw & 1][models[jobs[j].model].initial] : 0.0, residual[j], sw,
                status[j]);
  }
}

__global__ void k_gather_eval(const DevModel* __restrict__ models, const EvalJob* __restrict__ jobs, int njobs,
                              const int32_t* __restrict__ sweeps, const int32_t* __restrict__ status,
                              const double* __restrict__ residual, double* __restrict__ out) {
  const int m = njobs * MORAP_MAX_RHS;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < m; q += gridDim.x * blockDim.x) {
    const int j = q / MORAP_MAX_RHS, o = q % MORAP_MAX_RHS;
    const int sw = sweeps[q];
    pack_result(out, m, q, (o < jobs[j].nrhs && sw > 0) ? jobs[j].buf[o][sw & 1][models[jobs[j].model].initial] : 0.0,
                residual[q], sw, status[q]);
  }
}
