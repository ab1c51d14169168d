// Dataflow optimize batch (K1 as ONE persistent launch per optimize call).
//
// numerics.hpp:84-113 is a Jacobi iteration per job: sweep k + 1 of job j needs every state
// of sweep k of job j -- and nothing of any other job. The lock-step design (one launch per
// sweep of every active job, k_select between launches) pays a grid-wide drain, a launch and
// a selection pass per sweep. Here each job advances on its own: the tiles of one job-sweep
// are cut into work items (segments of <= kFlowSegMax consecutive tiles) in a device ring;
// the producer warp of each persistent CTA claims items in order, keeps the tiles whose
// inputs changed in the job's previous sweep (frozen-tile skipping, the test k_select ran,
// now done per segment by the producer's lanes) and streams them through the usual
// cp.async.bulk / mbarrier stages to the compute warps (cmp_tile: the same arithmetic, so
// the same bits). When the compute warps finish the last kept tile of a segment they fold
// the segment's residual into the job's and count the segment done; whoever completes the
// job's last segment (a compute thread, or the producer lane when a whole segment was
// skipped) runs the job's stop test (numerics.hpp:105-112) and, if it goes on, publishes
// the next sweep's segments at the ring's tail. Jobs of different lengths overlap; the
// device never drains between sweeps and the host waits once per optimize call.
//
// Memory ordering: compute threads store y / stamps -> named barrier -> one thread
// __threadfence + atomicSub(pending) (release chain); the finisher observes pending == 0,
// fences, writes the job's sweep number and pending count, and publishes items with
// st.release; producers read items with ld.acquire and issue fence.proxy.async before the
// bulk copies (generic-proxy writes of other SMs -> async-proxy reads).

constexpr int kFlowQ = 4;       // work items a producer warp claims / resolves per round
constexpr int kFlowSegMax = 8;  // tiles per work item (item a on producer lanes 8a .. 8a+7)

// Diagnostics (-DMORAP_FLOW_PROF): per-CTA clock64 totals of what the producer and compute
// warp 0 wait on; g_flowProf[cta * 8 + i]. Never compiled into the shipped library.
#ifdef MORAP_FLOW_PROF
__device__ unsigned long long g_flowProf[4096 * 8];
#define FLOW_PROF_T0(v) const long long v = clock64()
#define FLOW_PROF_ADD(i, v) (g_flowProf[blockIdx.x * 8 + (i)] += clock64() - (v))
#else
#define FLOW_PROF_T0(v)
#define FLOW_PROF_ADD(i, v)
#endif

struct FlowCtl {
  unsigned long long head;  // next ring position to claim
  unsigned long long padH[15];
  unsigned long long tail;  // next ring position to reserve (own 128-byte line: different L2 atomics)
  unsigned long long padT[15];
  int32_t remaining;        // jobs still iterating
  int32_t done;             // 1: every job stopped (or an error)
  int32_t err;              // 1: queue stalled (watchdog), 2: ring lap overrun
  int32_t pad;
  unsigned long long bytes, backups;          // every tile of every sweep (reference work)
  unsigned long long execBytes, execBackups;  // tiles actually swept
};

struct FlowArgs {
  const DevModel* models;
  const OptJob* jobs;
  const int4* cand;  // k_build_cand records, cand[job.candBase + lt]
  const int32_t* candOut;
  const int32_t* candOutG;
  const int32_t* stampAll;
  unsigned long long* ring;
  unsigned long long mask;  // ring capacity - 1 (power of two)
  int logCap;
  int skip;  // frozen-tile skipping on
  FlowCtl* fc;
  int32_t* jobSweep;                // sweep in flight per job
  int32_t* pending;                 // items of that sweep not yet done
  unsigned long long* delta;        // residual of the sweep in flight (max, as u64 bits)
  double eps;
  int cap;
  int32_t* sweeps;
  double* residual;
  int32_t* status;
};

// item: tag (16) | job (22) | first tile (20) | count - 1 (5); tag = lap % 65535 + 1 (0 = empty)
__device__ __forceinline__ unsigned long long flow_tag(unsigned long long pos, int logCap) {
  return ((pos >> logCap) % 65535ull) + 1ull;
}
__device__ __forceinline__ unsigned long long flow_item(unsigned long long tag, int job, int lt0, int cnt) {
  return (tag << 48) | (static_cast<unsigned long long>(job) << 25) | (static_cast<unsigned long long>(lt0) << 5) |
         static_cast<unsigned long long>(cnt - 1);
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_s32(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Tiles per work item for a sweep published while `remaining` jobs iterate: large items
// while many jobs keep every CTA busy (fewer claims), small ones when a few long jobs are
// left (their sweeps spread over more CTAs: shorter critical path).
__device__ __host__ __forceinline__ int flow_seg(int remaining) {
  return remaining >= 32 ? 8 : remaining >= 8 ? 4 : 2;
}

__device__ __forceinline__ int atom_add_acq_rel(int32_t* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Sweep k of `job` is complete (every item done, residual folded in). Single thread, right
// after the acq_rel decrement that took the job's pending count to zero (acquire side:
// the job's y / stamps / residual of sweep k are visible); the items are published with
// release stores (the sweep number, pending count and cleared residual precede them).
__device__ __forceinline__ void flow_finish(const FlowArgs& A, int job, int k) {
  const int k1 = k + 1;
  const double d = __longlong_as_double(static_cast<long long>(__ldcg(A.delta + job)));
  const bool stop = d <= A.eps || k1 >= A.cap;  // numerics.hpp:105-112
  A.sweeps[job] = k1;
  A.residual[job] = d;
  const OptJob& J = A.jobs[job];
  atomicAdd(&A.fc->bytes, J.bytesPerSweep);
  atomicAdd(&A.fc->backups, static_cast<unsigned long long>(J.nnz));
  if (stop) {
    A.status[job] = d <= A.eps ? MORAP_OK : MORAP_NON_CONVERGENCE;
    if (atom_add_acq_rel(&A.fc->remaining, -1) == 1) atomicExch(&A.fc->done, 1);
    return;
  }
  const int nt = A.models[J.model].ntiles;
  const int seg = flow_seg(ld_relaxed_s32(&A.fc->remaining));
  const int nseg = (nt + seg - 1) / seg;
  A.delta[job] = 0ull;
  A.jobSweep[job] = k1;
  A.pending[job] = nseg;
  unsigned long long p = atomicAdd(&A.fc->tail, static_cast<unsigned long long>(nseg));
  __threadfence();  // one release for all the items (a release per store costs ~0.5 us each)
  for (int s = 0; s < nseg; ++s, ++p)
    st_relaxed_u64(A.ring + (p & A.mask), flow_item(flow_tag(p, A.logCap), job, s * seg, min(seg, nt - s * seg)));
}

// Which of two 16-bit lap tags is newer (tags run 1..65535 cyclically): true when `tag` is
// ahead of `want` -- the slot was already rewritten for a later lap (never expected).
__device__ __forceinline__ bool flow_tag_ahead(unsigned long long tag, unsigned long long want) {
  const unsigned long long d = (tag + 65535ull - want) % 65535ull;
  return tag != 0 && d != 0 && d < 32768ull;
}

// Compute warps only run tiles: per tile, each warp folds its threads' |y - x| into one
// value in shared memory and releases the stage. The producer warp does all the
// bookkeeping when it sees a stage released (it waits for that anyway before refilling
// the stage, and polls released stages while it waits for work): residual max per
// segment, the job's atomics, and the finisher role -- so no compute warp ever waits on a
// global atomic or a CTA barrier.
__global__ void __launch_bounds__(kTmaThreads, MORAP_CMP_CTAS) k_opt_flow(FlowArgs A) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kCmpStages], empty[kCmpStages];
  __shared__ CmpInfo info[kCmpStages];
  __shared__ int32_t sK[kCmpStages];                 // sweep of the staged tile (compute warps)
  __shared__ int32_t sBk[kCmpStages][3];             // producer-private: job, sweep, segment end
  __shared__ double sWarpMax[kCmpStages][kConsumers / 32];
  __shared__ int32_t sPos[32][4];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < kCmpStages; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kConsumers / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const DevModel* __restrict__ models = A.models;
  const OptJob* __restrict__ jobs = A.jobs;

  if (tid >= kConsumers) {
    // ---- producer warp ------------------------------------------------------------
    // Lanes 0..kFlowQ-1 each hold a claim on one ring position; every round the warp tops the
    // claims up, reads the claimed slots together, and resolves all the items that are there
    // -- item a on lanes 8a..8a+7, one tile per lane (frozen-tile test, tile tables) -- so the
    // dependent load chain is paid once per up to 32 tiles, not once per segment.
    const int lane = tid & 31;
    const uint64_t pol = evict_first_policy(), polKeep = evict_last_policy();
    const int laneSh = lane == 6 || lane == 7 ? 3 : 2;
    const int laneDst = lane == 0 ? kCOffRow : lane == 1 ? kCOffTrn : lane == 2 ? kCOffSucc : lane == 6 ? kCOffX
                      : kCOffXw;
    int use = 0, booked = 0;  // stages issued / stages whose completion was booked
    int curJob = -1, curK = -1;
    double segMax = 0.0;      // residual of the segment being completed (lane 0)
    const unsigned char* myBase = nullptr;
    const DevModel* curM = nullptr;
    const OptJob* curJ = nullptr;
    unsigned long long exBytes = 0, exNnz = 0;  // a CTA streams several GB per C4 batch
    // one segment completion in flight (lane 0): its pending decrement's old value is only
    // looked at on the next completion or when the warp idles, so the atomic's round trip
    // overlaps other work; the finisher role is never lost (flushed before any wait)
    int outOld = 0, outJob = -1, outK = 0;
    auto flush = [&]() {
      if (lane == 0 && outJob >= 0) {
        if (outOld == 1) flow_finish(A, outJob, outK);
        outJob = -1;
      }
    };
    auto complete = [&](int job, int k) {  // lane 0: a segment of (job, sweep k) is done
      if (outJob >= 0 && outOld == 1) flow_finish(A, outJob, outK);
      outOld = atom_add_acq_rel(A.pending + job, -1);
      outJob = job;
      outK = k;
    };
    // book the completion of stage use `u` (its empty barrier phase completed)
    auto book = [&](int u) {
      const int b = u % kCmpStages;
      double m = lane < kConsumers / 32 ? sWarpMax[b][lane] : 0.0;
      m = warp_max(m);
      if (lane == 0) {
        segMax = fmax(segMax, m);
        if (sBk[b][2]) {  // the segment's last kept tile: the segment is done
          const int job = sBk[b][0];
          if (segMax > 0.0) atomicMax(A.delta + job, (unsigned long long)__double_as_longlong(segMax));
          complete(job, sBk[b][1]);
          segMax = 0.0;
        }
      }
      __syncwarp();
    };
    unsigned long long myPos = 0;  // lanes < kFlowQ: the claimed ring position
    int have = 0;
    const unsigned long long t0 = global_ns();
    for (int spin = 0;; ++spin) {
      // ---- top up the claims (kFlowQ positions per warp), read the claimed slots ----------
      const unsigned needMask = __ballot_sync(0xffffffffu, lane < kFlowQ && !have);
      if (needMask) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&A.fc->head, static_cast<unsigned long long>(__popc(needMask)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((needMask >> lane) & 1) {
          myPos = base + __popc(needMask & ((1u << lane) - 1u));
          have = 1;
        }
      }
      unsigned long long v = 0;
      int avail = 0;
      if (lane < kFlowQ && have) {
        v = ld_relaxed_u64(A.ring + (myPos & A.mask));
        const unsigned long long want = flow_tag(myPos, A.logCap), tag = v >> 48;
        avail = tag == want;
        if (!avail && flow_tag_ahead(tag, want)) {  // ring overrun: report, never compute on it
          atomicExch(&A.fc->err, 2);
          atomicExch(&A.fc->done, 1);
        }
      }
      const unsigned amask = __ballot_sync(0xffffffffu, avail);
      if (amask == 0) {  // nothing claimable yet: finish pending work, then poll
        flush();
        int stop = 0;
        if (lane == 0) {
          stop = ld_relaxed_s32(&A.fc->done);
          if ((spin & 63) == 63 && global_ns() - t0 > 60000000000ull) {  // 60 s in this batch: stalled
            atomicExch(&A.fc->err, 1);
            atomicExch(&A.fc->done, 1);
          }
        }
        if (__shfl_sync(0xffffffffu, stop, 0)) break;
        int released = 0;
        if (lane == 0 && booked < use) released = mbar_test(&empty[booked % kCmpStages], (booked / kCmpStages) & 1);
        if (__shfl_sync(0xffffffffu, released, 0)) book(booked++);
        else __nanosleep(64);
        continue;
      }
      FLOW_PROF_T0(pr);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire: what the items' publishers wrote
      fence_proxy_async();
      if (avail) have = 0;  // consumed
      // ---- resolve: item a on lanes 8a .. 8a+7, one tile per lane ------------------------
      const int a = lane >> 3, sub = lane & 7;
      const unsigned long long item = __shfl_sync(0xffffffffu, v, a);
      const int job = static_cast<int>((item >> 25) & 0x3FFFFFull);
      const int lt0 = static_cast<int>((item >> 5) & 0xFFFFFull);
      const int cnt = static_cast<int>(item & 31ull) + 1;
      const bool live = ((amask >> a) & 1) && sub < cnt;
      int keep = 0, k = 0;
      int mS0 = 0, mR0 = 0, mK0 = 0, mFits = 0, mWlo = 0, mWn = 0, mAll = 0, mSimple = 0, eS0 = 0, eR0 = 0, eK0 = 0;
      __syncwarp();
      if (live) {
        const OptJob& J = jobs[job];
        const int lt = lt0 + sub;
        k = __ldcg(A.jobSweep + job);
        keep = 1;
        if (A.skip && k > 0) {
          const int ci = J.candBase + lt;
          const int4 c = __ldg(A.cand + ci);
          if (c.z >= 0) {
            const int4* stamp = reinterpret_cast<const int4*>(A.stampAll);
            const unsigned u = static_cast<unsigned>(c.y);
            const int nw = (u >> kCandLtBits) & 15, no = (u >> (kCandLtBits + 4)) & 7, nout = u >> (kCandLtBits + 7);
            const int oo = __ldg(A.candOut + ci);
            int m = 0;
            for (int q = 0; q < nout; ++q) m = max(m, __ldcg(A.stampAll + __ldg(A.candOutG + oo + q)));
            for (int q = 0; q < nw; ++q) {
              const int4 w4 = __ldcg(stamp + (c.z >> 2) + q);
              m = max(m, max(max(w4.x, w4.y), max(w4.z, w4.w)));
            }
            for (int q = 0; q < no; ++q) {
              const int4 w4 = __ldcg(stamp + (c.w >> 2) + q);
              m = max(m, max(max(w4.x, w4.y), max(w4.z, w4.w)));
            }
            keep = m >= k;  // an input changed in sweep k - 1 (stamped k)
          }
        }
        if (keep) {
          const DevModel* M = &models[J.model];
          const int4* tp = reinterpret_cast<const int4*>(M->tiles + lt);
          const int4 d0 = tp[0], d1 = tp[1], e0 = tp[2];
          const int4 p0 = *reinterpret_cast<const int4*>(M->tilePos + lt);
          mS0 = d0.x; mR0 = d0.y; mK0 = d0.z; mFits = d0.w;
          mWlo = d1.x; mWn = d1.y; mAll = d1.z; mSimple = d1.w;
          eS0 = e0.x; eR0 = e0.y; eK0 = e0.z;
          sPos[lane][0] = p0.x; sPos[lane][1] = p0.y; sPos[lane][2] = p0.z;
        }
      }
      const unsigned kmask = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (lane == 0) FLOW_PROF_ADD(1, pr);
      {  // items whose tiles are all frozen are done already (job / sweep from the item's first lane)
        for (unsigned am = amask; am; am &= am - 1) {
          const int ia = __ffs(am) - 1;
          const int jb = __shfl_sync(0xffffffffu, job, 8 * ia), kk = __shfl_sync(0xffffffffu, k, 8 * ia);
          if (((kmask >> (8 * ia)) & 0xFFu) == 0 && lane == 0) complete(jb, kk);
        }
      }
      // ---- issue the kept tiles, item by item (segments stay contiguous) ------------------
      for (unsigned rest = kmask; rest; rest &= rest - 1, ++use) {
        const int q = __ffs(rest) - 1;
        const int tj = __shfl_sync(0xffffffffu, job, q), tk = __shfl_sync(0xffffffffu, k, q);
        const bool segEnd = ((kmask >> q) & ((0xFFu << (8 * (q >> 3))) >> q)) == 1u;  // last kept of its item
        if (tj != curJob || tk != curK) {  // uniform: this lane's stream base for the job / sweep
          curJob = tj;
          curK = tk;
          curJ = &jobs[tj];
          curM = &models[curJ->model];
          const void* bp = nullptr;
          switch (lane) {
            case 0: bp = curM->stW; break;
            case 1: bp = curM->rowW; break;
            case 2: bp = curM->trW; break;
            case 6:
            case 7: bp = curJ->buf[tk & 1]; break;
            default: break;
          }
          myBase = static_cast<const unsigned char*>(bp);
        }
        const int s0 = __shfl_sync(0xffffffffu, mS0, q), r0 = __shfl_sync(0xffffffffu, mR0, q);
        const int k0 = __shfl_sync(0xffffffffu, mK0, q), fits = __shfl_sync(0xffffffffu, mFits, q);
        const int wlo = __shfl_sync(0xffffffffu, mWlo, q), wn = __shfl_sync(0xffffffffu, mWn, q);
        const int allIn = __shfl_sync(0xffffffffu, mAll, q);
        const int simple = __shfl_sync(0xffffffffu, mSimple, q);
        const int s1 = __shfl_sync(0xffffffffu, eS0, q), r1 = __shfl_sync(0xffffffffu, eR0, q);
        const int k1 = __shfl_sync(0xffffffffu, eK0, q);
        exBytes += 4u * (k1 - k0) + 4u * (r1 - r0) + 20u * (s1 - s0);
        exNnz += static_cast<unsigned>(k1 - k0);
        const int b = use % kCmpStages;
        const int pos = lane < 3 ? sPos[q][lane] : 0;
        const int len = lane == 0 ? s1 - s0 : (lane == 1 ? r1 - r0 : k1 - k0);
        long long lo = lane < 6 ? pos : (lane == 6 ? s0 : wlo);
        long long hi = lane < 6 ? pos + len : (lane == 6 ? s1 : wlo + wn);
        if (lane > 7 || (lane >= 3 && lane <= 5)) lo = hi = 0;
        const uint64_t lp = lane >= 6 ? polKeep : pol;
        const long long a0 = (lo << laneSh) & ~15ll, z0 = ((hi << laneSh) + 15) & ~15ll;
        const uint32_t bytes = (myBase && fits && z0 > a0) ? static_cast<uint32_t>(z0 - a0) : 0u;
        const int off = static_cast<int>(((lo << laneSh) - a0) >> laneSh);
        const uint32_t txBytes = __reduce_add_sync(0xffffffffu, bytes);
        if (use >= kCmpStages) {  // refill: the stage's previous tile is done -- book it
          FLOW_PROF_T0(pe);
          mbar_wait_sleep(&empty[b], ((use / kCmpStages) - 1) & 1);
          if (lane == 0) FLOW_PROF_ADD(2, pe);
          FLOW_PROF_T0(pb);
          while (booked <= use - kCmpStages) book(booked++);
          if (lane == 0) FLOW_PROF_ADD(3, pb);
        }
        const int offX = __shfl_sync(0xffffffffu, off, 6);
        if (lane == 0) {
          CmpInfo rec;
          rec.t = lt0 + q;
          rec.job = tj;
          rec.fits = fits;
          rec.allIn = allIn;
          rec.simple = simple;
          rec.s0 = s0;
          rec.r0 = r0;
          rec.k0 = k0;
          rec.ns = s1 - s0;
          rec.offX = offX;
          rec.stamp = A.skip ? curJ->stamp : nullptr;
          rec.dict = curM->probDict;
          rec.classRho = curJ->classRho;
          rec.x = curJ->buf[tk & 1];
          rec.y = curJ->buf[(tk & 1) ^ 1];
          rec.policy = curJ->policy;
          rec.model = curM;
          rec.succG = curM->succ;
          rec.rho = curJ->rho;
          info[b] = rec;
          sK[b] = tk;
          sBk[b][0] = tj;
          sBk[b][1] = tk;
          sBk[b][2] = segEnd;
        }
        __syncwarp();
        uint64_t* bar = &full[b];
        if (lane == 0) {
          if (fits) mbar_expect_tx(bar, txBytes);
          else mbar_arrive(bar);
        }
        __syncwarp();
        if (bytes) bulk_g2s(smem + b * kCStageBytes + laneDst, myBase + a0, bytes, bar, lp);
      }
    }
    // every job stopped: nothing this CTA issued is still unbooked (a job stops only after
    // its last segment was booked); release the compute warps
    if (lane == 0) {
      if (exNnz) {
        atomicAdd(&A.fc->execBytes, exBytes);
        atomicAdd(&A.fc->execBackups, exNnz);
      }
      const int b = use % kCmpStages;
      if (use >= kCmpStages) mbar_wait_sleep(&empty[b], ((use / kCmpStages) - 1) & 1);
      info[b].t = -1;
      mbar_arrive(&full[b]);
    }
  } else {
    // ---- compute warps ------------------------------------------------------------
    const int lane = tid & 31, wid = tid >> 5;
    for (int use = 0;; ++use) {
      const int b = use % kCmpStages;
      FLOW_PROF_T0(cw);
      mbar_wait_sleep(&full[b], (use / kCmpStages) & 1);
      if (tid == 0) FLOW_PROF_ADD(4, cw);
      const CmpInfo v = info[b];
      if (v.t < 0) break;
      FLOW_PROF_T0(cc);
      const double m = warp_max(cmp_tile<false>(v, smem + b * kCStageBytes, tid, sK[b]));
      if (tid == 0) FLOW_PROF_ADD(5, cc);
#ifdef MORAP_FLOW_PROF
      if (tid == 0) g_flowProf[blockIdx.x * 8 + 6] += 1;
#endif
      if (lane == 0) sWarpMax[b][wid] = m;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);  // release.cta: y / stamps / the warp max
    }
  }
}
