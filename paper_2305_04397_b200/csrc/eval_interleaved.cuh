// K2i: the persistent evaluate kernel with the RHS interleaved (included by morap_cuda.cu
// after k_eval_persistent; same arguments plus two interleaved arrays).
//
// evaluateSchedulerOn (numerics.hpp:138-162) for a batch of policy chains whose rows have
// at most two transitions (every warehouse product) and at most four RHS per job, cached in
// shared memory like k_eval_persistent's cache path. What changes is the layout of the
// values: x of all RHS of a state sits in one 16- or 32-byte record, xi[parity][i][0..R),
// i the state's index in the batch (R = 2 or 4), and so does its reward, rhoI[i][0..R).
// A state update is then four 16-byte global accesses per R = 2 (own x, reward, two
// successors) plus the 16-byte store, where the per-RHS layout took four 8-byte loads and a
// store per RHS: half the LSU wavefronts for the gathers, which bound the sweep
// (profiles: ~10 us of LSU-limited compute per C2 sweep).
//
// Per-RHS stop rule (numerics.hpp:105-112 per RHS): a stopped RHS of a still-running job
// copies its value forward (y = x), so after the job's last sweep K_j the final value of
// every RHS is in xi[K_j & 1]; the kernel ends by scattering those into the per-RHS buffers
// buf[o][sweeps_o & 1] that the gather / fetch paths read. Arithmetic per RHS is the same
// rounded sequence as k_eval_persistent: bitwise identical results.

struct InterArgs {
  PersistArgs p;
  double* xi;    // 2 x total x R, zeroed (x = 0 at the start, numerics.hpp:141)
  double* rhoI;  // total x R, filled by the prologue from rhoC
  int R;         // 2 or 4
  int direct;    // the chosen row of each state comes from J.policy (no chain CSR built), its
                 // transitions from the model CSR (1) or from the compact sweep streams (2)
};

template <int R>
__global__ void __launch_bounds__(kPersistThreads, MORAP_PERSIST_MINB) k_eval_interleaved(InterArgs IA) {
  const PersistArgs& A = IA.p;
  __shared__ uint32_t sMask[kPersistMaxJobs];
  // per job: bit o = parity of the sweep after which RHS o stopped, bit 8 = parity of K_j,
  // the sweep after which the whole job stopped (where its final values sit in xi)
  __shared__ uint32_t sLast[kPersistMaxJobs];
  __shared__ unsigned long long sDelta[kPersistJobs * MORAP_MAX_RHS];
  __shared__ int sActive;
  const int tid = threadIdx.x;
  const long long total = A.statePrefix[A.njobs];
  const long long per = (total + gridDim.x - 1) / gridDim.x;
  const long long i0 = static_cast<long long>(blockIdx.x) * per;
  const long long i1 = min(total, i0 + per);
  const int nloc = static_cast<int>(max(0ll, i1 - i0));
  for (int j = tid; j < A.njobs; j += blockDim.x) {
    sMask[j] = A.mask[j];
    sLast[j] = 0;
  }
  int jBase = 0;
  if (i0 < total) {
    int lo = 0, hi = A.njobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (A.statePrefix[mid] <= i0) lo = mid; else hi = mid - 1;
    }
    jBase = lo;
  }
  // chain cache: transition count, both successors (int2) and both probabilities (double2)
  extern __shared__ __align__(16) unsigned char esm[];
  const int C = A.cacheStates;
  uint8_t* sN = esm;
  int2* sSucc = reinterpret_cast<int2*>(esm + ((C + 15) & ~15));
  double2* sProb = reinterpret_cast<double2*>(esm + ((C + 15) & ~15) + ((8 * static_cast<size_t>(C) + 15) & ~15ull));
  {
    int jl = jBase;
    for (int li = tid; li < nloc; li += blockDim.x) {
      const long long i = i0 + li;
      while (i >= A.statePrefix[jl + 1]) ++jl;
      const EvalJob& J = A.jobs[jl];
      const int sl = static_cast<int>(i - A.statePrefix[jl]);
      double r[R];
      if (IA.direct == 2) {
        // the same chain decoded from the sweep streams: the state's tile,
        // its state word (done), the chosen row's word (transition end, reward class), the
        // transition words (window offset or out-of-window index, probability index)
        const DevModel& M = A.models[J.model];
        int lo = 0, hi = M.ntiles - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (__ldg(M.tileStart + mid) <= sl) lo = mid; else hi = mid - 1;
        }
        const TileDesc& d = M.tiles[lo];
        const TilePos& P = M.tilePos[lo];
        int nl = 0, cls = 0;
        int2 sc = make_int2(0, 0);
        double2 pr = make_double2(0.0, 0.0);
        if (!(__ldg(M.stW + P.row + (sl - d.s0)) >> 21 & 1u)) {
          const int lr = J.policy[sl] - d.r0;
          const uint32_t rw = __ldg(M.rowW + P.trn + lr);
          const int kb = lr ? static_cast<int>(__ldg(M.rowW + P.trn + lr - 1) & 0x7FFu) : 0;
          nl = static_cast<int>(rw & 0x7FFu) - kb;
          cls = static_cast<int>(rw >> 11);
          auto succOf = [&](uint32_t w) {
            const unsigned o = w & 0xFFFFu;
            return o < 0x8000u ? d.wlo + static_cast<int>(o) : __ldg(M.outSucc + ((o & 0x7FFFu) | ((w >> 24) << 15)));
          };
          if (nl > 0) {
            const uint32_t w0 = __ldg(M.trW + P.succ + kb);
            sc.x = succOf(w0);
            pr.x = M.probDict[(w0 >> 16) & 0xFFu];
          }
          if (nl > 1) {
            const uint32_t w1 = __ldg(M.trW + P.succ + kb + 1);
            sc.y = succOf(w1);
            pr.y = M.probDict[(w1 >> 16) & 0xFFu];
          }
        }
        sN[li] = static_cast<uint8_t>(nl);
        sSucc[li] = sc;
        sProb[li] = pr;
#pragma unroll
        for (int o = 0; o < R; ++o) r[o] = o < J.nrhs && nl > 0 ? M.classTable[cls * M.K + J.objIdx[o]] : 0.0;
      } else if (IA.direct) {
        // the policy chain of k_chain_fill, read in place: the chosen row's transitions
        // (succ, model probability) and its reward per RHS; done states: empty, reward 0
        const DevModel& M = A.models[J.model];
        int nl = 0, kb = 0, row = 0;
        if (!M.done[sl]) {
          row = J.policy[sl];
          kb = M.trnOffset[row];
          nl = M.trnOffset[row + 1] - kb;
        }
        sN[li] = static_cast<uint8_t>(nl);
        sSucc[li] = make_int2(nl > 0 ? M.succ[kb] : 0, nl > 1 ? M.succ[kb + 1] : 0);
        sProb[li] = make_double2(nl > 0 ? model_prob(M, kb) : 0.0, nl > 1 ? model_prob(M, kb + 1) : 0.0);
#pragma unroll
        for (int o = 0; o < R; ++o)
          r[o] = o < J.nrhs && nl > 0 ? (J.rho[o] ? J.rho[o][row] : model_obj(M, J.objIdx[o], row)) : 0.0;
      } else {
        const int cbl = __ldg(J.chainOff + sl), nl = __ldg(J.chainOff + sl + 1) - cbl;
        sN[li] = static_cast<uint8_t>(nl);
        sSucc[li] = make_int2(nl > 0 ? __ldg(J.chainSucc + cbl) : 0, nl > 1 ? __ldg(J.chainSucc + cbl + 1) : 0);
        sProb[li] = make_double2(nl > 0 ? __ldg(J.chainProb + cbl) : 0.0, nl > 1 ? __ldg(J.chainProb + cbl + 1) : 0.0);
#pragma unroll
        for (int o = 0; o < R; ++o) r[o] = o < J.nrhs ? __ldg(J.rhoC[o] + sl) : 0.0;
      }
      double2* dst = reinterpret_cast<double2*>(IA.rhoI + i * R);
#pragma unroll
      for (int h = 0; h < R / 2; ++h) dst[h] = make_double2(r[2 * h], r[2 * h + 1]);
    }
  }
  __syncthreads();  // (rhoI rows are read back by the thread that wrote them)
  unsigned long long bytesAcc = 0, backupsAcc = 0;
  int k = 0;
  for (;; ++k) {
    const int parity = k & 1;
    unsigned long long* trace = MORAP_CTA_TRACE() ? MORAP_CTA_TRACE() + (static_cast<size_t>(k % kTraceSlots) * gridDim.x + blockIdx.x) * 4
                                           : nullptr;
    if (trace && tid == 0) trace[0] = global_ns();
    unsigned long long* slot = A.slots + static_cast<size_t>(k % 3) * A.njobs * MORAP_MAX_RHS;
    for (int q = tid; q < kPersistJobs * MORAP_MAX_RHS; q += blockDim.x) sDelta[q] = 0ull;
    __syncthreads();
    // (no __restrict__ / const-restrict on xr: it must not become a non-coherent load,
    // the previous sweep of this launch wrote it)
    const double* xr = IA.xi + static_cast<size_t>(parity) * total * R;
    double* xw = IA.xi + static_cast<size_t>(parity ^ 1) * total * R;
    int j = jBase, runJob = -1;
    double run[R];
#pragma unroll
    for (int o = 0; o < R; ++o) run[o] = 0.0;
    auto flush = [&]() {
      if (runJob < 0) return;
      const int rel = runJob - jBase;
#pragma unroll
      for (int o = 0; o < R; ++o) {
        if (run[o] > 0.0) {
          const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(run[o]));
          if (rel < kPersistJobs) atomicMax(&sDelta[rel * MORAP_MAX_RHS + o], bits);
          else atomicMax(&slot[runJob * MORAP_MAX_RHS + o], bits);
        }
        run[o] = 0.0;
      }
    };
#pragma unroll 2
    for (int li = tid; li < nloc; li += blockDim.x) {
      const long long i = i0 + li;
      while (i >= A.statePrefix[j + 1]) ++j;
      const uint32_t mk = sMask[j];
      if (!mk) continue;
      const int n = sN[li];
      const int2 sc = sSucc[li];
      const long long base = A.statePrefix[j];
      MORAP_CHECK(li < C && (n < 1 || (sc.x >= 0 && base + sc.x < A.statePrefix[j + 1])) &&
                  (n < 2 || (sc.y >= 0 && base + sc.y < A.statePrefix[j + 1])));
      // every load of the state first (x of the batch is read through L1: the grid
      // barrier's fences make the previous sweep's writes visible)
      double2 xs[R / 2], rh[R / 2], x0[R / 2], x1[R / 2];
      const double2* xsP = reinterpret_cast<const double2*>(xr + i * R);
      const double2* rhP = reinterpret_cast<const double2*>(IA.rhoI + i * R);
      const double2* x0P = reinterpret_cast<const double2*>(xr + (base + sc.x) * R);
      const double2* x1P = reinterpret_cast<const double2*>(xr + (base + sc.y) * R);
#pragma unroll
      for (int h = 0; h < R / 2; ++h) {
        xs[h] = xsP[h];
        rh[h] = rhP[h];
        x0[h] = n > 0 ? x0P[h] : make_double2(0.0, 0.0);
        x1[h] = n > 1 ? x1P[h] : make_double2(0.0, 0.0);
      }
      const double2 pr = sProb[li];
      if (j != runJob) {
        flush();
        runJob = j;
      }
      double y[R];
#pragma unroll
      for (int o = 0; o < R; ++o) {
        const double xo = o & 1 ? xs[o >> 1].y : xs[o >> 1].x;
        if (mk >> o & 1u) {
          double acc = o & 1 ? rh[o >> 1].y : rh[o >> 1].x;
          if (n > 0) acc = __dadd_rn(acc, __dmul_rn(pr.x, o & 1 ? x0[o >> 1].y : x0[o >> 1].x));
          if (n > 1) acc = __dadd_rn(acc, __dmul_rn(pr.y, o & 1 ? x1[o >> 1].y : x1[o >> 1].x));
          y[o] = __dadd_rn(0.0, __dmul_rn(1.0, acc));
          run[o] = fmax(run[o], fabs(__dsub_rn(y[o], xo)));
        } else {
          y[o] = xo;  // stopped RHS (or padding): carried forward
        }
      }
      double2* yP = reinterpret_cast<double2*>(xw + i * R);
#pragma unroll
      for (int h = 0; h < R / 2; ++h) yP[h] = make_double2(y[2 * h], y[2 * h + 1]);
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
      const uint32_t before = mk;
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
        if (st >= 0) {
          mk &= ~(1u << o);
          sLast[jj] |= static_cast<uint32_t>((k + 1) & 1) << o;
        }
      }
      sMask[jj] = mk;
      if (before && !mk) sLast[jj] |= static_cast<uint32_t>((k + 1) & 1) << 8;
      if (mk) sActive = 1;  // benign race: every writer stores 1
      if (blockIdx.x == 0)
        for (int o = 0; o < MORAP_MAX_RHS; ++o) nextClear[jj * MORAP_MAX_RHS + o] = 0ull;
    }
    __syncthreads();
    if (trace && tid == 0) trace[3] = global_ns();
    if (!sActive) break;
  }
  // final values of every RHS: xi[K_j & 1] -> buf[o][sweeps_o & 1] (this CTA's states)
  {
    int jl = jBase;
    for (int li = tid; li < nloc; li += blockDim.x) {
      const long long i = i0 + li;
      while (i >= A.statePrefix[jl + 1]) ++jl;
      const EvalJob& J = A.jobs[jl];
      const int sl = static_cast<int>(i - A.statePrefix[jl]);
      const uint32_t par = sLast[jl];
      const double* src = IA.xi + (static_cast<size_t>(par >> 8 & 1u) * total + i) * R;
      for (int o = 0; o < J.nrhs; ++o) J.buf[o][par >> o & 1u][sl] = src[o];
    }
  }
  if (blockIdx.x == 0) {
    if (tid == 0) A.ctl->sweepsDone = k + 1;
    for (int jj = tid; jj < A.njobs; jj += blockDim.x) A.mask[jj] = 0u;
    atomicAdd(&A.ctl->bytes, bytesAcc);
    atomicAdd(&A.ctl->backups, backupsAcc);
  }
}
