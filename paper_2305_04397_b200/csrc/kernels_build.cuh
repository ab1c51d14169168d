// Device product builder: the products of (agent, task) pairs built straight
// into device memory in the lean compact layout the sweeps read -- buildProduct
// (model.hpp:230-321), checkRewardFinite (model.hpp:163-206) and the host upload preparation
// (upload_prep.cuh: tiles, successor windows, compact streams, out-of-window lists) on the GPU.
// Included by morap_cuda.cu inside its anonymous namespace.
//
// One CTA builds one product at a time (persistent CTAs, two per SM, claim products from a
// counter), with every intermediate array in a per-CTA global workspace:
//   BFS       level-synchronous. The reference numbers product states in FIFO discovery order
//             (model.hpp:262-300); level by level that order is "by the first discovering edge",
//             edges ordered by (state, row, transition): pass A takes atomicMin of the edge index
//             per undiscovered (agent state, location) slot, pass B numbers the slots whose
//             minimum is the edge itself with a block scan in edge order, pass C writes the
//             level's successors. The edges of the level are the product's transitions in order,
//             so the CSR falls out of the same passes.
//   rows      rowOffset / trnOffset / done / reward-class candidates from the discovery order.
//   alphabet  first-occurrence order of the probabilities (per transition) and reward tuples
//             (per row) -- the dictionaries build_compact records in insertion order.
//   finite    the maximal avoid set as a parallel worklist over reverse edges (the same greatest
//             fixpoint as the sequential stack of maximalAvoidSet).
//   tiles     make_tiles' greedy packing by one warp (32 x 8 candidate ends per step; the
//             conditions are monotone, so the count of admissible ends is the tile's length),
//             then successor_window / layout_streams per tile, one warp per tile.
//   write     (mode 1) every array of the model, A then B, into its slot of the arena.
// Mode 0 ("measure") stops before the write and reports sizes, reward finiteness and an
// identity hash; the host deduplicates on those and builds only the distinct products.

#ifndef MORAP_BUILD_THREADS
#define MORAP_BUILD_THREADS 512
#endif
constexpr int kBT = MORAP_BUILD_THREADS;  // builder CTA threads (two CTAs per SM: A/B in DESIGN.md §9)
constexpr int kBuildCtasPerSm = 1024 / kBT;
constexpr int kBW = kBT / 32;
constexpr int kBuildMaxCand = 1024; // distinct probabilities / costs over all agents

struct BAgent {
  int32_t S, R, nnz, initial;
  const int32_t* row;    // S + 1
  const int32_t* trn;    // R + 1
  const int32_t* succ;   // nnz
  const int32_t* pcand;  // nnz: index into the probability alphabet
  const int32_t* ccand;  // R: index into the cost alphabet
  const int32_t* name;   // R: action-name id (identity hash)
  const int32_t* lset;   // S: label-set id
};

struct BTask {
  int32_t Q, L, initial, pad;
  const int32_t* delta;   // Q x L
  const uint8_t* flags;   // Q: 1 accepting, 2 trap, 4 pre-sink
  const int32_t* letter;  // per label-set id
};

struct BuildOut {
  int32_t status, S, R, nnz, rewardFinite, ntiles, maxRowNnz, nOutGrp, needB, nDict, nClass, pad;
  unsigned long long hash, bytes;
  DevModel dm;
};

struct BuildArgs {
  const BAgent* agents;
  const BTask* tasks;
  const int32_t* pairs;  // (agent, task) per product
  int npairs;
  const double* probs;  // probability alphabet (exact bit patterns; contains 1.0)
  const double* costs;  // cost alphabet
  int nProbs, nCosts, probOne, internalName;
  int mode;             // 0 measure, 1 write
  char* ws;
  size_t wsBytes;       // per CTA
  int32_t SQmax, Smax, Rmax, Nmax, SAmax, Tmax;  // workspace bounds (Tmax: tiles)
  char* arena;
  const unsigned long long* offsets;  // mode 1: arena offset of each product
  BuildOut* out;
  int* next;
};

struct BuildWs {
  int32_t *id, *minE, *let, *as, *qs, *eb, *ro, *to, *succ, *head, *fillc, *rev, *owner, *leaving, *closed, *F1, *F2,
      *tileStart, *grpCnt, *tileGrp, *bins;
  uint16_t *pc, *rcls;
  uint8_t *pidx, *done, *inF;
  TileDesc* desc;
  int4* tcnt;   // per tile: padded state / row / transition words, out-of-window transitions
  int4* tbase;  // their exclusive prefixes
  int32_t* outIdx;
};

__host__ __device__ constexpr int kBinsPerWarp(int Smax) { return Smax / 64 + 2; }

// Carves one CTA's workspace (base == nullptr: just the size).
__host__ __device__ inline size_t build_ws_layout(char* base, int SQ, int S, int R, int N, int SA, int T,
                                                  BuildWs* W) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off += (bytes + 255) / 256 * 256;
    return p;
  };
  BuildWs w;
  w.id = reinterpret_cast<int32_t*>(take(4ull * SQ));
  w.minE = reinterpret_cast<int32_t*>(take(4ull * SQ));
  w.let = reinterpret_cast<int32_t*>(take(4ull * SA));
  w.as = reinterpret_cast<int32_t*>(take(4ull * S));
  w.qs = reinterpret_cast<int32_t*>(take(4ull * S));
  w.eb = reinterpret_cast<int32_t*>(take(4ull * (S + 1)));
  w.ro = reinterpret_cast<int32_t*>(take(4ull * (S + 1)));
  w.to = reinterpret_cast<int32_t*>(take(4ull * (R + 1)));
  w.succ = reinterpret_cast<int32_t*>(take(4ull * N));
  w.pc = reinterpret_cast<uint16_t*>(take(2ull * N));
  w.pidx = reinterpret_cast<uint8_t*>(take(1ull * N));
  w.rcls = reinterpret_cast<uint16_t*>(take(2ull * R));
  w.done = reinterpret_cast<uint8_t*>(take(1ull * S));
  w.inF = reinterpret_cast<uint8_t*>(take(1ull * S));
  w.head = reinterpret_cast<int32_t*>(take(4ull * (S + 2)));
  w.fillc = reinterpret_cast<int32_t*>(take(4ull * S));
  w.rev = reinterpret_cast<int32_t*>(take(4ull * N));
  w.owner = reinterpret_cast<int32_t*>(take(4ull * R));
  w.leaving = reinterpret_cast<int32_t*>(take(4ull * R));
  w.closed = reinterpret_cast<int32_t*>(take(4ull * S));
  w.F1 = reinterpret_cast<int32_t*>(take(4ull * S));
  w.F2 = reinterpret_cast<int32_t*>(take(4ull * S));
  w.tileStart = reinterpret_cast<int32_t*>(take(4ull * (T + 1)));
  w.desc = reinterpret_cast<TileDesc*>(take(sizeof(TileDesc) * (T + 1ull)));
  w.tcnt = reinterpret_cast<int4*>(take(sizeof(int4) * (T + 1ull)));
  w.tbase = reinterpret_cast<int4*>(take(sizeof(int4) * (T + 1ull)));
  w.grpCnt = reinterpret_cast<int32_t*>(take(4ull * (T + 1)));
  w.outIdx = reinterpret_cast<int32_t*>(take(4ull * (T + 1)));
  w.tileGrp = reinterpret_cast<int32_t*>(take(4ull * kMaxOutGroups * T));
  w.bins = reinterpret_cast<int32_t*>(take(4ull * kBW * kBinsPerWarp(S)));
  if (W) *W = w;
  return off;
}

// ---- block primitives (every thread of the CTA calls them) ----------------------------
__device__ __forceinline__ int bscan_excl(int v, int* sh, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    sh[lane] = w;
  }
  __syncthreads();
  const int excl = x - v + (wid ? sh[wid - 1] : 0);
  total = sh[kBW - 1];
  __syncthreads();
  return excl;
}

__device__ __forceinline__ int breduce_max(int v, int* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  int r = sh[0];
  for (int i = 1; i < kBW; ++i) r = max(r, sh[i]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ int breduce_sum(int v, int* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  int r = 0;
  for (int i = 0; i < kBW; ++i) r += sh[i];
  __syncthreads();
  return r;
}

__device__ __forceinline__ unsigned long long breduce_sum64(unsigned long long v, unsigned long long* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  unsigned long long r = 0;
  for (int i = 0; i < kBW; ++i) r += sh[i];
  __syncthreads();
  return r;
}

// identity hash term: (array tag, index, value) -> 64 bits; the product hash is their sum
__device__ __forceinline__ unsigned long long hterm(unsigned tag, unsigned long long i, unsigned long long v) {
  unsigned long long z = v + 0x9e3779b97f4a7c15ull * (i + 1) + (static_cast<unsigned long long>(tag) << 58);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned long long dbits(double d) {
  return static_cast<unsigned long long>(__double_as_longlong(d));
}

__device__ __forceinline__ size_t up256(size_t n) { return (n + 255) / 256 * 256; }

// The maximal avoid set of a product in the workspace (model.cpp maximalAvoidSet): reverse
// edges by counting sort, then the removal worklist in parallel rounds. True iff it is empty.
__device__ bool build_reward_finite(const BuildWs& W, int S, int* sh, int& sCount, int& sCount2) {
  const int tid = threadIdx.x;
  for (int x = tid; x < S + 2; x += kBT) W.head[x] = 0;
  for (int x = tid; x < S; x += kBT) {
    W.inF[x] = W.done[x] ? 0 : 1;
    W.fillc[x] = 0;
  }
  if (tid == 0) {
    sCount = 0;
    sCount2 = 0;
  }
  __syncthreads();
  int inCount = 0;
  for (int x = tid; x < S; x += kBT) {
    if (!W.inF[x]) continue;
    ++inCount;
    int closed = 0;
    for (int r = W.ro[x]; r < W.ro[x + 1]; ++r) {
      W.owner[r] = x;
      int lv = 0;
      for (int k = W.to[r]; k < W.to[r + 1]; ++k) {
        const int t = W.succ[k];
        atomicAdd(&W.head[t + 1], 1);
        lv += W.inF[t] ? 0 : 1;
      }
      W.leaving[r] = lv;
      closed += lv == 0 ? 1 : 0;
    }
    W.closed[x] = closed;
  }
  inCount = breduce_sum(inCount, sh);
  {
    int run = 0;
    for (int base = 0; base <= S; base += kBT) {  // head[t] = first reverse edge of t
      const int x = base + tid;
      const int v = x <= S ? W.head[x + 1] : 0;
      int tot;
      const int ex = run + bscan_excl(v, sh, tot);
      if (x <= S) W.head[x] = ex;
      run += tot;
    }
  }
  __syncthreads();
  for (int x = tid; x < S; x += kBT) {
    if (!W.inF[x]) continue;
    for (int r = W.ro[x]; r < W.ro[x + 1]; ++r)
      for (int k = W.to[r]; k < W.to[r + 1]; ++k) {
        const int t = W.succ[k];
        W.rev[W.head[t] + atomicAdd(&W.fillc[t], 1)] = r;
      }
    if (W.closed[x] == 0) W.F1[atomicAdd(&sCount, 1)] = x;
  }
  __syncthreads();
  int removed = 0;
  {
    int* F = W.F1;
    int* G = W.F2;
    int nF = sCount;
    __syncthreads();
    while (nF > 0) {
      removed += nF;
      if (tid == 0) sCount2 = 0;
      __syncthreads();
      for (int i = tid; i < nF; i += kBT) {
        const int s = F[i];
        for (int e = W.head[s]; e < W.head[s + 1]; ++e) {
          const int r = W.rev[e];
          const int o = W.owner[r];
          if (atomicAdd(&W.leaving[r], 1) == 0 && atomicSub(&W.closed[o], 1) == 1) G[atomicAdd(&sCount2, 1)] = o;
        }
      }
      __syncthreads();
      nF = sCount2;
      int* tmp = F;
      F = G;
      G = tmp;
      __syncthreads();
    }
  }
  return removed == inCount;
}

__global__ void __launch_bounds__(kBT, kBuildCtasPerSm) k_build_products(BuildArgs A) {
  __shared__ int sh[kBW];
  __shared__ unsigned long long sh64[kBW];
  __shared__ int sFirstP[kBuildMaxCand], sFirstC[kBuildMaxCand + 1];
  __shared__ int sMapP[kBuildMaxCand], sMapC[kBuildMaxCand + 1];
  __shared__ int sProd, sCount, sCount2, sNt;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  BuildWs W;
  build_ws_layout(A.ws + blockIdx.x * A.wsBytes, A.SQmax, A.Smax, A.Rmax, A.Nmax, A.SAmax, A.Tmax, &W);
  const int binsPerWarp = kBinsPerWarp(A.Smax);

  for (;;) {
    if (tid == 0) sProd = atomicAdd(A.next, 1);
    __syncthreads();
    const int p = sProd;
    __syncthreads();
    if (p >= A.npairs) return;
    const BAgent ag = A.agents[A.pairs[2 * p]];
    const BTask tk = A.tasks[A.pairs[2 * p + 1]];
    const int SA = ag.S, Q = tk.Q, L = tk.L;
    const int SQ = SA * Q;
    BuildOut res{};
    res.status = MORAP_OK;

    // ---- BFS over (agent state, location) slots --------------------------------------
    for (int i = tid; i < SQ; i += kBT) {
      W.id[i] = -1;
      W.minE[i] = INT_MAX;
    }
    for (int s = tid; s < SA; s += kBT) W.let[s] = tk.letter[ag.lset[s]];
    for (int c = tid; c < A.nProbs; c += kBT) sFirstP[c] = INT_MAX;
    for (int c = tid; c <= A.nCosts; c += kBT) sFirstC[c] = INT_MAX;
    __syncthreads();
    if (tid == 0) {
      const int q0 = (tk.flags[tk.initial] & 4) ? tk.initial : tk.delta[tk.initial * L + W.let[ag.initial]];
      W.id[ag.initial * Q + q0] = 0;
      W.as[0] = ag.initial;
      W.qs[0] = q0;
    }
    __syncthreads();
    int fa = 0, fb = 1, ecur = 0;
    while (fa < fb) {
      int levelEdges = 0;
      for (int base = fa; base < fb; base += kBT) {  // pass A: first discovering edge per slot
        const int x = base + tid;
        int s = 0, q = 0, kb = 0, ne = 0;
        bool ps = false;
        if (x < fb) {
          s = W.as[x];
          q = W.qs[x];
          ps = (tk.flags[q] & 4) != 0;
          kb = ps ? 0 : ag.trn[ag.row[s]];
          ne = ps ? 1 : ag.trn[ag.row[s + 1]] - kb;
        }
        int tot;
        const int e0 = ecur + levelEdges + bscan_excl(ne, sh, tot);
        if (x < fb) {
          MORAP_CHECK(e0 + ne <= A.Nmax);
          W.eb[x] = e0;
          for (int i = 0; i < ne; ++i) {
            const int t = ps ? s : ag.succ[kb + i];
            const int slot = t * Q + tk.delta[q * L + W.let[t]];
            if (W.id[slot] < 0) atomicMin(&W.minE[slot], e0 + i);
          }
        }
        levelEdges += tot;
      }
      __syncthreads();
      int added = 0;
      for (int base = fa; base < fb; base += kBT) {  // pass B: number the new slots in edge order
        const int x = base + tid;
        int s = 0, q = 0, kb = 0, ne = 0, e0 = 0, cnt = 0;
        bool ps = false;
        if (x < fb) {
          s = W.as[x];
          q = W.qs[x];
          ps = (tk.flags[q] & 4) != 0;
          kb = ps ? 0 : ag.trn[ag.row[s]];
          ne = ps ? 1 : ag.trn[ag.row[s + 1]] - kb;
          e0 = W.eb[x];
          for (int i = 0; i < ne; ++i) {
            const int t = ps ? s : ag.succ[kb + i];
            const int slot = t * Q + tk.delta[q * L + W.let[t]];
            cnt += (W.id[slot] < 0 && W.minE[slot] == e0 + i) ? 1 : 0;
          }
        }
        int tot;
        int nid = fb + added + bscan_excl(cnt, sh, tot);
        if (x < fb && cnt)
          for (int i = 0; i < ne; ++i) {
            const int t = ps ? s : ag.succ[kb + i];
            const int qq = tk.delta[q * L + W.let[t]];
            const int slot = t * Q + qq;
            if (W.id[slot] < 0 && W.minE[slot] == e0 + i) {
              MORAP_CHECK(nid < A.Smax && slot < SQ);
              W.id[slot] = nid;
              W.as[nid] = t;
              W.qs[nid] = qq;
              ++nid;
            }
          }
        added += tot;
      }
      __syncthreads();
      for (int x = fa + tid; x < fb; x += kBT) {  // pass C: the level's transitions
        const int s = W.as[x], q = W.qs[x];
        const bool ps = (tk.flags[q] & 4) != 0;
        const int kb = ps ? 0 : ag.trn[ag.row[s]];
        const int ne = ps ? 1 : ag.trn[ag.row[s + 1]] - kb;
        const int e0 = W.eb[x];
        for (int i = 0; i < ne; ++i) {
          const int t = ps ? s : ag.succ[kb + i];
          W.succ[e0 + i] = W.id[t * Q + tk.delta[q * L + W.let[t]]];
          const int c = ps ? A.probOne : ag.pcand[kb + i];
          W.pc[e0 + i] = static_cast<uint16_t>(c);
          atomicMin(&sFirstP[c], e0 + i);
        }
      }
      ecur += levelEdges;
      fa = fb;
      fb += added;
      __syncthreads();
    }
    const int S = fb, nnz = ecur;
    if (tid == 0) W.eb[S] = nnz;

    // ---- rows ---------------------------------------------------------------------------
    int rcur = 0;
    for (int base = 0; base < S; base += kBT) {
      const int x = base + tid;
      int rc = 0;
      if (x < S) {
        const int s = W.as[x];
        rc = (tk.flags[W.qs[x]] & 4) ? 1 : ag.row[s + 1] - ag.row[s];
      }
      int tot;
      const int r0 = rcur + bscan_excl(rc, sh, tot);
      if (x < S) W.ro[x] = r0;
      rcur += tot;
    }
    const int R = rcur;
    if (tid == 0) {
      W.ro[S] = R;
      W.to[R] = nnz;
    }
    unsigned long long h = 0;
    int maxRow = 0;
    for (int x = tid; x < S; x += kBT) {
      const int s = W.as[x], q = W.qs[x];
      const uint8_t f = tk.flags[q];
      const bool ps = (f & 4) != 0;
      const int r0 = W.ro[x], e0 = W.eb[x];
      MORAP_CHECK(r0 + (ps ? 1 : ag.row[s + 1] - ag.row[s]) <= A.Rmax);
      W.done[x] = (f & 3) ? 1 : 0;
      h += hterm(1, x, (static_cast<unsigned long long>(r0) << 32) | static_cast<unsigned>(e0));
      h += hterm(2, x, f & 7);
      if (ps) {
        W.to[r0] = e0;
        W.rcls[r0] = static_cast<uint16_t>(A.nCosts);
        atomicMin(&sFirstC[A.nCosts], r0);
        h += hterm(3, r0, A.internalName);
        maxRow = max(maxRow, 1);
      } else {
        const int ar0 = ag.row[s], ar1 = ag.row[s + 1], k0 = ag.trn[ar0];
        for (int ar = ar0; ar < ar1; ++ar) {
          const int r = r0 + ar - ar0;
          W.to[r] = e0 + ag.trn[ar] - k0;
          const int c = ag.ccand[ar];
          W.rcls[r] = static_cast<uint16_t>(c);
          atomicMin(&sFirstC[c], r);
          h += hterm(3, r, ag.name[ar]);
          maxRow = max(maxRow, ag.trn[ar + 1] - ag.trn[ar]);
        }
      }
    }
    __syncthreads();

    // ---- alphabets in first-occurrence order (build_compact's insertion order) -----------
    int nDict = 0, nClass = 0;
    {
      int used = 0;
      for (int c = tid; c < A.nProbs; c += kBT) {
        const int f = sFirstP[c];
        int rank = -1;
        if (f != INT_MAX) {
          rank = 0;
          for (int d = 0; d < A.nProbs; ++d) rank += sFirstP[d] < f ? 1 : 0;
          ++used;
        }
        sMapP[c] = rank;
      }
      nDict = breduce_sum(used, sh);
      used = 0;
      for (int c = tid; c <= A.nCosts; c += kBT) {
        const int f = sFirstC[c];
        int rank = -1;
        if (f != INT_MAX) {
          rank = 0;
          for (int d = 0; d <= A.nCosts; ++d) rank += sFirstC[d] < f ? 1 : 0;
          ++used;
        }
        sMapC[c] = rank;
      }
      nClass = breduce_sum(used, sh);
    }
    // the hash sees the values in their dictionaries (candidate ids are call-local)
    for (int c = tid; c < A.nProbs; c += kBT)
      if (sMapP[c] >= 0) h += hterm(5, sMapP[c], dbits(A.probs[c]));
    for (int c = tid; c <= A.nCosts; c += kBT)
      if (sMapC[c] >= 0) h += hterm(6, sMapC[c], c < A.nCosts ? dbits(A.costs[c]) : 0x1ull);
    for (int k = tid; k < nnz; k += kBT) {
      W.pidx[k] = static_cast<uint8_t>(sMapP[W.pc[k]]);
      h += hterm(4, k, (static_cast<unsigned long long>(W.succ[k]) << 32) | W.pidx[k]);
    }
    for (int r = tid; r < R; r += kBT) {
      W.rcls[r] = static_cast<uint16_t>(sMapC[W.rcls[r]]);
      h += hterm(8, r, (static_cast<unsigned long long>(W.to[r]) << 32) | W.rcls[r]);
    }
    maxRow = breduce_max(maxRow, sh);

    // ---- reward finiteness: the maximal avoid set (model.cpp maximalAvoidSet) ------------
    // (measure pass only: the write pass builds products the host accepted as reward-finite)
    res.rewardFinite = A.mode == 0 ? (build_reward_finite(W, S, sh, sCount, sCount2) ? 1 : 0) : 1;

    // ---- tiles (make_tiles), one warp ---------------------------------------------------
    if (wid == 0) {
      int s = 0, nt = 0;
      if (lane == 0) W.tileStart[0] = 0;
      while (s < S && nt < A.Tmax) {  // (Tmax is a bound, never reached: checked below)
        const int rs = W.ro[s], ks = W.eb[s];
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = s + 1 + lane * 8 + i;
          const bool ok = e < S && e - s < kBlock && W.ro[e + 1] - rs <= kRowCap && W.eb[e + 1] - ks <= kNnzCap;
          cnt += ok ? 1 : 0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        const int e = s + 1 + cnt;
        if (lane == 0) {
          const int rows = W.ro[e] - rs, nz = W.eb[e] - ks;
          W.desc[nt] = TileDesc{s, rs, ks, rows <= kRowCap && nz <= kNnzCap ? 1 : 0, 0, 0, 0, 0};
          W.tileStart[nt + 1] = e;
        }
        ++nt;
        s = e;
      }
      if (lane == 0) {
        W.desc[nt] = TileDesc{S, R, nnz, 0, 0, 0, 0, 0};
        sNt = s < S ? -nt : nt;
      }
    }
    __syncthreads();
    if (sNt < 0) res.status = MORAP_SIZE_GUARD;  // the tile workspace bound was wrong: no model
    const int nt = sNt < 0 ? -sNt : sNt;

    // ---- per tile: successor window, flags, out-of-window lists (warp per tile) ---------
    for (int t = wid; t < nt; t += kBW) {
      TileDesc d = W.desc[t];
      const TileDesc e = W.desc[t + 1];
      const int k0 = d.k0, k1 = e.k0;
      int wn = min(kXWin, S), wlo = 0;
      if (k1 <= k0) {
        wn = 0;
      } else {
        int lo = INT_MAX, hi = -1;
        for (int k = k0 + lane; k < k1; k += 32) {
          lo = min(lo, W.succ[k]);
          hi = max(hi, W.succ[k]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
          hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (hi - lo < wn) {
          wlo = lo & ~1;
          wn = hi - wlo + 1;
        } else {  // best run of span 64-state bins (first maximum)
          int* bins = W.bins + static_cast<size_t>(wid) * binsPerWarp;
          const int nb = (hi - lo) / 64 + 1;
          for (int i = lane; i < nb; i += 32) bins[i] = 0;
          __syncwarp();
          for (int k = k0 + lane; k < k1; k += 32) atomicAdd(&bins[(W.succ[k] - lo) / 64], 1);
          __syncwarp();
          int carry = 0;
          for (int c = 0; c < nb; c += 32) {  // in-place inclusive prefix
            const int i = c + lane;
            int v = i < nb ? bins[i] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, v, o);
              if (lane >= o) v += y;
            }
            if (i < nb) bins[i] = carry + v;
            carry += __shfl_sync(0xffffffffu, v, 31);
          }
          __syncwarp();
          const int span = max(1, wn / 64 - 1);
          int best = -1, bestI = 0;
          for (int i = lane; i < nb; i += 32) {
            const int run = bins[i] - (i >= span ? bins[i - span] : 0);
            if (run > best) {
              best = run;
              bestI = i;
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const int ob = __shfl_xor_sync(0xffffffffu, best, o), oi = __shfl_xor_sync(0xffffffffu, bestI, o);
            if (ob > best || (ob == best && oi < bestI)) {
              best = ob;
              bestI = oi;
            }
          }
          const int bestBin = max(0, bestI - span + 1);
          wlo = max(0, min(lo + bestBin * 64, S - wn)) & ~1;
          __syncwarp();
        }
      }
      d.wlo = wlo;
      d.wn = wn;
      const bool f = d.fits != 0;
      int outCnt = 0, simple = 1;
      if (f)
        for (int k = k0 + lane; k < k1; k += 32)
          outCnt += static_cast<unsigned>(W.succ[k] - wlo) >= static_cast<unsigned>(wn) ? 1 : 0;
      for (int r = d.r0 + lane; r < e.r0; r += 32) simple &= W.to[r + 1] - W.to[r] <= 2 ? 1 : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        outCnt += __shfl_xor_sync(0xffffffffu, outCnt, o);
        simple &= __shfl_xor_sync(0xffffffffu, simple, o);
      }
      d.simple = simple;
      d.allIn = f && outCnt == 0 ? 1 : 0;
      int ng = 0;
      int* grp = W.tileGrp + static_cast<size_t>(t) * kMaxOutGroups;
      if (!f) {
        ng = -1;
      } else if (outCnt) {  // sorted distinct stamp groups, by repeated minimum
        int last = -1;
        for (;;) {
          int m = INT_MAX;
          for (int k = k0 + lane; k < k1; k += 32) {
            const int sk = W.succ[k];
            if (static_cast<unsigned>(sk - wlo) >= static_cast<unsigned>(wn) && (sk >> 5) > last) m = min(m, sk >> 5);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
          if (m == INT_MAX) break;
          if (ng == kMaxOutGroups) {
            ng = -1;
            break;
          }
          if (lane == 0) grp[ng] = m;
          ++ng;
          last = m;
        }
      }
      const int ns = f ? e.s0 - d.s0 : 0, nr = f ? e.r0 - d.r0 : 0, nz = f ? k1 - k0 : 0;
      if (lane == 0) {
        W.desc[t] = d;
        W.tcnt[t] = make_int4((ns + 3) & ~3, (nr + 3) & ~3, (nz + 3) & ~3, outCnt);
        W.grpCnt[t] = ng < 0 ? 1 : ng;
        if (ng < 0) grp[0] = -1;
      }
    }
    __syncthreads();
    int4 tot4 = make_int4(0, 0, 0, 0);
    int nOutGrp = 0, fitsAll = 1;
    for (int base = 0; base < nt; base += kBT) {  // slice positions, outSucc bases, outIdx
      const int t = base + tid;
      const int4 c = t < nt ? W.tcnt[t] : make_int4(0, 0, 0, 0);
      const int g = t < nt ? W.grpCnt[t] : 0;
      if (t < nt && !W.desc[t].fits) fitsAll = 0;
      int a, b, z, o, gg;
      const int ea = bscan_excl(c.x, sh, a), eb = bscan_excl(c.y, sh, b), ez = bscan_excl(c.z, sh, z),
                eo = bscan_excl(c.w, sh, o), eg = bscan_excl(g, sh, gg);
      if (t < nt) {
        W.tbase[t] = make_int4(tot4.x + ea, tot4.y + eb, tot4.z + ez, tot4.w + eo);
        W.outIdx[t] = nOutGrp + eg;
      }
      tot4.x += a;
      tot4.y += b;
      tot4.z += z;
      tot4.w += o;
      nOutGrp += gg;
    }
    if (tid == 0) W.outIdx[nt] = nOutGrp;
    fitsAll = breduce_sum(fitsAll ? 0 : 1, sh) == 0 ? 1 : 0;
    const int nStW = tot4.x, nRowW = tot4.y, nTrW = tot4.z, nOutSucc = tot4.w;
    const int nclassT = nClass ? nClass : 1;  // build_compact: an empty table becomes K zeros

    // hash of the remaining identity fields; sizes of the model block (A then B)
    h += hterm(7, 0, static_cast<unsigned long long>(S) << 32 | static_cast<unsigned>(R));
    h += hterm(7, 1, static_cast<unsigned long long>(nnz));
    h = breduce_sum64(h, sh64);
    const size_t lenA = up256(4ull * (nt + 1)) + up256(sizeof(TileDesc) * (nt + 1ull)) + up256(8ull * nDict) +
                        up256(16ull * nclassT) + up256(4ull * nStW) + up256(4ull * nRowW) + up256(4ull * nTrW) +
                        up256(sizeof(TilePos) * static_cast<size_t>(nt)) + up256(4ull * (nt + 1)) +
                        up256(4ull * nOutGrp) + up256(4ull * nOutSucc);
    const size_t lenB = up256(4ull * (S + 1)) + up256(4ull * (R + 1)) + up256(4ull * nnz) + up256(1ull * S) +
                        up256(1ull * nnz) + up256(2ull * R);
    if (nDict > 256 || nClass > kMaxClasses || nOutSucc >= (1 << 23)) res.status = MORAP_INVALID_CONFIG;
    res.S = S;
    res.R = R;
    res.nnz = nnz;
    res.ntiles = nt;
    res.maxRowNnz = maxRow;
    res.nOutGrp = nOutGrp;
    res.needB = fitsAll ? 0 : 1;
    res.nDict = nDict;
    res.nClass = nclassT;
    res.hash = h;
    res.bytes = lenA + lenB;

    if (A.mode == 1 && res.status == MORAP_OK) {
      // ---- write the model block --------------------------------------------------------
      char* cur = A.arena + A.offsets[p];
      auto put = [&](size_t bytes) {
        char* at = cur;
        cur += up256(bytes);
        return at;
      };
      DevModel dm{};
      int32_t* tileStart = reinterpret_cast<int32_t*>(put(4ull * (nt + 1)));
      TileDesc* tiles = reinterpret_cast<TileDesc*>(put(sizeof(TileDesc) * (nt + 1ull)));
      double* dict = reinterpret_cast<double*>(put(8ull * nDict));
      double* table = reinterpret_cast<double*>(put(16ull * nclassT));
      uint32_t* stW = reinterpret_cast<uint32_t*>(put(4ull * nStW));
      uint32_t* rowW = reinterpret_cast<uint32_t*>(put(4ull * nRowW));
      uint32_t* trW = reinterpret_cast<uint32_t*>(put(4ull * nTrW));
      TilePos* pos = reinterpret_cast<TilePos*>(put(sizeof(TilePos) * static_cast<size_t>(nt)));
      int32_t* outIdx = reinterpret_cast<int32_t*>(put(4ull * (nt + 1)));
      int32_t* outGrp = reinterpret_cast<int32_t*>(put(4ull * nOutGrp));
      int32_t* outSucc = reinterpret_cast<int32_t*>(put(4ull * nOutSucc));
      int32_t* ro = reinterpret_cast<int32_t*>(put(4ull * (S + 1)));
      int32_t* to = reinterpret_cast<int32_t*>(put(4ull * (R + 1)));
      int32_t* succ = reinterpret_cast<int32_t*>(put(4ull * nnz));
      uint8_t* done = reinterpret_cast<uint8_t*>(put(1ull * S));
      uint8_t* pidx = reinterpret_cast<uint8_t*>(put(1ull * nnz));
      uint16_t* rcls = reinterpret_cast<uint16_t*>(put(2ull * R));
      for (int x = tid; x <= S; x += kBT) ro[x] = W.ro[x];
      for (int r = tid; r <= R; r += kBT) to[r] = W.to[r];
      for (int k = tid; k < nnz; k += kBT) {
        succ[k] = W.succ[k];
        pidx[k] = W.pidx[k];
      }
      for (int x = tid; x < S; x += kBT) done[x] = W.done[x];
      for (int r = tid; r < R; r += kBT) rcls[r] = W.rcls[r];
      for (int t = tid; t <= nt; t += kBT) {
        tileStart[t] = W.tileStart[t];
        tiles[t] = W.desc[t];
        outIdx[t] = W.outIdx[t];
        if (t < nt) {
          const int4 b = W.tbase[t];
          pos[t] = TilePos{b.x, b.y, b.z, 0};
          const int g0 = W.outIdx[t], ng = W.grpCnt[t];
          for (int i = 0; i < ng; ++i) outGrp[g0 + i] = W.tileGrp[static_cast<size_t>(t) * kMaxOutGroups + i];
        }
      }
      for (int c = tid; c < A.nProbs; c += kBT)
        if (sMapP[c] >= 0) dict[sMapP[c]] = A.probs[c];
      for (int c = tid; c <= A.nCosts; c += kBT)
        if (sMapC[c] >= 0) {
          table[2 * sMapC[c]] = c < A.nCosts ? A.costs[c] : 0.0;
          table[2 * sMapC[c] + 1] = c < A.nCosts ? 0.0 : 1.0;
        }
      if (nClass == 0 && tid < 2) table[tid] = 0.0;
      for (int t = wid; t < nt; t += kBW) {  // the sweep streams (fill_streams), warp per tile
        const TileDesc d = W.desc[t], e = W.desc[t + 1];
        const int4 b = W.tbase[t], c = W.tcnt[t];
        const bool f = d.fits != 0;
        const int ns = f ? e.s0 - d.s0 : 0, nr = f ? e.r0 - d.r0 : 0, nz = f ? e.k0 - d.k0 : 0;
        for (int i = lane; i < c.x; i += 32) {
          uint32_t w = 0u;
          if (i < ns) {
            const int q = d.s0 + i;
            w = static_cast<uint32_t>(W.ro[q + 1] - d.r0) | (static_cast<uint32_t>(W.eb[q + 1] - d.k0) << 10) |
                (W.done[q] ? 1u << 21 : 0u);
          }
          stW[b.x + i] = w;
        }
        for (int i = lane; i < c.y; i += 32)
          rowW[b.y + i] = i < nr ? static_cast<uint32_t>(W.to[d.r0 + i + 1] - d.k0) |
                                       (static_cast<uint32_t>(W.rcls[d.r0 + i]) << 11)
                                 : 0u;
        int j = b.w;  // the model's out-of-window transitions so far
        for (int i0 = 0; i0 < c.z; i0 += 32) {
          const int i = i0 + lane;
          uint32_t w = 0xFFFFu;
          bool out = false;
          int sk = 0;
          if (i < nz) {
            sk = W.succ[d.k0 + i];
            const unsigned o = static_cast<unsigned>(sk - d.wlo);
            out = o >= static_cast<unsigned>(d.wn);
            w = o;
          }
          const unsigned m = __ballot_sync(0xffffffffu, out);
          if (out) {
            const unsigned jj = static_cast<unsigned>(j + __popc(m & ((1u << lane) - 1u)));
            w = 0x8000u | (jj & 0x7FFFu) | ((jj >> 15) << 24);
            outSucc[jj] = sk;
          }
          if (i < nz) w |= static_cast<uint32_t>(W.pidx[d.k0 + i]) << 16;
          if (i < c.z) trW[b.z + i] = w;
          j += __popc(m);
        }
      }
      dm.rowOffset = ro;
      dm.trnOffset = to;
      dm.succ = succ;
      dm.done = done;
      dm.tiles = tiles;
      dm.tileStart = tileStart;
      dm.probIdx = pidx;
      dm.probDict = dict;
      dm.rclass = rcls;
      dm.classTable = table;
      dm.stW = stW;
      dm.rowW = rowW;
      dm.trW = trW;
      dm.outSucc = outSucc;
      dm.tilePos = pos;
      dm.outIdx = outIdx;
      dm.outGrp = outGrp;
      dm.S = S;
      dm.R = R;
      dm.nnz = nnz;
      dm.initial = 0;
      dm.ntiles = nt;
      dm.K = 2;
      dm.rewardFinite = res.rewardFinite;
      dm.compact = 1;
      dm.nclass = nclassT;
      dm.nOutSucc = nOutSucc;
      dm.nDict = nDict;
      dm.nStW = nStW;
      dm.nRowW = nRowW;
      dm.nTrW = nTrW;
      dm.bytesPerSweep = 4ull * nnz + 4ull * R + 20ull * S;
      dm.bytesPerEval = 0;  // set on the host (the same formula as pack_models)
      res.dm = dm;
    }
    __syncthreads();
    if (tid == 0) A.out[p] = res;
  }
}
