// Host side of the upload: tiling, successor windows, compact streams, validation.
// Included by morap_cuda.cu inside its anonymous namespace (one translation unit: the
// kernels, their launch code and the C ABI share these definitions).

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
  std::vector<int32_t> outSucc;               // out-of-window successors, in transition order
};

// The sweep streams of a compact model, tile-major: each tile's slice of every stream
// starts on a 16-byte boundary (padded), so one bulk copy per stream lands at offset 0 of
// its stage region. u16 window offsets succW = succ - wlo inside the tile's x window
// (outside: bit 15 set and j = the model's j-th out-of-window transition, outSucc[j], in
// bits 0-14 and 24-31 -- allIn tiles have none, so their words keep bits 24-31 clear), u16
// ends relative to the tile, allIn / simple flags per tile.
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
  c.outSucc.clear();
  for (size_t t = 0; t < nt; ++t) {
    TileDesc& d = desc[t];
    const TileDesc& e = desc[t + 1];
    if (d.fits)  // the successors outside the window, in transition order (the sweep reads
                 // them through outSucc instead of the full succ array)
      for (int k = d.k0; k < e.k0; ++k)
        if (static_cast<unsigned>(v.succ[k] - d.wlo) >= static_cast<unsigned>(d.wn)) c.outSucc.push_back(v.succ[k]);
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
  if (c.outSucc.size() >= (1u << 23)) c.ok = false;  // the transition word indexes outSucc with 23 bits
}

void fill_streams(const morap_csr_view& v, const std::vector<TileDesc>& desc, const CompactStream& c, uint32_t* stW,
                  uint32_t* rowW, uint32_t* trW) {
  const size_t nt = desc.size() - 1;
  unsigned j = 0;  // out-of-window transitions of the model so far (< 2^23, checked at layout)
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
        uint32_t word = o;
        if (o >= static_cast<unsigned>(d.wn)) {  // the model's j-th out-of-window transition
          word = 0x8000u | (j & 0x7FFFu) | ((j >> 15) << 24);
          ++j;
        }
        trW[z++] = word | (static_cast<uint32_t>(c.idx[k]) << 16);
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
