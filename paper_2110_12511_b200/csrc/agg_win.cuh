// agg_win.cuh — tier-2 wedge aggregation for starts with more partners than a
// CTA hash table holds (kCtaCap).  One CTA per start (or per window group of a
// start when a batch has few starts).
//
// Partner ids are processed one coarse id WINDOW (kWinIds ids) at a time; this
// replaces the paper's per-thread n-element wedge array, which on
// B200 would be an HBM array with one random atomic per wedge.
//   * sparse window: a shared-memory bitmap records first occurrences (one
//     atomicOr per wedge) and a repeat table counts the partners seen again;
//     repeats are emitted with w = 1 + repeats;
//   * dense window (many entries, or repeats overflowing the table): packed
//     counters (2..32 bits, the smallest width that holds the start's list
//     count) over sub-windows; fields with a count >= 2 are emitted.
// Lists are sorted, so each list's part of a window is one contiguous segment.
// For starts with up to win_pre lists the segment bounds of every window, the
// list bases and per-window chunk prefixes are computed once per start into
// per-CTA scratch; a window's segments are cut into chunks that warps take
// dynamically (coalesced 16-byte loads).  Starts with more lists search their
// segments window by window.
#pragma once
// (included inside namespace pbng by kernels_cd.cuh, after agg_mid.cuh)

#ifndef PBNG_WIN_LOG_IDS
#define PBNG_WIN_LOG_IDS 20
#endif
#ifndef PBNG_WIN_MAX_W
#define PBNG_WIN_MAX_W 64
#endif
#ifndef PBNG_WIN_THREADS
#define PBNG_WIN_THREADS 1024
#endif
#ifndef PBNG_WIN_CTAS
#define PBNG_WIN_CTAS 1
#endif
#ifndef PBNG_WIN_LOG_DUP
#define PBNG_WIN_LOG_DUP 13
#endif
constexpr uint32_t kWinThreads = PBNG_WIN_THREADS;
constexpr uint32_t kWinCtas = PBNG_WIN_CTAS;           // resident CTAs per SM
constexpr uint32_t kWinLists = PBNG_WIN_THREADS;       // lists per batch (bounds precomputed when the start has <= this many)
constexpr uint64_t kWinIds = 1ull << PBNG_WIN_LOG_IDS;  // ids per window
constexpr uint32_t kWinBitWords = (uint32_t)(kWinIds / 32);
constexpr uint32_t kWinLogDup = PBNG_WIN_LOG_DUP;
constexpr uint32_t kWinDupSlots = 1u << kWinLogDup;   // repeat table (key << 32 | repeats)
constexpr uint32_t kWinDupCap = kWinDupSlots / 2;
#ifndef PBNG_WIN_CHUNK
#define PBNG_WIN_CHUNK 256
#endif
#ifndef PBNG_SEG_DEPTH
#define PBNG_SEG_DEPTH 2
#endif
constexpr int kSegDepth = PBNG_SEG_DEPTH;  // 16-byte loads per lane issued together
#ifndef PBNG_DENSE_DEPTH
#define PBNG_DENSE_DEPTH 4
#endif
constexpr int kDenseDepth = PBNG_DENSE_DEPTH;
#ifndef PBNG_WIN_FAST
#define PBNG_WIN_FAST 1
#endif
#ifndef PBNG_COMBINE
#define PBNG_COMBINE 0
#endif
#ifndef PBNG_COMBINE_DENSE
#define PBNG_COMBINE_DENSE 0
#endif
#ifndef PBNG_DENSE_CHUNK
#define PBNG_DENSE_CHUNK 1024
#endif
#ifndef PBNG_DENSE_TOUCH
#define PBNG_DENSE_TOUCH 0
#endif
constexpr uint32_t kWinChunk = PBNG_WIN_CHUNK ? PBNG_WIN_CHUNK : 512;  // entries per warp task
static_assert(kWinChunk % 4 == 0 && PBNG_DENSE_CHUNK % 4 == 0, "chunks are cut at 16-byte aligned positions");

// bitmap windows with many entries use 256-entry chunks read two 16-byte loads
// per lane at a time (more bytes in flight); smaller ones 128-entry chunks
#ifndef PBNG_BIG_WIN
#define PBNG_BIG_WIN (~0ull)  // off: 256-entry chunks measured no better overall (config 4 worse)
#endif
__device__ __forceinline__ uint32_t bitmap_chunk(unsigned long long entries) {
  return entries >= PBNG_BIG_WIN ? 2 * kWinChunk : kWinChunk;
}

// chunk size for a window of `entries` entries (PBNG_WIN_CHUNK = 0: about two
// chunks per warp, 128..1024; else fixed)
__device__ __forceinline__ uint32_t win_chunk(unsigned long long entries) {
  if (PBNG_WIN_CHUNK) return PBNG_WIN_CHUNK;
  unsigned long long c = (entries / 64 + 127) & ~127ull;
  return c < 128 ? 128u : (c > 1024 ? 1024u : (uint32_t)c);
}

struct WinSmem {
  uint32_t bits[kWinBitWords];           // 128 KB bitmap of the window
  unsigned long long dup[kWinDupSlots];  // 64 KB repeat table (key << 32 | repeats)
  uint16_t dslot[kWinDupCap];            // filled slots of the repeat table
  uint32_t cpre[kWinLists + 1];       // exclusive prefix of chunk counts of the batch
  uint32_t segS[kWinLists];           // segment [segS, segT) of each list of the batch
  uint32_t segT[kWinLists];
  unsigned long long segB[kWinLists]; // partner-array base of each list of the batch
  uint32_t scan[33];
  unsigned long long ek[PBNG_WIN_MAX_W];  // entries per coarse window (relative to the first window, kWinMaxW)
  uint32_t ctot[PBNG_WIN_MAX_W];          // chunks per coarse window (fast path)
};

struct WinShared {
  uint32_t over, ndup, next, t;
  unsigned long long acc;
};

__device__ __forceinline__ void win_dup_insert(WinSmem& S, WinShared& sh, uint32_t k) {
  uint32_t h = (k * 0x9E3779B1u) >> (32 - kWinLogDup);
  const unsigned long long mine = ((unsigned long long)k << 32) | 1ull;
  for (uint32_t probe = 0;; probe++) {
    unsigned long long cur = ((volatile unsigned long long*)S.dup)[h];
    if ((uint32_t)(cur >> 32) == k) {
      atomicAdd(reinterpret_cast<uint32_t*>(&S.dup[h]), 1u);
      return;
    }
    if (cur == kEmptySlot) {
      cur = atomicCAS(&S.dup[h], kEmptySlot, mine);
      if (cur == kEmptySlot) {
        const uint32_t i = atomicAdd(&sh.ndup, 1u);
        if (i < kWinDupCap) S.dslot[i] = (uint16_t)h;
        else sh.over = 1;
        return;
      }
      if ((uint32_t)(cur >> 32) == k) {
        atomicAdd(reinterpret_cast<uint32_t*>(&S.dup[h]), 1u);
        return;
      }
    }
    if (probe >= kDupProbe) {
      sh.over = 1;
      return;
    }
    h = (h + 1) & (kWinDupSlots - 1);
  }
}

__device__ __forceinline__ uint32_t win_dup_lookup(const WinSmem& S, uint32_t k) {
  uint32_t h = (k * 0x9E3779B1u) >> (32 - kWinLogDup);
  for (uint32_t probe = 0; probe <= kDupProbe + 1; probe++) {
    const unsigned long long cur = S.dup[h];
    if ((uint32_t)(cur >> 32) == k) return (uint32_t)cur;
    if (cur == kEmptySlot) return 0;
    h = (h + 1) & (kWinDupSlots - 1);
  }
  return 0;
}

// first index in p[lo, hi) with p[i] >= key
__device__ __forceinline__ uint32_t lb_range(const uint32_t* __restrict__ p, uint32_t lo, uint32_t hi, uint32_t key) {
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Visit the entries p[i0, i1) with a whole warp: fn(ok, x) is called
// warp-convergently (ok = the lane holds an entry).  The 16-byte aligned body is
// read 512 entries per step, four independent 16-byte loads per lane issued
// before any entry is used, so each warp keeps 2 KB of loads in flight.
template <int D = kSegDepth, class Fn>
__device__ __forceinline__ void seg_visit(const uint32_t* __restrict__ p, uint64_t i0, uint64_t i1, Fn& fn) {
  const uint32_t ln = lane_id();
  uint64_t h = (i0 + 3) & ~3ull;  // first 16-byte aligned index
  if (h > i1) h = i1;
  {
    const bool ok = i0 + ln < h;
    fn(ok, ok ? p[i0 + ln] : 0u);
  }
  const uint64_t t = h + ((i1 - h) & ~3ull);  // end of the aligned body
  for (uint64_t q0 = h; q0 < t; q0 += 128 * D) {
    uint4 v[D];
    bool ok[D];
#pragma unroll
    for (int j = 0; j < D; j++) {
      const uint64_t q = q0 + 128 * j + 4 * ln;
      ok[j] = q < t;
      v[j] = ok[j] ? __ldg(reinterpret_cast<const uint4*>(p + q)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < D; j++) {
      fn(ok[j], v[j].x);
      fn(ok[j], v[j].y);
      fn(ok[j], v[j].z);
      fn(ok[j], v[j].w);
    }
  }
  {
    const bool ok = t + ln < i1;
    fn(ok, ok ? p[t + ln] : 0u);
  }
}

// Mark the entries p[i0, i1) (all inside the window starting at `a`) in the
// bitmap; repeats go to the table.
// Lanes of one warp step hold distinct ids of one sorted list, so in dense
// id ranges several lanes hit the same word: with PBNG_COMBINE the lanes of a
// word are grouped (match_any), their bits / increments combined and one lane
// issues the atomic, instead of the shared-memory unit serialising them.
template <int D = 1>
__device__ __forceinline__ void win_mark(const uint32_t* __restrict__ p, uint64_t i0, uint64_t i1, uint32_t a,
                                         uint32_t skip, WinSmem& S, WinShared& sh) {
  const uint32_t ln = lane_id();
  auto one = [&](bool ok, uint32_t x) {
    const bool act = ok && x != skip;
    const uint32_t o = x - a;
    PBNG_DCHECK(!act || o < kWinIds);  // the entry lies in the window
    const uint32_t bit = 1u << (o & 31);
    if (PBNG_COMBINE) {
      const uint32_t wd = act ? o >> 5 : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(kFull, wd);
      const uint32_t leader = __ffs(peers) - 1;
      const uint32_t orv = __reduce_or_sync(peers, act ? bit : 0u);
      uint32_t old = 0;
      if (act && ln == leader) old = atomicOr(&S.bits[wd], orv);
      old = __shfl_sync(peers, old, leader);
      if (act && (old & bit)) win_dup_insert(S, sh, x);
    } else if (act) {
      if (atomicOr(&S.bits[o >> 5], bit) & bit) win_dup_insert(S, sh, x);
    }
  };
  seg_visit<D>(p, i0, i1, one);
}

// Zero the first nwords words of the window array with 16-byte stores (whole CTA).
__device__ __forceinline__ void win_clear(uint32_t* bits, uint32_t nwords) {
  uint4* b4 = reinterpret_cast<uint4*>(bits);
  const uint32_t n4 = (nwords + 3) >> 2;  // the array holds a multiple of 4 words
  for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x) b4[i] = make_uint4(0, 0, 0, 0);
}

// Σ repeats of the entries p[i0, i1) (pass 2 of vertex-priority counting)
__device__ __forceinline__ unsigned long long win_sum(const uint32_t* __restrict__ p, uint64_t i0, uint64_t i1,
                                                      uint32_t skip, const WinSmem& S) {
  unsigned long long cs = 0;
  for (uint64_t q = i0 + lane_id(); q < i1; q += 32) {
    const uint32_t x = p[q];
    if (x != skip) cs += win_dup_lookup(S, x);
  }
  return warp_sum(cs);
}

// One pass over the segments in [a, b) of every list (coarse window k): the
// segments are cut into chunks of kWinChunk entries that warps take
// dynamically; fn(i0, i1, e) is called by a whole warp for the partner
// entries [i0, i1) of list e.  Returns whether any entry was visited.
template <class L, class Fn>
__device__ __forceinline__ bool win_pass(const L& lists, uint64_t e0, uint64_t nl, bool pre,
                                         const uint32_t* __restrict__ bnd, uint32_t W, uint32_t k, uint64_t wa,
                                         uint64_t wb, uint64_t a, uint64_t b, const uint32_t* __restrict__ partner,
                                         WinSmem& S, WinShared& sh, Fn& fn, uint32_t chunk = kWinChunk,
                                         const uint32_t* __restrict__ sub = nullptr, uint32_t sj = 0,
                                         uint32_t sstride = 0, unsigned long long* pc = nullptr,
                                         const unsigned long long* __restrict__ gb = nullptr) {
  // gb (optional, with sub): the list bases the start's tables already hold (one load
  // instead of the three dependent ones of lists.get, in a phase where one warp works)
  // sub (optional): precomputed bounds of list i's sub-window sj at sub[i * sstride + sj]
  const uint32_t tid = threadIdx.x, ln = lane_id();
  bool any = false;
  for (uint64_t bs = 0; bs < nl; bs += kWinLists) {
    const uint32_t nb = (uint32_t)(nl - bs < kWinLists ? nl - bs : kWinLists);
    const long long tc0 = pc ? clock64() : 0;
    uint32_t nch = 0;
    if (tid < nb) {
      const uint64_t i = bs + tid;
      uint64_t base;
      uint32_t len = 0;
      if (gb && sub) base = gb[i];
      else lists.get(e0 + i, base, len);
      const uint32_t* p = partner + base;
      uint32_t s, t;
      if (sub) {
        s = sub[i * sstride + sj];
        t = sub[i * sstride + sj + 1];
      } else if (pre) {
        const uint32_t c0 = bnd[i * (W + 1) + k], c1 = bnd[i * (W + 1) + k + 1];
        s = a == wa ? c0 : lb_range(p, c0, c1, (uint32_t)a);
        t = b == wb ? c1 : lb_range(p, s, c1, (uint32_t)b);
      } else {
        s = lb_range(p, 0, len, (uint32_t)a);
        t = lb_range(p, s, len, (uint32_t)b);
      }
      S.segS[tid] = s;
      S.segT[tid] = t;
      S.segB[tid] = base;
      // chunks are cut at 16-byte aligned positions of the partner array (chunk is a
      // multiple of 4): only the first and last chunk of a segment have an unaligned
      // head / tail, each of which costs seg_visit a load round trip of its own
      nch = t > s ? (uint32_t)((((base + s) & 3) + (t - s) + chunk - 1) / chunk) : 0u;
    }
    uint32_t tot;
    const uint32_t cp = block_excl_scan(nch, S.scan, &tot);
    if (tid < nb) S.cpre[tid] = cp;
    if (tid == 0) {
      S.cpre[nb] = tot;
      sh.next = 0;
    }
    __syncthreads();
    any |= tot != 0;
    const long long tc1 = pc ? clock64() : 0;
    for (;;) {
      uint32_t c = 0;
      if (ln == 0) c = atomicAdd(&sh.next, 1u);
      c = __shfl_sync(kFull, c, 0);
      if (c >= tot) break;
      uint32_t lo = 0, hi = nb;  // list lo: cpre[lo] <= c < cpre[lo + 1]
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (S.cpre[mid] <= c) lo = mid; else hi = mid;
      }
      const uint64_t base = S.segB[lo];
      const uint64_t i0s = base + S.segS[lo], i1e = base + S.segT[lo];
      const uint64_t cut = (i0s & ~3ull) + (uint64_t)(c - S.cpre[lo]) * chunk;  // aligned chunk start
      fn(cut > i0s ? cut : i0s, cut + chunk < i1e ? cut + chunk : i1e, e0 + bs + lo);
    }
    __syncthreads();
    if (pc && tid == 0) {
      atomicAdd(&pc[6], (unsigned long long)(tc1 - tc0));
      atomicAdd(&pc[7], (unsigned long long)(clock64() - tc1));
      atomicAdd(&pc[5], (unsigned long long)nb);
    }
  }
  return any;
}

// Dense sub-window: counters of `lb` = log2(bits) packed 32/bits per word; the
// field width is the smallest of 2, 4, 8, 16, 32 bits that holds the number of
// lists of the start (w counts lists, each list holds an id at most once), so a
// start with few lists counts 256K or 512K ids per pass over the 128 KB array
// (w <= number of lists).
constexpr uint32_t kDenseIds = kWinBitWords * 2;
#ifndef PBNG_DENSE_ENTRIES
#define PBNG_DENSE_ENTRIES 65536
#endif
constexpr uint64_t kDenseEntries = PBNG_DENSE_ENTRIES;  // coarse windows with more entries go dense
constexpr uint32_t kWinMaxW = PBNG_WIN_MAX_W;  // windows whose entry counts are kept in shared memory

// Dense marking: one atomicAdd per wedge; the first increment of a word
// appends the word to the touched list (kept in the repeat table's memory,
// which dense mode does not use), so the sweep visits touched words only.
constexpr uint32_t kTouchCap = kWinDupSlots * 2;
// dense sweep: queued hit words per warp; the queues take the shared memory from the
// repeat table up to the segment tables, all scratch that is refilled before its next use
constexpr uint32_t kSweepQ = (uint32_t)((offsetof(WinSmem, scan) - offsetof(WinSmem, dup)) / 8) / (kWinThreads / 32);
static_assert(kSweepQ >= 64 && offsetof(WinSmem, dup) % 8 == 0, "dense sweep queue: a warp appends up to 64 words between drains");
__device__ __forceinline__ uint32_t dense_log_bits(uint64_t nl) {
  return nl < 4 ? 1u : nl < 16 ? 2u : nl < 256 ? 3u : nl < 65536 ? 4u : 5u;  // log2 of 2..32 bits
}

__device__ __forceinline__ void dense_mark(const uint32_t* __restrict__ p, uint64_t i0, uint64_t i1, uint32_t a,
                                           uint32_t skip, uint32_t lb, uint32_t* cnt, uint32_t* touch,
                                           uint32_t* ntouch) {
  const uint32_t ln = lane_id();
  const uint32_t lf = 5 - lb;  // log2 fields per word
  auto one = [&](bool ok, uint32_t x) {
    bool fresh = false;
    uint32_t wd = 0;
    const bool act = ok && x != skip;
    const uint32_t o = x - a;
    PBNG_DCHECK(!act || (o >> lf) < kWinBitWords);  // the entry lies in the dense sub-window
    const uint32_t inc = 1u << ((o & ((1u << lf) - 1)) << lb);
    if (PBNG_COMBINE_DENSE) {
      wd = act ? o >> lf : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(kFull, wd);
      const uint32_t leader = __ffs(peers) - 1;
      const uint32_t sum = __reduce_add_sync(peers, act ? inc : 0u);  // distinct fields: no carries
      if (act && ln == leader) fresh = atomicAdd(&cnt[wd], sum) == 0u;
    } else if (!PBNG_DENSE_TOUCH) {
      if (act) atomicAdd(&cnt[o >> lf], inc);  // no touched list: the sweep reads every word
      return;
    } else if (act) {
      wd = o >> lf;
      fresh = atomicAdd(&cnt[wd], inc) == 0u;
    }
    const uint32_t m = __ballot_sync(kFull, fresh);
    if (m) {
      const uint32_t leader = __ffs(m) - 1;
      uint32_t base = 0;
      if (ln == leader) base = atomicAdd(ntouch, (uint32_t)__popc(m));
      base = __shfl_sync(kFull, base, leader);
      const uint32_t slot = base + __popc(m & lanemask_lt());
      if (fresh && slot < kTouchCap) touch[slot] = wd;
    }
  };
  seg_visit<kDenseDepth>(p, i0, i1, one);
}
__device__ __forceinline__ uint32_t dense_get(const uint32_t* cnt, uint32_t o, uint32_t lb) {
  const uint32_t lf = 5 - lb, bits = 1u << lb;
  const uint32_t v = cnt[o >> lf] >> ((o & ((1u << lf) - 1)) << lb);
  return bits == 32 ? v : v & ((1u << bits) - 1);
}

// Aggregate w(start, x) over all wedges of one start (lists e in [e0, e1),
// partner ids x < idspace, x != skip) and call emit(x, w) for every x with
// w >= 2; with Pass2, pass2(e, Σ (w - 1)) over the entries of list e (chunk-wise
// partial sums).  Whole CTA; bitmap zero and table empty on entry and exit.
// bnd: per-CTA scratch of kWinLists * (wmax + 1) entries.
// A coarse window with many entries (or whose repeats overflow the table) is
// counted densely in sub-windows instead of bitmap + repeat table.
// Only coarse windows [g * W / G, (g + 1) * W / G) are processed (a start may
// be split into G independent window groups when a batch has few starts).
template <class L, class Emit, class Pass2 = NoPass2>
__device__ __forceinline__ void win_agg_one(const L& lists, uint64_t e0, uint64_t e1, uint32_t skip,
                                            uint32_t idspace, uint32_t g, uint32_t G,
                                            const uint32_t* __restrict__ partner, WinSmem& S, WinShared& sh,
                                            uint32_t* __restrict__ bnd, uint32_t pre_lists, Emit& emit,
                                            Counters* cnt, bool prof, const Pass2& pass2 = Pass2()) {
  unsigned long long* dbg = cnt->dbg;        // path counters
  unsigned long long* prof_clk = cnt->prof;  // PBNG_TRACE phase clocks: [1] tables, [2] bitmap, [3] dense
  const uint32_t tid = threadIdx.x, bd = blockDim.x, ln = lane_id(), wid = tid >> 5, nw = bd >> 5;
  const uint64_t nl = e1 - e0;
  // id range [lo, hi) of this unit: whole coarse windows when the start is split
  // into at most as many groups as it has windows, else equal id ranges (small
  // batches of heavy starts, so that every SM has work)
  uint64_t lo, hi;
  {
    const uint32_t Wall = (uint32_t)(((uint64_t)idspace + kWinIds - 1) / kWinIds);
    if (G <= Wall) {
      lo = (uint64_t)g * Wall / G * kWinIds;
      hi = (uint64_t)(g + 1) * Wall / G * kWinIds;
    } else {
      const uint64_t span = (((uint64_t)idspace + G - 1) / G + 31) & ~31ull;
      lo = (uint64_t)g * span;
      hi = lo + span;
    }
    lo = lo < idspace ? lo : idspace;
    hi = hi < idspace ? hi : idspace;
  }
  if (lo >= hi) return;
  // windows k in [0, W): ids [lo + k * kWinIds, min(lo + (k + 1) * kWinIds, hi))
  const uint32_t W = (uint32_t)((hi - lo + kWinIds - 1) / kWinIds);
  const uint32_t k0 = 0, k1 = W;
  // fast path: every list's window bounds, base and per-window chunk prefixes
  // are computed once per start (per-CTA scratch), so a window needs no scan
  const uint32_t PL = pre_lists;  // scratch stride (lists) of the precomputed tables
  const bool pre = nl <= PL && k1 - k0 <= kWinMaxW;
  const uint32_t lb = dense_log_bits(nl);                 // dense counter width 2^lb bits
  const uint32_t SW = kWinBitWords << (5 - lb);           // ids per dense pass
  const uint32_t W1 = W + 1;
  uint32_t* cpg = bnd + (uint64_t)PL * W1;  // [kr * PL + i]
  unsigned long long* gbase = reinterpret_cast<unsigned long long*>(cpg + (uint64_t)PL * W1);
  const long long tp0 = clock64();
  for (uint32_t k = tid; k < kWinMaxW; k += bd) S.ek[k] = 0;
  __syncthreads();
  if (pre) {
    // bnd[i * (W + 1) + k] = first entry of list i with id >= min(lo + k * kWinIds, hi)
    for (uint32_t i = wid; i < nl; i += nw) {
      uint64_t base;
      uint32_t len;
      lists.get(e0 + i, base, len);
      if (ln == 0) gbase[i] = base;
      if (len <= 32) {
        // short list: one coalesced load, every bound by a ballot count
        const uint32_t x = ln < len ? partner[base + ln] : 0xFFFFFFFFu;
        uint32_t prev = 0;
        for (uint32_t k = k0; k <= k1; k++) {
          const uint64_t key = lo + (uint64_t)k * kWinIds;
          const uint32_t kk = key < hi ? (uint32_t)key : (uint32_t)hi;
          const uint32_t v = __popc(__ballot_sync(kFull, x < kk));
          if (ln == 0) {
            bnd[(uint64_t)i * W1 + k] = v;
            if (k > k0 && v > prev) atomicAdd(&S.ek[k - 1 - k0], (unsigned long long)(v - prev));
          }
          prev = v;
        }
        continue;
      }
      uint32_t prev = 0;
      for (uint32_t kb = k0; kb <= k1; kb += 32) {
        const uint32_t k = kb + ln;
        uint32_t v = 0;
        if (k <= k1) {
          const uint64_t key = lo + (uint64_t)k * kWinIds;
          v = lb_range(partner + base, 0, len, key < hi ? (uint32_t)key : (uint32_t)hi);
          bnd[(uint64_t)i * W1 + k] = v;
        }
        uint32_t left = __shfl_up_sync(kFull, v, 1);
        if (ln == 0) left = prev;
        if (k > k0 && k <= k1 && v > left) atomicAdd(&S.ek[k - 1 - k0], (unsigned long long)(v - left));
        prev = __shfl_sync(kFull, v, 31);
      }
    }
    __syncthreads();
    if (nl <= 32) {
      // few lists: one warp scans every window's chunk counts (no CTA barriers)
      if (wid == 0) {
        for (uint32_t k = k0; k < k1; k++) {
          const uint32_t ch = bitmap_chunk(S.ek[k - k0]);
          const uint32_t nch = ln < nl ? (bnd[(uint64_t)ln * W1 + k + 1] - bnd[(uint64_t)ln * W1 + k] +
                                          ch - 1) / ch : 0u;
          uint32_t incl = nch;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (ln >= (uint32_t)o) incl += y;
          }
          if (ln < nl) cpg[(uint64_t)(k - k0) * PL + ln] = incl - nch;
          if (ln == 31) S.ctot[k - k0] = incl;
        }
      }
    } else
    for (uint32_t k = k0; k < k1; k++) {
      uint32_t carry = 0;
      for (uint32_t t0 = 0; t0 < nl; t0 += bd) {
        const uint32_t i = t0 + tid;
        uint32_t nch = 0;
        const uint32_t ch = bitmap_chunk(S.ek[k - k0]);
        if (i < nl) nch = (bnd[(uint64_t)i * W1 + k + 1] - bnd[(uint64_t)i * W1 + k] + ch - 1) / ch;
        uint32_t tot;
        const uint32_t cp = block_excl_scan(nch, S.scan, &tot);
        if (i < nl) cpg[(uint64_t)(k - k0) * PL + i] = carry + cp;
        carry += tot;
      }
      if (tid == 0) S.ctot[k - k0] = carry;
    }
  }
  __syncthreads();
  if (prof && tid == 0) atomicAdd(&prof_clk[1], (unsigned long long)(clock64() - tp0));
  for (uint32_t k = k0; k < k1; k++) {
    const uint64_t wa = lo + (uint64_t)k * kWinIds;
    const uint64_t wb = wa + kWinIds < hi ? wa + kWinIds : hi;
    const uint32_t kr = k - k0;
    bool dense = pre && S.ek[kr] > kDenseEntries;
    if (pre && S.ek[kr] == 0) continue;
    if (!dense && pre && PBNG_WIN_FAST) {
      // ---- fast path: bitmap + repeat table, chunks statically split over warps
      if (tid == 0) {
        sh.over = 0;
        sh.ndup = 0;
        sh.next = 0;
      }
      const uint32_t tot = S.ctot[kr];
      const uint32_t* cp = cpg + (uint64_t)kr * PL;
      const bool insm = nl <= kWinLists;  // the row fits shared memory
      if (insm)
        for (uint32_t i = tid; i < nl; i += bd) S.cpre[i] = cp[i];
      const uint32_t* crow = insm ? S.cpre : cp;
      const uint32_t wch = bitmap_chunk(S.ek[kr]);
      __syncthreads();
      // warps take chunks dynamically; chunk c belongs to the largest list i with cpre[i] <= c
      auto run = [&](auto&& fn) {
        for (;;) {
          uint32_t c = 0;
          if (ln == 0) c = atomicAdd(&sh.next, 1u);
          c = __shfl_sync(kFull, c, 0);
          if (c >= tot) break;
          uint32_t lo = 0, hi = (uint32_t)nl;
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (crow[mid] <= c) lo = mid; else hi = mid;
          }
          const uint64_t sbeg = gbase[lo] + bnd[(uint64_t)lo * W1 + k], send = gbase[lo] + bnd[(uint64_t)lo * W1 + k + 1];
          const uint64_t q0 = sbeg + (uint64_t)(c - crow[lo]) * wch;
          fn(q0, q0 + wch < send ? q0 + wch : send, e0 + lo);
        }
      };
      const long long tm0 = clock64();
      // kSegDepth 16-byte loads per lane in flight per warp step (chunk = 128 * kSegDepth entries: one step)
      if (wch > kWinChunk)
        run([&](uint64_t i0, uint64_t i1, uint64_t) { win_mark<2 * kSegDepth>(partner, i0, i1, (uint32_t)wa, skip, S, sh); });
      else
        run([&](uint64_t i0, uint64_t i1, uint64_t) { win_mark<kSegDepth>(partner, i0, i1, (uint32_t)wa, skip, S, sh); });
      __syncthreads();
      const long long tm1 = clock64();
      if (prof && tid == 0) atomicAdd(&prof_clk[2], (unsigned long long)(tm1 - tm0));
      const bool over = sh.over != 0;
      const uint32_t nd = min(sh.ndup, kWinDupCap);
      if (Pass2::kOn && !over && nd) {
        if (tid == 0) sh.next = 0;
        __syncthreads();
        run([&](uint64_t i0, uint64_t i1, uint64_t e) {
          const unsigned long long cs = win_sum(partner, i0, i1, skip, S);
          if (ln == 0 && cs) pass2(e, cs);
        });
        __syncthreads();
      }
      const uint32_t nwords = (uint32_t)((wb - wa + 31) >> 5);
      win_clear(S.bits, nwords);
      for (uint32_t i = tid; i < nd; i += bd) {
        const uint32_t sl = S.dslot[i];
        const unsigned long long v = S.dup[sl];
        S.dup[sl] = kEmptySlot;
        if (!over) emit((uint32_t)(v >> 32), (uint32_t)v + 1u);
      }
      if (tid == 0) atomicAdd(&dbg[over ? 1 : 0], 1ull);
      if (over) {
        for (uint32_t i = tid; i < kWinDupSlots; i += bd) S.dup[i] = kEmptySlot;
        dense = true;
      }
      __syncthreads();
      if (!dense) continue;
    } else if (!dense) {
      // bitmap of first occurrences + repeat table over the whole window
      if (tid == 0) {
        sh.over = 0;
        sh.ndup = 0;
      }
      __syncthreads();
      auto mark = [&](uint64_t i0, uint64_t i1, uint64_t) { win_mark(partner, i0, i1, (uint32_t)wa, skip, S, sh); };
      const uint32_t chunk = kWinChunk;
      const bool any = win_pass(lists, e0, nl, pre, bnd, W, k, wa, wb, wa, wb, partner, S, sh, mark, chunk);
      const bool over = sh.over != 0;
      const uint32_t nd = min(sh.ndup, kWinDupCap);
      if (Pass2::kOn && any && !over && nd) {
        auto sum = [&](uint64_t i0, uint64_t i1, uint64_t e) {
          const unsigned long long cs = win_sum(partner, i0, i1, skip, S);
          if (ln == 0 && cs) pass2(e, cs);
        };
        win_pass(lists, e0, nl, pre, bnd, W, k, wa, wb, wa, wb, partner, S, sh, sum, chunk);
      }
      if (any) {
        const uint32_t nwords = (uint32_t)((wb - wa + 31) >> 5);
        win_clear(S.bits, nwords);
        for (uint32_t i = tid; i < nd; i += bd) {
          const uint32_t sl = S.dslot[i];
          const unsigned long long v = S.dup[sl];
          S.dup[sl] = kEmptySlot;
          if (!over) emit((uint32_t)(v >> 32), (uint32_t)v + 1u);
        }
      }
      if (!over) {
        if (tid == 0) atomicAdd(&dbg[0], 1ull);
        __syncthreads();
        continue;
      }
      for (uint32_t i = tid; i < kWinDupSlots; i += bd) S.dup[i] = kEmptySlot;
      if (tid == 0) atomicAdd(&dbg[1], 1ull);
      __syncthreads();
    }
    // dense counting in sub-windows of SW ids; with tables, every list's
    // sub-window bounds are found at once (a warp per list, a lane per bound)
    const long long td0 = clock64();
    if (prof && tid == 0 && pre) {
      atomicAdd(&cnt->prof3[3], S.ek[kr]);
      atomicAdd(&cnt->prof3[4], 1ull);
    }
    const uint32_t NS = (uint32_t)((wb - wa + SW - 1) / SW);
    uint32_t* sub = nullptr;
    if (pre && NS <= 32) {
      sub = reinterpret_cast<uint32_t*>(gbase + PL);  // PL * 33 entries
      for (uint32_t i = wid; i < nl; i += nw) {
        const uint32_t c0 = bnd[(uint64_t)i * W1 + k], c1 = bnd[(uint64_t)i * W1 + k + 1];
        const uint32_t* p = partner + gbase[i];
        for (uint32_t j = ln; j <= NS; j += 32) {
          const uint64_t key = wa + (uint64_t)j * SW;
          sub[(uint64_t)i * 33 + j] = j == 0 ? c0 : (key >= wb ? c1 : lb_range(p, c0, c1, (uint32_t)key));
        }
      }
      __syncthreads();
      if (prof && tid == 0) atomicAdd(&cnt->prof3[0], (unsigned long long)(clock64() - td0));
    }
    for (uint64_t a = wa; a < wb; a += SW) {
      const uint32_t sj = (uint32_t)((a - wa) / SW);
      const uint64_t b = a + SW < wb ? a + SW : wb;
      uint32_t* touch = reinterpret_cast<uint32_t*>(S.dup);
      if (tid == 0) sh.ndup = 0;  // touched-word count
      const uint32_t fpw = 1u << (5 - lb);  // fields per word
      const uint32_t nwords = (uint32_t)((b - a + fpw - 1) / fpw);
      // Replicas: when the sub-window's counters fill only part of the array
      // (late partitions: a few hundred live ids, millions of wedges per start),
      // warps count into R copies (warp w into copy w mod R) so that they do not
      // serialise on the same shared words; the sweep adds the copies (field-wise:
      // every copy's field is at most the total, which the field width holds).
      const uint32_t stride = (nwords + 3) & ~3u;
      uint32_t R = 1;
      if (!Pass2::kOn && !PBNG_DENSE_TOUCH)
        while (2 * R <= 32 && 2 * R * stride <= kWinBitWords) R *= 2;
      uint32_t* mycnt = S.bits + (wid & (R - 1)) * stride;
      __syncthreads();
      auto mark = [&](uint64_t i0, uint64_t i1, uint64_t) {
        dense_mark(partner, i0, i1, (uint32_t)a, skip, lb, mycnt, touch, &sh.ndup);
      };
      const uint32_t chunk = PBNG_DENSE_CHUNK ? PBNG_DENSE_CHUNK : (pre ? win_chunk(S.ek[kr] * SW / kWinIds) : kWinChunk);
      const long long tq0 = prof ? clock64() : 0;
      const bool any = win_pass(lists, e0, nl, pre, bnd, W, k, wa, wb, a, b, partner, S, sh, mark, chunk, sub, sj, 33,
                                prof ? cnt->prof3 : nullptr, sub ? gbase : nullptr);
      const long long tq1 = prof ? clock64() : 0;
      if (prof && tid == 0) atomicAdd(&cnt->prof3[1], (unsigned long long)(tq1 - tq0));
      if (!any) continue;
      if (Pass2::kOn) {
        auto sum = [&](uint64_t i0, uint64_t i1, uint64_t e) {
          unsigned long long cs = 0;
          for (uint64_t q = i0 + ln; q < i1; q += 32) {
            const uint32_t x = partner[q];
            if (x != skip) cs += dense_get(S.bits, x - (uint32_t)a, lb) - 1u;
          }
          cs = warp_sum(cs);
          if (ln == 0 && cs) pass2(e, cs);
        };
        win_pass(lists, e0, nl, pre, bnd, W, k, wa, wb, a, b, partner, S, sh, sum, chunk, sub, sj, 33);
      }
      const uint32_t nt = sh.ndup;
      const bool listed = PBNG_DENSE_TOUCH && nt <= kTouchCap;
      // fields with count >= 2 have a bit above their lowest bit set: find them
      // with one mask per word and visit only those
      const uint32_t bits = 1u << lb;
      const uint32_t fmask = bits == 32 ? 0xFFFFFFFFu : (1u << bits) - 1;
      const uint32_t lows = lb == 1 ? 0x55555555u : lb == 2 ? 0x11111111u : lb == 3 ? 0x01010101u
                          : lb == 4 ? 0x00010001u : 0x00000001u;
      auto sweep_word = [&](uint32_t i, uint32_t v) {
        uint32_t m = v & ~lows;
        while (m) {
          const uint32_t f = (uint32_t)(__ffs(m) - 1) >> lb;
          emit((uint32_t)a + i * fpw + f, (v >> (f << lb)) & fmask);
          m &= ~(fmask << (f << lb));
        }
      };
      if (listed) {
        for (uint32_t t = tid; t < nt; t += bd) {
          const uint32_t i = touch[t];
          const uint32_t v = S.bits[i];
          if (v) {
            S.bits[i] = 0;
            sweep_word(i, v);
          }
        }
      } else {
        // Words holding a field >= 2 are rare (a few percent), so emitting straight
        // from the scan leaves one or two lanes of a warp active per emit (measured:
        // the sweep took 36% of the dense cycles, issue-bound on that divergence).
        // Each warp instead queues its hit words (ballot-compacted, kSweepQ) and
        // drains the queue a word per lane.
        uint4* b4 = reinterpret_cast<uint4*>(S.bits);
        uint2* q = reinterpret_cast<uint2*>(S.dup) + wid * kSweepQ;
        uint32_t nq = 0;
        const uint32_t n4 = (nwords + 3) >> 2;
        auto drain = [&]() {
          __syncwarp();
          for (uint32_t i = ln; i < nq; i += 32) {
            const uint2 e = q[i];
            sweep_word(e.x, e.y);
          }
          nq = 0;
          __syncwarp();
        };
        for (uint32_t t0 = wid * 32; t0 < n4; t0 += bd) {
          const uint32_t t = t0 + ln;
          uint4 v = make_uint4(0, 0, 0, 0);
          if (t < n4) {
            v = b4[t];
            for (uint32_t r = 1; r < R; r++) {
              const uint4 y = b4[r * (stride >> 2) + t];
              if (y.x | y.y | y.z | y.w) {
                b4[r * (stride >> 2) + t] = make_uint4(0, 0, 0, 0);
                v.x += y.x;
                v.y += y.y;
                v.z += y.z;
                v.w += y.w;
              }
            }
            if (v.x | v.y | v.z | v.w) b4[t] = make_uint4(0, 0, 0, 0);
          }
          const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (uint32_t c = 0; c < 4; c++) {
            if ((c & 1) == 0 && nq > kSweepQ - 64) drain();
            const bool hit = (vv[c] & ~lows) != 0;
            const uint32_t hm = __ballot_sync(kFull, hit);
            if (hit) q[nq + __popc(hm & lanemask_lt())] = make_uint2(4 * t + c, vv[c]);
            nq += __popc(hm);
          }
        }
        drain();
      }
      if (tid == 0) atomicAdd(&dbg[2], 1ull);
      __syncthreads();
      if (prof && tid == 0) atomicAdd(&cnt->prof3[2], (unsigned long long)(clock64() - tq1));
    }
    // the repeat table's memory held touched words: empty it again
    for (uint32_t i = tid; i < kWinDupSlots; i += bd) S.dup[i] = kEmptySlot;
    __syncthreads();
    if (prof && tid == 0) atomicAdd(&prof_clk[3], (unsigned long long)(clock64() - td0));
  }
}

template <int MODE>
__global__ void __launch_bounds__(kWinThreads, kWinCtas) k_agg_win(AggArgs a) {
  extern __shared__ __align__(16) unsigned char wsm[];
  WinSmem& S = *reinterpret_cast<WinSmem*>(wsm);
  __shared__ WinShared sh;
  for (uint32_t i = threadIdx.x; i < kWinBitWords; i += blockDim.x) S.bits[i] = 0;
  for (uint32_t i = threadIdx.x; i < kWinDupSlots; i += blockDim.x) S.dup[i] = kEmptySlot;
  uint32_t* bnd = a.win_bnd + (uint64_t)blockIdx.x * a.win_cap;
  const uint32_t G = a.win_split;
  const uint64_t n = (uint64_t)*a.count * G;
  const auto L = agg_lists<MODE>(a);
  unsigned long long upd = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      sh.t = atomicAdd(a.ticket, 1u);
      sh.acc = 0;
    }
    __syncthreads();
    const uint32_t t = sh.t;
    if (t >= n) break;
    const uint32_t u = a.list[t / G].x;
    uint64_t acc = 0;
    auto out = [&](uint32_t k, uint32_t w) { emit<MODE>(a, u, k, w, acc, upd); };
    const long long ts0 = clock64();
    win_agg_one(L, a.offU[u], a.offU[u + 1], u, MODE == 2 ? u : a.idspace, t % G, G, a.adjV, S, sh, bnd, a.win_pre, out, a.c,
                a.win_prof);
    if (a.win_prof && threadIdx.x == 0) {
      const bool tab = a.offU[u + 1] - a.offU[u] <= a.win_pre;
      atomicAdd(tab ? &a.c->prof[0] : &a.c->prof2[0], (unsigned long long)(clock64() - ts0));
      atomicAdd(tab ? &a.c->prof2[2] : &a.c->prof2[1], 1ull);
    }
    if (MODE == 0) {
      acc = warp_sum(acc);
      if (lane_id() == 0 && acc) atomicAdd(&sh.acc, (unsigned long long)acc);
      __syncthreads();
      if (threadIdx.x == 0 && sh.acc) red_add_u64(&a.support[u], sh.acc);  // support zeroed by the caller
    }
    __syncthreads();
  }
  if (MODE == 1) flush_updates(a, upd);
}

// List-split mode (CD peel) for small batches of heavy starts over a small live
// id range: the late CD partitions hold the densest core — a few hundred to a
// few thousand live vertices, each start with 10^5-10^6 lists of which only a
// handful of entries are live — where a CTA per start (or per id range) spends
// its time walking list descriptors one CTA at a time.  Here a unit is (start,
// list range j of G): the CTA counts w(start, x) over its lists into shared
// counters over the ids [0, range) (32-bit, one per id; R per-warp copies when
// the range is small), adds them to the start's global counters gcnt[s][x], and
// the unit that finishes last (per-start ticket, threadfence pattern) sweeps
// gcnt[s] and emits C(w,2) for w >= 2.  Every live partner id is
// below `range` (= 1 + largest live id); stale entries above it are skipped.
template <int MODE>
__global__ void __launch_bounds__(kWinThreads, kWinCtas) k_agg_lsplit(AggArgs a, uint32_t range, uint32_t* gcnt,
                                                                      uint32_t* done) {
  extern __shared__ __align__(16) unsigned char wsm[];
  WinSmem& S = *reinterpret_cast<WinSmem*>(wsm);
  __shared__ WinShared sh;
  __shared__ uint32_t s_last;
  const uint32_t tid = threadIdx.x, bd = blockDim.x, wid = tid >> 5, nw = bd >> 5;
  const uint32_t G = a.win_split;
  const uint64_t n = (uint64_t)*a.count * G;
  const auto L = agg_lists<MODE>(a);
  const uint32_t stride = (range + 3) & ~3u;
  PBNG_DCHECK(stride <= kWinBitWords);
  uint32_t R = 1;
  while (2 * R <= nw && 2 * R * stride <= kWinBitWords) R *= 2;
  for (uint32_t i = tid; i < R * stride; i += bd) S.bits[i] = 0u;
  uint32_t* my = S.bits + (wid & (R - 1)) * stride;
  unsigned long long upd = 0;
  for (;;) {
    if (tid == 0) sh.t = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const uint32_t t = sh.t;
    if (t >= n) break;
    const uint32_t si = t / G, j = t % G;
    const uint32_t u = a.list[si].x;
    const uint64_t e0 = a.offU[u], d = a.offU[u + 1] - e0;
    const uint64_t l0 = e0 + d * j / G, l1 = e0 + d * (j + 1) / G;
    auto f = [&](bool ok, uint32_t x, uint64_t) {
      if (ok && x != u && x < range) atomicAdd(&my[x], 1u);
    };
    // lists in chunks of blockDim (a warp per 32 lists, short lists flattened
    // over the lanes); lists of >= blockDim entries are walked by the whole CTA
    // (in the dense core a start's few thousand lists each hold most live ids)
    cta_wedges(L, l0, l1, a.adjV, S.segS, &sh.ndup, f);
    __syncthreads();
    uint32_t* g = gcnt + (uint64_t)si * stride;
    for (uint32_t i = tid; i < range; i += bd) {
      uint32_t v = 0;
      for (uint32_t r = 0; r < R; r++) {
        v += S.bits[r * stride + i];
        S.bits[r * stride + i] = 0u;
      }
      if (v) atomicAdd(&g[i], v);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&done[si], 1u) == G - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      uint64_t acc = 0;
      for (uint32_t i = tid; i < range; i += bd) {
        const uint32_t w = __ldcg(&g[i]);
        if (w >= 2) emit<MODE>(a, u, i, w, acc, upd);
      }
    }
    __syncthreads();
  }
  if (MODE == 1) flush_updates(a, upd);
}
