// agg_hash.cuh — CTA-tier wedge aggregation in packed shared-memory hash
// tables over degree-mass windows of the partner ids.
//
// For one start s (a frontier vertex in CD, or a count start) the wedges
// s -> v -> x are aggregated into w(s, x) = number of s's lists holding x, and
// C(w,2) is emitted for w >= 2 (CD batch update P:987-991).  The
// paper keeps a private n-element wedge array per thread; here a
// CTA keeps a hash table of packed 32-bit slots
//     slot = (x + 1) << cb | w        (0 = empty, w < 2^cb)
// in shared memory, so one insert is one atomicCAS (a first occurrence) or a
// CAS plus an atomicAdd (a repeat).  w counts lists and a list holds x at most
// once, so w <= d_s; starts are routed here only when d_s < 2^cb, hence the
// count field never carries into the key.
//
// A start whose entries exceed the table's capacity is split by partner id
// into GROUPS of consecutive windows.  The 32 windows are fixed once per
// decomposition with equal edge mass (window k = ids [wb[k], wb[k+1]) with
// wb[k] = first id whose CSR offset reaches k·m/32; ids are ranks by
// decreasing degree, so a list's entries spread about evenly over the
// windows).  The bounds of every list in every window come from a row
// table kept for lists longer than kRowMin (refreshed when the list is
// compacted) or, for short lists, from ballots over the list itself, so no
// per-start binary search is needed.  Windows are grouped greedily up to the
// capacity; the table is swept (emit + clear) once per group, and its size
// follows the group's entries, so a start costs O(entries) and never a pass
// over the id space.  A start with a single window above capacity is passed
// on to the windowed-bitmap tier (agg_win.cuh) before any of its work is done.
#pragma once
// (included inside namespace pbng by kernels_cd.cuh, after agg_win.cuh)

#ifndef PBNG_HASH_SLOTS
#define PBNG_HASH_SLOTS 10240
#endif
#ifndef PBNG_HASH_FILTER_LOG
#define PBNG_HASH_FILTER_LOG 16
#endif
#ifndef PBNG_HASH_FILTER
#define PBNG_HASH_FILTER 1
#endif
#ifndef PBNG_HASH_THREADS
#define PBNG_HASH_THREADS 384
#endif
#ifndef PBNG_HASH_CTAS
#define PBNG_HASH_CTAS 3
#endif
#ifndef PBNG_HASH_MAX_PB
#define PBNG_HASH_MAX_PB (1u << 17)
#endif
constexpr uint32_t kHashSlots = PBNG_HASH_SLOTS;        // 40 KB table per CTA, 3 CTAs per SM
constexpr uint32_t kHashThreads = PBNG_HASH_THREADS;
constexpr uint32_t kHashCtas = PBNG_HASH_CTAS;          // resident CTAs per SM
constexpr uint32_t kHashCap = kHashSlots / 2;           // entries per group (distinct partners <= entries): load <= 1/2
constexpr uint32_t kHashLists = 128;                    // lists per start (d_s < kHashLists)
constexpr uint32_t kHashMaxPb = PBNG_HASH_MAX_PB;       // classify: larger starts go to the bitmap tier
constexpr uint32_t kHW = 32;                            // degree-mass windows
constexpr uint32_t kRowMin = 64;                        // lists with more entries keep a window-bound row
constexpr uint32_t kHashChunk = 128;                    // positions per warp step (4 per lane)
#ifndef PBNG_HASH_BDEPTH
#define PBNG_HASH_BDEPTH 2
#endif
constexpr int kHashBDepth = PBNG_HASH_BDEPTH;           // phase B: 16-byte loads per lane per chunk
constexpr uint32_t kFiltLog = PBNG_HASH_FILTER_LOG;     // membership filter: 2^kFiltLog bits (8 KB)
constexpr uint32_t kFiltWords = 1u << (kFiltLog - 5);

struct HashSmem {
  uint32_t tab[kHashSlots];
  uint32_t filt[kFiltWords];             // one bit per inserted partner (hash-addressed), see hash_lookup_inc
  unsigned long long lbase[kHashLists];  // partner-array base of list i
  uint32_t llen[kHashLists];             // entries of list i
  uint32_t bnd[kHashLists][kHW + 1];     // first entry of list i in window k (bnd[i][kHW] = llen[i])
  uint32_t pre[kHashLists + 1];          // exclusive prefix of the current group's segment lengths
  uint32_t seg0[kHashLists];             // first entry of list i in the current group
  uint32_t ek[kHW];                      // entries per window
  uint32_t gk[kHW + 1];                  // group g = windows [gk[g], gk[g + 1])
  uint32_t wb[kHW + 1];                  // window id boundaries
  uint32_t ng, demote, t, tot, next, hl, hlen;
  unsigned long long acc;
};

// The table is probed in buckets of 4 slots (one 16-byte shared load): a
// partner already present is found with one load and counted with one
// atomicAdd; a new one takes the bucket's first empty slot with one atomicCAS.
// At load <= 1/2 a bucket overflows rarely, so warps do not wait on long
// linear-probing chains (the first version, one CAS per slot probed, spent
// ~7 probe rounds per warp insert step at load 2/3).
__device__ __forceinline__ bool hash_count(uint32_t* tab, uint32_t TB, uint32_t cb, uint32_t x) {
  const uint32_t kx = x + 1u, key = kx << cb;
  uint32_t b = __umulhi(x * 0x9E3779B1u, TB);
  const uint4* tab4 = reinterpret_cast<const uint4*>(tab);
  for (uint32_t probes = 0;; probes++) {
    PBNG_DCHECK(probes <= TB);  // load <= 1/2: a free slot always exists
    const uint4 q = tab4[b];
    const uint32_t v[4] = {q.x, q.y, q.z, q.w};
    int hit = -1, emp = -1;
#pragma unroll
    for (int j = 3; j >= 0; j--) {
      if ((v[j] >> cb) == kx) hit = j;
      if (v[j] == 0u) emp = j;
    }
    if (hit >= 0) {
      atomicAdd(&tab[4 * b + hit], 1u);
      return false;
    }
    if (emp >= 0) {
      const uint32_t old = atomicCAS(&tab[4 * b + emp], 0u, key | 1u);
      if (old == 0u) return true;
      if ((old >> cb) == kx) {
        atomicAdd(&tab[4 * b + emp], 1u);
        return false;
      }
      continue;  // the slot went to another partner: look at the bucket again
    }
    if (++b == TB) b = 0;
  }
}

// Membership filter of the table's keys: bit filt_bit(x) is set when x is
// inserted, so a lookup of a partner that is not in the table (on power-law
// graphs almost every entry of the largest list H) costs one shared load and
// no probe loop.  The ncu source view of the first version (no filter) put
// 93% of k_agg_hash's instructions in H's probe loop: 32 lanes probing in
// lockstep walk ~2.9 buckets per lookup at load 1/2 (one lane's collision
// stalls the warp).
__device__ __forceinline__ uint32_t filt_bit(uint32_t x) { return (x * 0x85EBCA6Bu) >> (32 - kFiltLog); }
__device__ __forceinline__ void filt_set(uint32_t* filt, uint32_t x) {
  const uint32_t f = filt_bit(x);
  atomicOr(&filt[f >> 5], 1u << (f & 31));
}
__device__ __forceinline__ bool filt_has(const uint32_t* filt, uint32_t x) {
  if (!PBNG_HASH_FILTER) return true;
  const uint32_t f = filt_bit(x);
  return (filt[f >> 5] >> (f & 31)) & 1u;
}

// Row table:// Row table: for every list with more than kRowMin entries (static degree),
// rows[rowid[v] * (kHW + 1) + k] = first entry of the live list with id >= wb[k]
// (k < kHW; [kHW] = live length).  One warp per list, one lane per window.
__global__ void k_rows_fill(uint32_t n, const uint32_t* __restrict__ vs, const uint32_t* __restrict__ nvs,
                            const uint32_t* __restrict__ rowid, const uint64_t* __restrict__ offV,
                            const uint32_t* __restrict__ adjL, const uint32_t* __restrict__ ld,
                            const uint32_t* __restrict__ wb, uint32_t* __restrict__ rows) {
  const uint32_t ln = lane_id();
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t cnt = vs ? *nvs : n;
  const uint32_t key = wb[ln];
  for (uint64_t i = gw; i < cnt; i += nw) {
    const uint32_t v = vs ? vs[i] : (uint32_t)i;
    const uint32_t r = rowid[v];
    if (r == 0xFFFFFFFFu) continue;
    const uint32_t* p = adjL + offV[v];
    const uint32_t L = ld[v];
    uint32_t a = 0, b = L;  // first index with p[idx] >= key
    while (a < b) {
      const uint32_t mid = (a + b) >> 1;
      if (p[mid] < key) a = mid + 1; else b = mid;
    }
    uint32_t* row = rows + (uint64_t)r * (kHW + 1);
    row[ln] = a;
    if (ln == 0) row[kHW] = L;
  }
}

// row index of every list with static degree > kRowMin (order arbitrary)
__global__ void k_rows_ids(uint32_t nV, const uint64_t* __restrict__ offV, uint32_t* __restrict__ rowid,
                           uint32_t* nrows) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nV; v += (uint64_t)gridDim.x * blockDim.x) {
    const bool big = offV[v + 1] - offV[v] > kRowMin;
    const uint32_t m = __ballot_sync(__activemask(), big);
    uint32_t base = 0;
    const uint32_t leader = __ffs(m) - 1;
    if (m && lane_id() == leader) base = atomicAdd(nrows, (uint32_t)__popc(m));
    base = __shfl_sync(__activemask(), base, leader);
    rowid[v] = big ? base + __popc(m & lanemask_lt()) : 0xFFFFFFFFu;
  }
}

// wb[k] = first id u with offU[u] >= k·m/kHW (k < kHW), wb[kHW] = 0xFFFFFFFF
__global__ void k_mass_windows(uint32_t nU, uint64_t m, const uint64_t* __restrict__ offU, uint32_t* __restrict__ wb) {
  const uint32_t k = threadIdx.x;
  if (k > kHW) return;
  if (k == kHW) {
    wb[k] = 0xFFFFFFFFu;
    return;
  }
  const uint64_t target = m * k / kHW;
  uint32_t a = 0, b = nU;
  while (a < b) {
    const uint32_t mid = (a + b) >> 1;
    if (offU[mid] < target) a = mid + 1; else b = mid;
  }
  wb[k] = a;
}

// A partner seen only in the start's LARGEST list H has w = 1 and contributes
// nothing, so H's entries never enter the table: the other lists are inserted
// first, then every entry of H only looks its partner up and counts it if
// present (one 16-byte load; no CAS, no slot taken).  On power-law graphs H is
// usually a hub list holding most of the start's entries, so the table holds
// the short lists' entries only and most entries cost a lookup.
__device__ __forceinline__ void hash_lookup_inc(uint32_t* tab, uint32_t TB, uint32_t cb, uint32_t x) {
  const uint32_t kx = x + 1u;
  uint32_t b = __umulhi(x * 0x9E3779B1u, TB);
  const uint4* tab4 = reinterpret_cast<const uint4*>(tab);
  for (;;) {
    const uint4 q = tab4[b];
    const uint32_t v[4] = {q.x, q.y, q.z, q.w};
    bool empty = false;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if ((v[j] >> cb) == kx) {
        atomicAdd(&tab[4 * b + j], 1u);
        return;
      }
      empty |= v[j] == 0u;
    }
    if (empty) return;  // inserts take the first empty slot of the probe sequence: x is absent
    if (++b == TB) b = 0;
  }
}

// Aggregate one start: lists e in [e0, e1) (fewer than kHashLists), partner ids
// x with x != skip and x < lim; emit(x, w) for w >= 2.  Returns false (nothing
// done) when some window holds more than kHashCap inserted entries.  Whole
// CTA; table empty on entry and exit.
template <class L, class Emit>
__device__ __forceinline__ bool hash_agg_one(const L& lists, uint64_t e0, uint64_t e1, uint32_t skip, uint32_t lim,
                                             const uint32_t* __restrict__ partner, const uint32_t* __restrict__ rowid,
                                             const uint32_t* __restrict__ rows, uint32_t cb, HashSmem& S,
                                             Emit& emit, unsigned long long* stat) {
  const uint32_t tid = threadIdx.x, ln = lane_id(), wid = tid >> 5, nw = blockDim.x >> 5;
  const uint32_t d = (uint32_t)(e1 - e0);
  // list descriptors
  for (uint32_t i = tid; i < d; i += blockDim.x) {
    uint64_t base;
    uint32_t len;
    lists.get(e0 + i, base, len);
    S.lbase[i] = base;
    S.llen[i] = len;
  }
  __syncthreads();
  // total entries and the largest list H (warp 0)
  if (wid == 0) {
    uint32_t s = 0, best = 0, bi = 0;
    for (uint32_t i = ln; i < d; i += 32) {
      const uint32_t l = S.llen[i];
      s += l;
      if (l > best) {
        best = l;
        bi = i;
      }
    }
    s = warp_sum(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint32_t ob = __shfl_xor_sync(kFull, best, o), oi = __shfl_xor_sync(kFull, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (ln == 0) {
      S.tot = s - best;  // entries inserted into the table
      S.hl = bi;
      S.demote = 0;
    }
  }
  __syncthreads();
  const uint32_t ins_total = S.tot, hl = S.hl;
  if (ins_total <= kHashCap) {
    // one group covering every id
    if (tid == 0) {
      S.gk[0] = 0;
      S.gk[1] = kHW;
      S.ng = 1;
    }
    for (uint32_t i = tid; i < d; i += blockDim.x) {
      S.bnd[i][0] = 0;
      S.bnd[i][kHW] = S.llen[i];
    }
  } else {
    // window bounds of every list: row table or ballots over a short list
    for (uint32_t k = tid; k < kHW; k += blockDim.x) S.ek[k] = 0;
    __syncthreads();
    for (uint32_t i = wid; i < d; i += nw) {
      const uint32_t len = S.llen[i];
      const uint32_t* p = partner + S.lbase[i];
      uint32_t b = 0;
      if (len > kRowMin) {
        const uint32_t v = lists.mid(e0 + i);
        b = min(rows[(uint64_t)rowid[v] * (kHW + 1) + ln], len);
      } else {
        const uint32_t x0 = ln < len ? p[ln] : 0xFFFFFFFFu;
        const uint32_t x1 = ln + 32 < len ? p[ln + 32] : 0xFFFFFFFFu;
        for (uint32_t k = 0; k < kHW; k++) {
          const uint32_t key = S.wb[k];
          const uint32_t c = __popc(__ballot_sync(kFull, x0 < key)) + __popc(__ballot_sync(kFull, x1 < key));
          if (ln == k) b = c;
        }
      }
      if (ln == 0) b = 0;  // window 0 starts at id 0
      S.bnd[i][ln] = b;
      if (ln == 0) S.bnd[i][kHW] = len;
      const uint32_t nb = __shfl_down_sync(kFull, b, 1);
      const uint32_t end = ln == 31 ? len : nb;
      if (i != hl && end > b) atomicAdd(&S.ek[ln], end - b);  // table entries per window
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t ng = 0, acc = 0, kend = kHW;  // windows from kend on hold only ids >= lim
      while (kend > 1 && S.wb[kend - 1] >= lim) kend--;
      S.gk[0] = 0;
      for (uint32_t k = 0; k < kend; k++) {
        const uint32_t ek = S.ek[k];
        if (ek > kHashCap) {
          S.demote = 1;
          break;
        }
        if (acc + ek > kHashCap) {
          S.gk[++ng] = k;
          acc = 0;
        }
        acc += ek;
      }
      S.gk[++ng] = kend;
      S.ng = ng;
    }
  }
  __syncthreads();
  if (S.demote) return false;
  const uint32_t ng = S.ng;
  if (tid == 0 && stat) {
    atomicAdd(&stat[0], 1ull);
    if (ng > 1) {
      atomicAdd(&stat[1], 1ull);
      atomicAdd(&stat[2], (unsigned long long)ng);
    }
  }
  const uint32_t cmask = (1u << cb) - 1u;
  for (uint32_t g = 0; g < ng; g++) {
    const uint32_t ka = S.gk[g], kb = S.gk[g + 1];
    // segment of every list in the group, exclusive prefix of the inserted
    // lists' lengths (H counts 0 here; warp 0)
    if (wid == 0) {
      uint32_t carry = 0;
      for (uint32_t i0 = 0; i0 < d; i0 += 32) {
        const uint32_t i = i0 + ln;
        uint32_t len = 0;
        if (i < d) {
          const uint32_t s0 = S.bnd[i][ka];
          len = S.bnd[i][kb] - s0;
          S.seg0[i] = s0;
          if (i == hl) {
            S.hlen = len;
            len = 0;
          }
        }
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, incl, o);
          if (ln >= (uint32_t)o) incl += y;
        }
        if (i < d) S.pre[i] = carry + incl - len;
        carry += __shfl_sync(kFull, incl, 31);
      }
      if (ln == 0) S.pre[d] = carry;
    }
    __syncthreads();
    const uint32_t gt = S.pre[d];
    // table size follows the inserted entries (distinct partners <= entries): 2 slots per entry
    const uint32_t T = min(kHashSlots, max(256u, (gt * 2 + 63) & ~63u));
    const uint32_t TB = T / 4;
    // phase A: insert the other lists; warps take 128-position chunks dynamically
    for (;;) {
      uint32_t c = 0;
      if (ln == 0) c = atomicAdd(&S.next, 1u);
      const uint32_t p0 = __shfl_sync(kFull, c, 0) * kHashChunk;
      if (p0 >= gt) break;
      // list of the chunk's first position (same for all lanes: broadcast reads)
      uint32_t l0 = 0, hi = d;
      while (hi - l0 > 1) {
        const uint32_t mid = (l0 + hi) >> 1;
        if (S.pre[mid] <= p0) l0 = mid; else hi = mid;
      }
      uint32_t x[4];
      bool ok[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint32_t p = p0 + 32 * j + ln;
        ok[j] = p < gt;
        x[j] = 0;
        if (ok[j]) {
          uint32_t lo = l0;  // list lo: pre[lo] <= p < pre[lo + 1]
          while (S.pre[lo + 1] <= p) lo++;
          PBNG_DCHECK(lo < d && lo != hl && S.seg0[lo] + (p - S.pre[lo]) < S.llen[lo]);
          x[j] = partner[S.lbase[lo] + S.seg0[lo] + (p - S.pre[lo])];
        }
      }
#pragma unroll
      for (int j = 0; j < 4; j++)
        if (ok[j] && x[j] != skip && x[j] < lim && hash_count(S.tab, TB, cb, x[j])) filt_set(S.filt, x[j]);
    }
    __syncthreads();
    // phase B: H's segment looks its partners up (one contiguous run)
    if (gt) {
      const uint32_t hn = S.hlen;
      const uint32_t* hp = partner + S.lbase[hl] + S.seg0[hl];
      // 16-byte loads: virtual positions q = i + mis over the aligned run ab[],
      // chunks of 128 * kHashBDepth positions, every lane's kHashBDepth loads
      // issued before any entry is used (one memory round trip per chunk).  A
      // load only touches the 16-byte block of a valid entry (never past the
      // allocation).
      const uint32_t mis = (uint32_t)(((uintptr_t)hp & 15u) >> 2);
      const uint4* ab = reinterpret_cast<const uint4*>(hp - mis);
      const uint32_t qend = hn + mis;
      if (tid == 0) S.next = 0;
      __syncthreads();
      for (;;) {
        uint32_t c = 0;
        if (ln == 0) c = atomicAdd(&S.next, 1u);
        const uint32_t q0 = __shfl_sync(kFull, c, 0) * (128u * kHashBDepth);
        if (q0 >= qend) break;
        uint4 v[kHashBDepth];
#pragma unroll
        for (int j = 0; j < kHashBDepth; j++) {
          const uint32_t q = q0 + 128u * j + 4u * ln;
          v[j] = q < qend ? ab[q >> 2] : make_uint4(skip, skip, skip, skip);
        }
#pragma unroll
        for (int j = 0; j < kHashBDepth; j++) {
          const uint32_t q = q0 + 128u * j + 4u * ln;
          const uint32_t e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
          for (int t = 0; t < 4; t++) {
            const uint32_t x = e[t];
            const bool ok = q + t >= mis && q + t < qend;
            if (ok && x != skip && x < lim && filt_has(S.filt, x)) hash_lookup_inc(S.tab, TB, cb, x);
          }
        }
      }
      __syncthreads();
    }
    if (tid == 0) S.next = 0;
    uint4* tab4 = reinterpret_cast<uint4*>(S.tab);
    auto one = [&](uint32_t v) {
      const uint32_t w = v & cmask;
      if (w >= 2) emit((v >> cb) - 1u, w);
    };
    uint4* filt4 = reinterpret_cast<uint4*>(S.filt);
    for (uint32_t s = tid; s < kFiltWords / 4; s += blockDim.x) filt4[s] = make_uint4(0u, 0u, 0u, 0u);
    for (uint32_t s = tid; s < T / 4; s += blockDim.x) {
      const uint4 v = tab4[s];
      if (v.x | v.y | v.z | v.w) {
        tab4[s] = make_uint4(0u, 0u, 0u, 0u);
        one(v.x);
        one(v.y);
        one(v.z);
        one(v.w);
      }
    }
    __syncthreads();
  }
  return true;
}

// Tier-1 kernel.  MODE 0 COUNT / 1 PEEL / 2 LINK (as emit<MODE>), MODE 3 =
// vertex-priority count with starts in U (kernels_vp.cuh: lists cut at cutV,
// lasts below the start; C(w,2) to the last and to the start).
// Starts that do not fit (a window above capacity) are appended to tier 2.
template <int MODE, class L>
__device__ __forceinline__ void hash_tier(const AggArgs& a, const L& lists, HashSmem& S) {
  for (uint32_t k = threadIdx.x; k <= kHW; k += blockDim.x) S.wb[k] = a.wb[k];
  for (uint32_t i = threadIdx.x; i < kHashSlots; i += blockDim.x) S.tab[i] = 0u;
  for (uint32_t i = threadIdx.x; i < kFiltWords; i += blockDim.x) S.filt[i] = 0u;
  if (threadIdx.x == 0) S.next = 0;
  const uint32_t n = *a.count;
  unsigned long long upd = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      S.t = atomicAdd(a.ticket, 1u);
      S.acc = 0;
    }
    __syncthreads();
    const uint32_t i = S.t;
    if (i >= n) break;
    const uint2 it = a.list[i];
    const uint32_t u = it.x;
    const uint64_t e0 = a.offU[u], e1 = a.offU[u + 1];
    uint64_t acc = 0;
    bool done;
    if constexpr (MODE == 3) {
      auto out = [&](uint32_t k, uint32_t w) {
        if (a.part[k] == kUnassigned) {
          const uint64_t dd = choose2(w);
          red_add_u64(&a.support[k], dd);
          acc += dd;
        }
      };
      done = hash_agg_one(lists, e0, e1, 0xFFFFFFFFu, u, a.adjV, a.rowid, a.rows, a.cb, S, out, a.c->hashc);
    } else {
      auto out = [&](uint32_t k, uint32_t w) { emit<MODE>(a, u, k, w, acc, upd); };
      done = hash_agg_one(lists, e0, e1, u, MODE == 2 ? u : 0xFFFFFFFFu, a.adjV, a.rowid, a.rows, a.cb, S, out,
                          a.c->hashc);
    }
    if (!done) {
      if (threadIdx.x == 0) {
        a.tier2[atomicAdd(a.ntier2, 1u)] = it;
        atomicAdd(&a.c->hashc[3], 1ull);
      }
    } else if (MODE == 0 || MODE == 3) {
      acc = warp_sum(acc);
      if (lane_id() == 0 && acc) atomicAdd(&S.acc, (unsigned long long)acc);
      __syncthreads();
      if (threadIdx.x == 0) {
        if (MODE == 0) a.support[u] = S.acc;
        else if (S.acc) red_add_u64(&a.support[u], S.acc);
      }
    }
    __syncthreads();
  }
  if (MODE == 1) flush_updates(a, upd);
}

template <int MODE>
__global__ void __launch_bounds__(kHashThreads, kHashCtas) k_agg_hash(AggArgs a) {
  extern __shared__ __align__(16) unsigned char hsm_[];
  HashSmem& S = *reinterpret_cast<HashSmem*>(hsm_);
  hash_tier<MODE>(a, agg_lists<MODE>(a), S);
}
