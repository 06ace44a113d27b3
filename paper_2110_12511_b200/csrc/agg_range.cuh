// agg_range.cuh — tier-1 wedge aggregation: one CTA per vertex, partner ids
// processed one RANGE of up to kWindow ids at a time in shared memory.
//
// A frontier vertex u next to large lists has more distinct partners u' than a
// CTA's shared memory can index (the paper keeps a private n-element counter
// array per thread; on B200 that array would live in HBM and every
// wedge would be a random global atomic).  Most partners share a single
// neighbour with u (w = 1, no butterfly), so:
//   * a shared-memory BITMAP over the window [a, a + kWindow) records first
//     occurrences: one native 32-bit atomicOr per wedge, fully convergent;
//   * a repeat (bit already set) is counted in a small open-addressing table
//     keyed by u'; only these partners (w >= 2) are emitted, with
//     w = 1 + repeats.
// Partner lists are sorted by id, so each list is consumed window by window
// through a cursor and every wedge (u, v, u') is read exactly once, coalesced
// (16-byte loads, 128 ids per warp step).  Lists are cut into pieces of
// kPiece entries that warps take dynamically, so hub lists never serialise on
// one warp; piece cursors live in per-CTA global scratch (L2-resident).  If
// the repeats of a window overflow the table, the window is rewound and halved.
#pragma once
// (included inside namespace pbng by kernels_cd.cuh)

constexpr uint32_t kBitWords = 32768;              // bitmap words: window of 2^20 ids
constexpr uint64_t kWindow = (uint64_t)kBitWords * 32;
constexpr uint32_t kDupSlots = 8192;               // repeat table (key << 32 | repeats)
constexpr uint32_t kDupCap = kDupSlots / 2;
constexpr uint32_t kDupProbe = 32;
constexpr uint32_t kActMax = 2048;                 // active pieces queued per pass
constexpr uint64_t kEmptySlot = 0xFFFFFFFF00000000ull;

struct Pieces {         // per-CTA global scratch, capacity `cap` pieces
  uint64_t* pos;        // cursor (absolute index into the partner array)
  uint64_t* end;        // end of the piece (absolute)
  uint64_t* save;       // cursor at the start of the current window (replay)
  uint32_t* head;       // id at the cursor (0xFFFFFFFF when exhausted)
  uint32_t* srange;     // window attempt that last wrote save[]
  uint64_t* pedge;      // edge index of the list the piece belongs to
};

// No second pass (CD peel / one-sided count).
struct NoPass2 {
  static constexpr bool kOn = false;
  __device__ void operator()(uint64_t, unsigned long long) const {}
};

struct RangeShared {
  uint32_t np, over, t, nact, next, ndup;
  unsigned long long acc;
};

struct RangeSmem {
  uint32_t bits[kBitWords];
  unsigned long long dup[kDupSlots];
  uint16_t dslot[kDupSlots];
  uint32_t act[kActMax];
};

// Count one more occurrence of k in the repeat table.
__device__ __forceinline__ void dup_insert(RangeSmem& S, RangeShared& sh, uint32_t k) {
  uint32_t h = (k * 0x9E3779B1u) >> (32 - 13);
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
        if (i < kDupCap) S.dslot[i] = (uint16_t)h;
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
    h = (h + 1) & (kDupSlots - 1);
  }
}

// Repeats recorded for k in the current window (0 when k occurred once).
__device__ __forceinline__ uint32_t dup_lookup(const RangeSmem& S, uint32_t k) {
  uint32_t h = (k * 0x9E3779B1u) >> (32 - 13);
  for (uint32_t probe = 0; probe <= kDupProbe + 1; probe++) {
    const unsigned long long cur = S.dup[h];
    if ((uint32_t)(cur >> 32) == k) return (uint32_t)cur;
    if (cur == kEmptySlot) return 0;
    h = (h + 1) & (kDupSlots - 1);
  }
  return 0;
}

// One warp consumes a piece from cursor pk (< ek) while ids < b, marking every
// id != u in the window bitmap.  On return pk is the new cursor and nxt the id
// found there (or ~0u).
__device__ __forceinline__ void walk_piece(uint64_t& pk, uint64_t ek, uint32_t a, uint32_t b, uint32_t& nxt,
                                           uint32_t u, const uint32_t* __restrict__ adjL, bool vec, RangeSmem& S,
                                           RangeShared& sh) {
  const uint32_t ln = lane_id();
  for (;;) {
    const uint64_t a0 = pk & ~3ull;
    const uint64_t q = a0 + 4ull * ln;
    uint32_t x[4];
    if (vec && q + 3 < ek) {
      const uint4 v4 = __ldg(reinterpret_cast<const uint4*>(adjL + q));
      x[0] = v4.x;
      x[1] = v4.y;
      x[2] = v4.z;
      x[3] = v4.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; i++) x[i] = q + i < ek ? adjL[q + i] : 0xFFFFFFFFu;
    }
    uint32_t inm = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const bool in = q + i >= pk && q + i < ek && x[i] < b;
      inm += in;
      if (in && x[i] != u) {
        const uint32_t o = x[i] - a;
        const uint32_t bit = 1u << (o & 31);
        if (atomicOr(&S.bits[o >> 5], bit) & bit) dup_insert(S, sh, x[i]);
      }
    }
    const uint32_t nin = warp_sum(inm);  // in-range entries form the prefix [pk, pk + nin)
    pk += nin;
    if (pk >= ek) {
      nxt = 0xFFFFFFFFu;
      return;
    }
    if (pk < a0 + 128) {  // the window ends inside this block: report the id at pk
      const uint32_t o = (uint32_t)(pk - a0);
      const uint32_t el = o & 3;
      const uint32_t pick = el == 0 ? x[0] : el == 1 ? x[1] : el == 2 ? x[2] : x[3];
      nxt = __shfl_sync(kFull, pick, o >> 2);
      return;
    }
  }
}

// Aggregate w(u, u') over every wedge of u and call emit(u', w) once per
// distinct partner with w >= 2.  Call with the whole CTA; on entry and exit
// the bitmap is zero and the repeat table empty.
//
// Pass2 (vertex-priority counting, start on the non-peel side): after each
// window, the wedges of every list piece are walked again and the repeats of
// their partners summed per list: pass2(edge, Σ (w - 1) over its w >= 2 entries).
template <class L, class Emit, class Pass2 = NoPass2>
__device__ __forceinline__ void range_agg_one(const L& lists, uint64_t e0, uint64_t e1, uint32_t u,
                                              uint32_t idspace, const uint32_t* __restrict__ adjL, RangeSmem& S,
                                              const Pieces& pc, RangeShared& sh, Emit& emit,
                                              unsigned long long* dbg, const Pass2& pass2 = Pass2()) {
  const uint32_t tid = threadIdx.x, bd = blockDim.x, ln = lane_id(), w = tid >> 5, nw = bd >> 5;
  const bool vec = (reinterpret_cast<uintptr_t>(adjL) & 15) == 0;
  if (tid == 0) sh.np = 0;
  __syncthreads();
  // cut the partner lists into pieces (virtual neighbours)
  for (uint64_t e = e0 + tid; e < e1; e += bd) {
    uint64_t base;
    uint32_t len;
    lists.get(e, base, len);
    const uint32_t np = (len + kPiece - 1) / kPiece;
    if (!np) continue;
    const uint32_t slot = atomicAdd(&sh.np, np);
    for (uint32_t k = 0; k < np; k++) {
      const uint64_t p = base + (uint64_t)k * kPiece;
      pc.pos[slot + k] = p;
      pc.end[slot + k] = base + (uint64_t)min(len, (k + 1) * kPiece);
      pc.head[slot + k] = 0;  // unknown: the first window's walk finds it
      pc.srange[slot + k] = 0;
      if (Pass2::kOn) pc.pedge[slot + k] = e;
    }
  }
  __syncthreads();
  const uint32_t np = sh.np;
  uint64_t width = kWindow;
  uint64_t a = 0;
  uint32_t rid = 0;  // window attempt id (tags which pieces a replay must rewind)
  while (a < idspace) {
    const uint64_t b64 = a + width < idspace ? a + width : idspace;
    const uint32_t b = (uint32_t)b64;
    rid++;
    if (tid == 0) {
      sh.over = 0;
      sh.ndup = 0;
    }
    uint32_t any = 0;  // did any piece have ids in this window
    for (uint32_t pw = 0; pw < np; pw += kActMax) {
      const uint32_t pe = np - pw < kActMax ? np : pw + kActMax;
      if (tid == 0) {
        sh.nact = 0;
        sh.next = 0;
      }
      __syncthreads();
      for (uint32_t j0 = pw + w * 32; j0 < pe; j0 += nw * 32) {
        const uint32_t j = j0 + ln;
        const bool act = j < pe && pc.head[j] < b;
        warp_append(act, j, S.act, &sh.nact);
      }
      __syncthreads();
      const uint32_t nact = sh.nact;
      any |= nact;
      for (;;) {
        uint32_t t = 0;
        if (ln == 0) t = atomicAdd(&sh.next, 1u);
        t = __shfl_sync(kFull, t, 0);
        if (t >= nact) break;
        const uint32_t j = S.act[t];
        uint64_t pk = pc.pos[j];
        const uint64_t ek = pc.end[j];
        if (ln == 0) {
          pc.save[j] = pk;
          pc.srange[j] = rid;
        }
        uint32_t nxt;
        walk_piece(pk, ek, (uint32_t)a, b, nxt, u, adjL, vec, S, sh);
        if (ln == 0) {
          pc.pos[j] = pk;
          pc.head[j] = nxt;
        }
      }
      __syncthreads();
    }
    const bool over = sh.over != 0;
    const uint32_t nd = min(sh.ndup, kDupCap);
    if (Pass2::kOn && any && !over && nd) {
      // second walk over this window's wedges: repeats of their partners per list
      if (tid == 0) sh.next = 0;
      __syncthreads();
      for (;;) {
        uint32_t t = 0;
        if (ln == 0) t = atomicAdd(&sh.next, 1u);
        t = __shfl_sync(kFull, t, 0);
        if (t >= np) break;
        if (pc.srange[t] != rid) continue;
        const uint64_t p0 = pc.save[t], p1 = pc.pos[t];
        unsigned long long cs = 0;
        for (uint64_t q = p0 + ln; q < p1; q += 32) {
          const uint32_t x = adjL[q];
          if (x != u) cs += dup_lookup(S, x);
        }
        cs = warp_sum(cs);
        if (ln == 0 && cs) pass2(pc.pedge[t], cs);
      }
      __syncthreads();
    }
    if (any) {
      // clear the window bitmap and drain the repeat table
      const uint32_t nwords = (uint32_t)((b64 - a + 31) >> 5);
      for (uint32_t i = tid; i < nwords; i += bd) S.bits[i] = 0;
      for (uint32_t i = tid; i < nd; i += bd) {
        const uint32_t sl = S.dslot[i];
        const unsigned long long v = S.dup[sl];
        S.dup[sl] = kEmptySlot;
        if (!over) emit((uint32_t)(v >> 32), (uint32_t)v + 1u);
      }
    }
    if (over) {
      // repeats of this window overflow the table: rewind and halve (rare)
      for (uint32_t i = tid; i < kDupSlots; i += bd) S.dup[i] = kEmptySlot;
      for (uint32_t j = tid; j < np; j += bd) {
        if (pc.srange[j] != rid) continue;
        const uint64_t p = pc.save[j];
        pc.pos[j] = p;
        pc.head[j] = adjL[p];
      }
      width = width > 32 ? width / 2 : 32;
      if (tid == 0) atomicAdd(&dbg[1], 1ull);
      __syncthreads();
      continue;
    }
    if (tid == 0) atomicAdd(&dbg[0], 1ull);
    __syncthreads();
    a = b64;
    // repeats are dense only in parts of the id space (low ranks = high degree):
    // widen again once a window used a small part of the table
    if (width < kWindow && nd < kDupCap / 4) width *= 2;
  }
}

template <int MODE>
__global__ void __launch_bounds__(kRangeThreads, 1) k_agg_range(AggArgs a) {
  extern __shared__ __align__(16) unsigned char rsm[];
  RangeSmem& S = *reinterpret_cast<RangeSmem*>(rsm);
  __shared__ RangeShared sh;
  for (uint32_t i = threadIdx.x; i < kBitWords; i += blockDim.x) S.bits[i] = 0;
  for (uint32_t i = threadIdx.x; i < kDupSlots; i += blockDim.x) S.dup[i] = kEmptySlot;
  const uint64_t cap = a.piece_cap;
  const Pieces pc{a.piece_pos + blockIdx.x * cap, a.piece_end + blockIdx.x * cap, a.piece_save + blockIdx.x * cap,
                  a.piece_head + blockIdx.x * cap, a.piece_srange + blockIdx.x * cap, nullptr};
  const uint32_t n = *a.count;
  const CdLists L{a.adjU, a.offV, a.ld};
  unsigned long long upd = 0;
  for (;;) {
    if (threadIdx.x == 0) sh.t = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const uint32_t i = sh.t;
    if (threadIdx.x == 0) sh.acc = 0;
    __syncthreads();
    if (i >= n) break;
    const uint32_t u = a.list[i].x;
    uint64_t acc = 0;
    auto out = [&](uint32_t k, uint32_t w) { emit<MODE>(a, k, w, acc, upd); };
    range_agg_one(L, a.offU[u], a.offU[u + 1], u, a.nU, a.adjV, S, pc, sh, out, a.c->dbg);
    if (MODE == 0) {
      acc = warp_sum(acc);
      if (lane_id() == 0 && acc) atomicAdd(&sh.acc, (unsigned long long)acc);
      __syncthreads();
      if (threadIdx.x == 0) a.support[u] = sh.acc;
    }
  }
  if (MODE == 1) {
    upd = warp_sum(upd);
    if (lane_id() == 0 && upd) atomicAdd(&a.c->updates, upd);
  }
}
