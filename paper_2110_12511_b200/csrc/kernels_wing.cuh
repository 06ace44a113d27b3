// kernels_wing.cuh — BE-Index construction and
// wing decomposition by level-synchronous batch bloom peeling on it (§8(f) f4,
// the BE-Index update of Alg.3 P:644-674 applied to a whole level at once as
// in the batch bloom updates of P:1452-1490).
//
// BE-Index.  "Each pair of endpoint vertices {start, last} of wedges explored
// during counting represents the dominating set of a bloom (with last as the
// highest priority vertex) containing the edges {start, mid} and {mid, last}
// for all midpoints mid ... edges {start, mid} and {mid, last} are twins"
// (P:627-634).  So the blooms are the (start, last) pairs of Alg.1 (the same
// priority walk as kernels_edge.cuh) with c = wedge_count >= 2, the bloom
// number is c, and its c twin pairs are the wedges (mid, last).  Layout:
//   bloom_off[nb+1]  first pair of bloom b (pairs of a bloom are contiguous)
//   bloom_k[nb]      bloom number k_B (initially c)
//   bloom_dom[nb]    dominant pair: (start, last) in rank labels of one side,
//                    bit 31 of .x = side of the dominant set (0 U, 1 V)
//   pair[np]         (e1, e2): canonical edge ids (positions in the relabeled
//                    U CSR) of {start, mid} and {mid, last}
//   pair_bloom[np]   owning bloom
// Built in two runs over the starts (sizes, then fill), one persistent CTA
// per start with dense per-CTA counters over the last ids in global memory.
//
// Wing peeling (level-synchronous, exact supports, no clamp):
//   level k = max(k, min live support); S = live edges with support <= k get
//   θ = k; each pair of a bloom with an edge in S dies.  For a bloom with
//   k_B live pairs of which d die this round (Property 1): every
//   surviving edge of a dying pair loses its k_B - 1 butterflies in B, every
//   edge of a surviving pair loses d; k_B -= d.  Every butterfly lies in
//   exactly one bloom (Property 2), so supports stay exact;
//   decrements that cross k put the edge into the next round at the same k.
#pragma once
#include "kernels_edge.cuh"

namespace pbng {

constexpr uint32_t kBeThreads = 256;
constexpr uint32_t kBeInvalid = 0xFFFFFFFFu;

struct BeArgs {
  EdgeArgs a;                          // walk of one start side (accS/accM unused)
  const uint32_t* __restrict__ mirM2U; // mid-side CSR position -> canonical id (start side U: V->U map)
  const uint32_t* __restrict__ mirS2U; // start-side position -> canonical id (start side V)
  uint32_t side;                       // 0: starts in U, 1: starts in V
  uint32_t* cnt;                       // per CTA: nS counters
  uint32_t* bidx;                      // per CTA: nS bloom index within the start (kBeInvalid = none)
  uint32_t* pbase;                     // per CTA: nS pair base within the start
  unsigned long long* nb_s;            // sizes run: blooms per start
  unsigned long long* np_s;            // sizes run: pairs per start
  const unsigned long long* bS;        // fill run: first bloom of each start (exclusive scan)
  const unsigned long long* pS;        // fill run: first pair of each start
  unsigned long long* bloom_off;
  uint32_t* bloom_k;
  uint2* bloom_dom;
  uint2* pair;
  uint32_t* pair_bloom;
  uint32_t* ticket;
};

// Visit every wedge (e = start-side position of mid, f = mid-side position of
// last, last) of start s: warps take 32 mids at a time, prefixes flattened.
template <class F>
__device__ __forceinline__ void be_walk(const EdgeArgs& a, uint32_t s, uint32_t wi, uint32_t nw, F& fn) {
  const uint32_t ln = lane_id();
  const uint64_t e0 = a.offS[s], e1 = a.offS[s + 1];
  for (uint64_t g = e0 + 32ull * wi; g < e1; g += 32ull * nw) {
    const uint64_t e = g + ln;
    uint32_t len = 0;
    uint64_t base = 0;
    if (e < e1) {
      const uint32_t mid = a.adjS[e];
      base = a.offM[mid];
      len = edge_lower_bound(a.adjM + base, a.cutM[mid], s);
    }
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (ln >= (uint32_t)o) incl += y;
    }
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - len;
    for (uint32_t kb = 0; kb < total; kb += 32) {
      const uint32_t k = kb + ln;
      uint32_t pos = 0;
#pragma unroll
      for (uint32_t step = 16; step > 0; step >>= 1) {
        const uint32_t y = __shfl_sync(kFull, incl, pos + step - 1);
        if (y <= k) pos += step;
      }
      const uint32_t owner = pos > 31 ? 31 : pos;
      const uint32_t oex = __shfl_sync(kFull, excl, owner);
      const uint64_t ob = __shfl_sync(kFull, base, owner);
      const uint64_t oe = __shfl_sync(kFull, e, owner);
      if (k < total) {
        const uint64_t f = ob + (k - oex);
        fn(oe, f, a.adjM[f]);
      }
    }
  }
}

struct BeCount {
  uint32_t* cnt;
  __device__ __forceinline__ void operator()(uint64_t, uint64_t, uint32_t last) { atomicAdd(&cnt[last], 1u); }
};
struct BeClear {
  uint32_t* cnt;
  uint32_t* bidx;
  __device__ __forceinline__ void operator()(uint64_t, uint64_t, uint32_t last) {
    __stcg(&cnt[last], 0u);
    __stcg(&bidx[last], kBeInvalid);
  }
};
// sizes run: pairs = wedges with c >= 2, blooms = distinct such lasts
struct BeSize {
  uint32_t* cnt;
  uint32_t* bidx;
  uint32_t* s_nb;
  uint32_t* s_np;
  __device__ __forceinline__ void operator()(uint64_t, uint64_t, uint32_t last) {
    if (__ldcg(&cnt[last]) < 2) return;
    atomicAdd(s_np, 1u);
    if (atomicCAS(&bidx[last], kBeInvalid, 0u) == kBeInvalid) atomicAdd(s_nb, 1u);
  }
};
// fill run, pass A: the first wedge of each bloom claims its index and pair range
struct BeAssign {
  const BeArgs* b;
  uint32_t s;
  unsigned long long* s_acc;  // (blooms << 40) | pairs: one atomic keeps bloom order = pair order
  __device__ __forceinline__ void operator()(uint64_t, uint64_t, uint32_t last) {
    const uint32_t c = __ldcg(&b->cnt[last]);
    if (c < 2) return;
    if (atomicCAS(&b->bidx[last], kBeInvalid, kBeInvalid - 1) != kBeInvalid) return;
    const unsigned long long old = atomicAdd(s_acc, (1ull << 40) | c);
    const uint32_t li = (uint32_t)(old >> 40);
    const uint32_t pb = (uint32_t)(old & ((1ull << 40) - 1));
    const uint64_t bid = b->bS[s] + li;
    b->bloom_off[bid] = b->pS[s] + pb;
    b->bloom_k[bid] = c;
    b->bloom_dom[bid] = make_uint2(s | (b->side << 31), last);
    __stcg(&b->pbase[last], pb);
    __stcg(&b->bidx[last], li);
  }
};
// fill run, pass F: each wedge of a bloom takes a slot (count down the counter)
struct BeFill {
  const BeArgs* b;
  uint32_t s;
  __device__ __forceinline__ void operator()(uint64_t e, uint64_t f, uint32_t last) {
    const uint32_t li = __ldcg(&b->bidx[last]);
    if (li == kBeInvalid) return;
    const uint32_t r = atomicSub(&b->cnt[last], 1u) - 1u;
    const uint64_t p = b->pS[s] + __ldcg(&b->pbase[last]) + r;
    const uint32_t e1 = b->side == 0 ? (uint32_t)e : b->mirS2U[e];   // {start, mid}
    const uint32_t e2 = b->side == 0 ? b->mirM2U[f] : (uint32_t)f;   // {mid, last}
    b->pair[p] = make_uint2(e1, e2);
    b->pair_bloom[p] = (uint32_t)(b->bS[s] + li);
  }
};

// FILL = false: sizes run (nb_s, np_s); true: fill run.  Starts with fewer
// than two mids or id 0 have no bloom and are skipped without a walk.
template <bool FILL>
__global__ void __launch_bounds__(kBeThreads) k_be_build(BeArgs b) {
  __shared__ uint32_t s_i, s_nb, s_np;
  __shared__ unsigned long long s_acc;
  const uint32_t w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const EdgeArgs& a = b.a;
  BeArgs* bp = &b;
  const uint64_t per = a.nS;
  bp->cnt += blockIdx.x * per;
  bp->bidx += blockIdx.x * per;
  bp->pbase += blockIdx.x * per;
  for (;;) {
    if (threadIdx.x == 0) {
      s_i = atomicAdd(b.ticket, 1u);
      s_nb = 0;
      s_np = 0;
      s_acc = 0;
    }
    __syncthreads();
    const uint32_t s = s_i;
    if (s >= a.nS) break;
    if (s == 0 || a.offS[s + 1] - a.offS[s] < 2) {
      if (!FILL && threadIdx.x == 0) b.nb_s[s] = b.np_s[s] = 0ull;
      __syncthreads();
      continue;
    }
    BeCount c1{b.cnt};
    be_walk(a, s, w, nw, c1);
    __syncthreads();
    if (!FILL) {
      BeSize sz{b.cnt, b.bidx, &s_nb, &s_np};
      be_walk(a, s, w, nw, sz);
      __syncthreads();
      if (threadIdx.x == 0) {
        b.nb_s[s] = s_nb;
        b.np_s[s] = s_np;
      }
    } else {
      BeAssign as{bp, s, &s_acc};
      be_walk(a, s, w, nw, as);
      __syncthreads();
      BeFill fl{bp, s};
      be_walk(a, s, w, nw, fl);
      __syncthreads();
    }
    BeClear cl{b.cnt, b.bidx};
    be_walk(a, s, w, nw, cl);
    __syncthreads();
  }
}

__global__ void k_iota(uint64_t n, uint32_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)i;
}

// caller edge i (caller CSR of the output side) -> canonical id, inverted:
// r2c[canonical] = i
__global__ void k_edge_r2c(uint32_t nX, uint64_t m, const uint64_t* __restrict__ offX,
                           const uint32_t* __restrict__ idxX, const uint32_t* __restrict__ rankX,
                           const uint32_t* __restrict__ rankY, const uint64_t* __restrict__ offXr,
                           const uint32_t* __restrict__ adjXr, uint32_t* __restrict__ r2c) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nX;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (offX[mid] <= i) lo = mid; else hi = mid;
    }
    const uint32_t rx = rankX[lo], ry = rankY[idxX[i]];
    const uint64_t bx = offXr[rx];
    r2c[bx + edge_lower_bound(adjXr + bx, (uint32_t)(offXr[rx + 1] - bx), ry)] = (uint32_t)i;
  }
}

// BE-Index in caller terms: pairs as caller edge positions, dominant pairs as
// caller vertex labels (bit 31 of the first = side of the dominant set)
__global__ void k_be_export(uint64_t nb, uint64_t np, const uint2* __restrict__ pair, const uint32_t* __restrict__ r2c,
                            const uint2* __restrict__ dom, const uint32_t* __restrict__ invU,
                            const uint32_t* __restrict__ invV, uint32_t* __restrict__ out_pair,
                            uint32_t* __restrict__ out_dom) {
  const uint64_t n = np > nb ? np : nb;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < np) {
      const uint2 pr = pair[i];
      out_pair[2 * i] = r2c[pr.x];
      out_pair[2 * i + 1] = r2c[pr.y];
    }
    if (i < nb) {
      const uint2 d = dom[i];
      const uint32_t side = d.x >> 31, x = d.x & 0x7FFFFFFFu;
      const uint32_t* inv = side ? invV : invU;
      out_dom[2 * i] = inv[x] | (side << 31);
      out_dom[2 * i + 1] = inv[d.y];
    }
  }
}

// canonical id of every V-CSR entry (v, u): position of v in u's sorted U list
__global__ void k_be_mirror(uint32_t nV, uint64_t m, const uint64_t* __restrict__ offV,
                            const uint32_t* __restrict__ adjV, const uint64_t* __restrict__ offU,
                            const uint32_t* __restrict__ adjU, uint32_t* __restrict__ mirV2U) {
  for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < m; f += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nV;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (offV[mid] <= f) lo = mid; else hi = mid;
    }
    const uint32_t u = adjV[f];
    const uint64_t b = offU[u];
    mirV2U[f] = (uint32_t)(b + edge_lower_bound(adjU + b, (uint32_t)(offU[u + 1] - b), lo));
  }
}

// ---------------------------------------------------------------- wing peel
struct WingCtl {
  uint32_t nS, nX, nT;   // current S, next S (crossers), touched blooms
  uint32_t nlive;        // live list length after a level scan
  unsigned long long minsup;
};

struct WingArgs {
  uint64_t m;
  uint64_t nb;
  const unsigned long long* __restrict__ bloom_off;
  uint32_t* bloom_k;
  uint32_t* bloom_d;
  const uint2* __restrict__ pair;
  const uint32_t* __restrict__ pair_bloom;
  uint32_t* pstate;                     // 0 live, 1 dying (this round), 2 dead
  const unsigned long long* __restrict__ inc_off;  // per edge: its pairs
  const uint32_t* __restrict__ inc;
  unsigned long long* sup;
  uint64_t* theta;
  uint8_t* alive;
  uint32_t* live;                       // live edge list (compacted at level scans)
  uint32_t* S;
  uint32_t* X;
  uint32_t* T;
  WingCtl* ctl;
};

// support of every edge from the index: Σ_{B ∋ e} (k_B - 1) (Property 1)
__global__ void k_wing_init(WingArgs w) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < w.bloom_off[w.nb];
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = w.bloom_k[w.pair_bloom[p]];
    const uint2 pr = w.pair[p];
    atomicAdd(&w.sup[pr.x], (unsigned long long)(k - 1));
    atomicAdd(&w.sup[pr.y], (unsigned long long)(k - 1));
  }
}
__global__ void k_wing_inc_count(WingArgs w, unsigned long long* deg) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < w.bloom_off[w.nb];
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 pr = w.pair[p];
    atomicAdd(&deg[pr.x], 1ull);
    atomicAdd(&deg[pr.y], 1ull);
  }
}
__global__ void k_wing_inc_fill(WingArgs w, unsigned long long* cur, uint32_t* inc) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < w.bloom_off[w.nb];
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 pr = w.pair[p];
    inc[atomicAdd(&cur[pr.x], 1ull)] = (uint32_t)p;
    inc[atomicAdd(&cur[pr.y], 1ull)] = (uint32_t)p;
  }
}

// Level scan: compact the live list (drop peeled edges) and take its minimum support.
__global__ void k_wing_scan(WingArgs w, uint32_t n, const uint32_t* __restrict__ in, uint32_t* out) {
  unsigned long long mn = ~0ull;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x; i0 < n; i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    bool keep = false;
    uint32_t e = 0;
    if (i < n) {
      e = in[i];
      keep = w.alive[e];
      if (keep) mn = min(mn, w.sup[e]);
    }
    warp_append(keep, e, out, &w.ctl->nlive);
  }
  mn = warp_min_u64(mn);
  if (lane_id() == 0 && mn != ~0ull) atomicMin(&w.ctl->minsup, mn);
}

// S = live edges with support <= k (after a level change)
__global__ void k_wing_select(WingArgs w, uint32_t n, unsigned long long k) {
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x; i0 < n; i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    bool take = false;
    uint32_t e = 0;
    if (i < n) {
      e = w.live[i];
      take = w.alive[e] && w.sup[e] <= k;
    }
    warp_append(take, e, w.S, &w.ctl->nS);
  }
}

// peel S: θ = k, not alive; every live pair of an S edge starts dying, and its
// bloom is listed once
__global__ void k_wing_claim(WingArgs w, uint32_t n, unsigned long long k) {
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t ln = lane_id();
  for (uint64_t i = gw; i < n; i += nw) {
    const uint32_t e = w.S[i];
    if (ln == 0) w.theta[e] = k;
    for (uint64_t j = w.inc_off[e] + ln; j < w.inc_off[e + 1]; j += 32) {
      const uint32_t p = w.inc[j];
      if (w.pstate[p] != 0 || atomicCAS(&w.pstate[p], 0u, 1u) != 0u) continue;
      const uint32_t b = w.pair_bloom[p];
      if (atomicAdd(&w.bloom_d[b], 1u) == 0) w.T[atomicAdd(&w.ctl->nT, 1u)] = b;
    }
  }
}
// S edges leave the graph after every claim of this round has seen them
__global__ void k_wing_kill(WingArgs w, uint32_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    w.alive[w.S[i]] = 0;
}

__device__ __forceinline__ void wing_dec(WingArgs& w, uint32_t x, unsigned long long d, unsigned long long k) {
  const unsigned long long old = atomicAdd(&w.sup[x], (unsigned long long)(0ull - d));
  if (old > k && old - d <= k) w.X[atomicAdd(&w.ctl->nX, 1u)] = x;  // crosses the level: next round
}

// warp per touched bloom
__global__ void k_wing_update(WingArgs w, uint32_t n, unsigned long long k) {
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t ln = lane_id();
  for (uint64_t i = gw; i < n; i += nw) {
    const uint32_t b = w.T[i];
    const uint32_t kb = w.bloom_k[b], d = w.bloom_d[b];
    for (uint64_t p = w.bloom_off[b] + ln; p < w.bloom_off[b + 1]; p += 32) {
      const uint32_t st = w.pstate[p];
      if (st == 2) continue;
      const uint2 pr = w.pair[p];
      if (st == 1) {
        if (kb > 1) {
          if (w.alive[pr.x]) wing_dec(w, pr.x, kb - 1, k);
          if (w.alive[pr.y]) wing_dec(w, pr.y, kb - 1, k);
        }
        w.pstate[p] = 2;
      } else {
        wing_dec(w, pr.x, d, k);
        wing_dec(w, pr.y, d, k);
      }
    }
    __syncwarp();
    if (ln == 0) {
      w.bloom_k[b] = kb - d;
      w.bloom_d[b] = 0;
    }
  }
}

// ---------------------------------------------------------------- device-driven peel
// The whole peel in ONE persistent launch (one CTA per SM, co-resident by a
// cooperative launch): the phases of the host-driven loop above, separated by a
// grid barrier instead of a kernel boundary and a counter read-back.  Config 3
// runs 147,592 rounds of a few dozen edges each; host-driven, every round costs
// three launches and two stream synchronisations (~0.2 ms), here two grid
// barriers.  Counters are double-buffered so that a counter is reset only in a
// phase in which no thread reads or adds to it:
//   cnt[2]  lengths of the S / X lists (SX[cs] is peeled, SX[cs^1] collects the
//           crossers); nT[2] touched blooms of round r in nT[r & 1].
struct WingDev {
  uint32_t cnt[2];
  uint32_t nT[2];
  uint32_t nlive;
  uint32_t pad;
  unsigned long long minsup;
  unsigned long long bar;      // grid barrier: arrivals so far (monotonic)
  unsigned long long levels, rounds;
  unsigned long long clk[4];   // CTA 0 thread 0: cycles in level scans, selects, claim phases, update phases
  uint32_t cntC[2];            // candidate band: lengths of the two candidate lists
  unsigned long long minC;     // minimum live support among the candidates
};
constexpr uint32_t kWingThreads = 1024;
constexpr uint32_t kWingBigLen = 32;    // pair lists longer than this are walked by a whole CTA
constexpr uint32_t kWingBigMax = 1u << 22;  // ... up to this length (the flattened range of a CTA stays below 2^32)
constexpr uint32_t kWingBigCap = 256;   // ... up to this many per CTA and phase (more: the warp walks them)

__device__ __forceinline__ void wing_grid_sync(unsigned long long* bar, unsigned long long& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    epoch += gridDim.x;
    __threadfence();
    atomicAdd(bar, 1ull);
    while (*(volatile unsigned long long*)bar < epoch) {
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kWingThreads, 1) k_wing_peel(WingArgs w, uint32_t* live0, uint32_t* live1,
                                                                  uint32_t* sx0, uint32_t* sx1, uint32_t* cand0,
                                                                  uint32_t* cand1, WingDev* c) {
  const uint32_t ln = lane_id();
  const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  const bool lead = gt == 0;
  unsigned long long epoch = 0, k = 0, levels = 0, rounds = 0;
  uint32_t* live[2] = {live0, live1};
  uint32_t* SX[2] = {sx0, sx1};
  uint32_t* Cand[2] = {cand0, cand1};
  uint32_t nlive = (uint32_t)w.m, cur = 0;
  __shared__ uint32_t big[kWingBigCap];  // per CTA: long pair lists left to the whole CTA (edge / bloom,
  __shared__ uint32_t biglen[kWingBigCap], bigpre[kWingBigCap], bigkb[kWingBigCap], bigd[kWingBigCap];  // length, prefix, k_B, d)
  __shared__ uint32_t scanbuf[33];
  __shared__ uint32_t nbig;
  const uint32_t wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  unsigned long long clk[4] = {0, 0, 0, 0};
  long long tc = clock64();
  auto lap = [&](int i) {
    const long long t = clock64();
    clk[i] += (unsigned long long)(t - tc);
    tc = t;
  };
  for (;;) {
    // --- level scan: compact the live list, minimum live support
    {
      const uint32_t* in = live[cur];
      uint32_t* out = live[cur ^ 1];
      unsigned long long mn = ~0ull;
      for (uint64_t i0 = gt - ln; i0 < nlive; i0 += nt) {
        const uint64_t i = i0 + ln;
        bool keep = false;
        uint32_t e = 0;
        if (i < nlive) {
          e = __ldcg(in + i);
          keep = __ldcg(w.alive + e);
          if (keep) mn = min(mn, __ldcg(w.sup + e));
        }
        warp_append(keep, e, out, &c->nlive);
      }
      mn = warp_min_u64(mn);
      if (ln == 0 && mn != ~0ull) atomicMin(&c->minsup, mn);
    }
    wing_grid_sync(&c->bar, epoch);
    lap(0);
    cur ^= 1;
    nlive = *(volatile uint32_t*)&c->nlive;
    if (nlive == 0) break;
    k = max(k, *(volatile unsigned long long*)&c->minsup);
    // --- candidate band: the levels k .. B are peeled from the candidate list C = live edges
    // with support <= B (an edge whose support falls to <= B later is appended by the update
    // that takes it there), so the next level is the minimum over C, not over the live list:
    // the full scan above runs once per band instead of once per level
    const unsigned long long B = k + max(16ull, k >> 2);
    // S = live edges with support <= k, C = ... <= B (every listed edge is alive)
    for (uint64_t i0 = gt - ln; i0 < nlive; i0 += nt) {
      const uint64_t i = i0 + ln;
      bool take = false, cand = false;
      uint32_t e = 0;
      if (i < nlive) {
        e = __ldcg(live[cur] + i);
        const unsigned long long s = __ldcg(w.sup + e);
        take = s <= k;
        cand = s <= B;
      }
      warp_append(take, e, SX[0], &c->cnt[0]);
      warp_append(cand, e, Cand[0], &c->cntC[0]);
    }
    wing_grid_sync(&c->bar, epoch);
    lap(1);
    if (lead) {  // every thread read them before the barrier above
      c->nlive = 0;
      c->minsup = ~0ull;
    }
    uint32_t cc = 0;
    for (;;) {  // levels of the band
    levels++;
    uint32_t cs = 0;
    bool any = false;
    for (;;) {
      const uint32_t nS = *(volatile uint32_t*)&c->cnt[cs];
      if (nS == 0) break;
      any = true;
      const uint32_t r = (uint32_t)(rounds & 1);
      rounds++;
      // --- claim (k_wing_claim) + kill: the claim reads no `alive`, so S leaves here
      if (lead) c->nT[r ^ 1] = 0;
      const uint32_t* S = SX[cs];
      auto claim = [&](uint64_t j) {
        const uint32_t p = w.inc[j];
        if (__ldcg(w.pstate + p) != 0 || atomicCAS(&w.pstate[p], 0u, 1u) != 0u) return;
        const uint32_t b = w.pair_bloom[p];
        if (atomicAdd(&w.bloom_d[b], 1u) == 0) w.T[atomicAdd(&c->nT[r], 1u)] = b;
      };
      // S edges go round-robin over the CTAs (edge i to CTA i mod grid), a warp per edge;
      // pair lists longer than a warp step are left to the whole CTA, which walks all of
      // its deferred lists as one flattened range (a warp walking 10^3..10^5 pairs alone,
      // three dependent loads per step, set the length of the round)
      if (threadIdx.x == 0) nbig = 0;
      __syncthreads();
      for (uint64_t i = blockIdx.x + (uint64_t)gridDim.x * wib; i < nS; i += (uint64_t)gridDim.x * nwb) {
        const uint32_t e = __ldcg(S + i);
        if (ln == 0) {
          w.theta[e] = k;
          w.alive[e] = 0;
        }
        const uint64_t j0 = w.inc_off[e], j1 = w.inc_off[e + 1];
        uint32_t slot = kWingBigCap;
        if (j1 - j0 > kWingBigLen && j1 - j0 <= kWingBigMax) {
          if (ln == 0) slot = atomicAdd(&nbig, 1u);
          slot = __shfl_sync(kFull, slot, 0);
          if (slot < kWingBigCap) {
            if (ln == 0) {
              big[slot] = e;
              biglen[slot] = (uint32_t)(j1 - j0);
            }
            continue;
          }
        }
        for (uint64_t j = j0 + ln; j < j1; j += 32) claim(j);
      }
      __syncthreads();
      {
        const uint32_t n = min(nbig, kWingBigCap);
        uint32_t tot;
        const uint32_t pre = block_excl_scan(threadIdx.x < n ? biglen[threadIdx.x] : 0u, scanbuf, &tot);
        if (threadIdx.x < n) bigpre[threadIdx.x] = pre;
        __syncthreads();
        for (uint32_t f = threadIdx.x; f < tot; f += blockDim.x) {
          uint32_t lo = 0, hi = n;  // largest j with bigpre[j] <= f
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (bigpre[mid] <= f) lo = mid; else hi = mid;
          }
          claim(w.inc_off[big[lo]] + (f - bigpre[lo]));
        }
      }
      wing_grid_sync(&c->bar, epoch);
      lap(2);
      // --- batch bloom update (k_wing_update); crossers go to SX[cs ^ 1]
      const uint32_t nT = *(volatile uint32_t*)&c->nT[r];
      if (lead) c->cnt[cs] = 0;
      uint32_t* X = SX[cs ^ 1];
      uint32_t* nX = &c->cnt[cs ^ 1];
      uint32_t* CL = Cand[cc];
      uint32_t* nCL = &c->cntC[cc];
      auto dec = [&](uint32_t x, unsigned long long d) {
        const unsigned long long old = atomicAdd(&w.sup[x], (unsigned long long)(0ull - d));
        if (old > k && old - d <= k) X[atomicAdd(nX, 1u)] = x;
        if (old > B && old - d <= B) CL[atomicAdd(nCL, 1u)] = x;  // enters the band
      };
      auto upd_pair = [&](uint64_t p, uint32_t kb, uint32_t d) {
        const uint32_t st = __ldcg(w.pstate + p);
        if (st == 2) return;
        const uint2 pr = w.pair[p];
        if (st == 1) {
          if (kb > 1) {
            if (__ldcg(w.alive + pr.x)) dec(pr.x, kb - 1);
            if (__ldcg(w.alive + pr.y)) dec(pr.y, kb - 1);
          }
          w.pstate[p] = 2;
        } else {
          dec(pr.x, d);
          dec(pr.y, d);
        }
      };
      if (threadIdx.x == 0) nbig = 0;
      __syncthreads();
      for (uint64_t i = blockIdx.x + (uint64_t)gridDim.x * wib; i < nT; i += (uint64_t)gridDim.x * nwb) {
        const uint32_t b = __ldcg(w.T + i);
        const uint64_t p0 = w.bloom_off[b], p1 = w.bloom_off[b + 1];
        const uint32_t kb = __ldcg(w.bloom_k + b), d = __ldcg(w.bloom_d + b);
        uint32_t slot = kWingBigCap;
        if (p1 - p0 > kWingBigLen && p1 - p0 <= kWingBigMax) {  // a bloom of more than a warp step: the whole CTA, flattened (below)
          if (ln == 0) slot = atomicAdd(&nbig, 1u);
          slot = __shfl_sync(kFull, slot, 0);
          if (slot < kWingBigCap) {
            if (ln == 0) {
              big[slot] = b;
              biglen[slot] = (uint32_t)(p1 - p0);
              bigkb[slot] = kb;
              bigd[slot] = d;
            }
            continue;
          }
        }
        for (uint64_t p = p0 + ln; p < p1; p += 32) upd_pair(p, kb, d);
        __syncwarp();
        if (ln == 0) {
          w.bloom_k[b] = kb - d;
          w.bloom_d[b] = 0;
        }
      }
      __syncthreads();
      {
        const uint32_t n = min(nbig, kWingBigCap);
        uint32_t tot;
        const uint32_t pre = block_excl_scan(threadIdx.x < n ? biglen[threadIdx.x] : 0u, scanbuf, &tot);
        if (threadIdx.x < n) bigpre[threadIdx.x] = pre;
        __syncthreads();
        for (uint32_t f = threadIdx.x; f < tot; f += blockDim.x) {
          uint32_t lo = 0, hi = n;
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (bigpre[mid] <= f) lo = mid; else hi = mid;
          }
          upd_pair(w.bloom_off[big[lo]] + (f - bigpre[lo]), bigkb[lo], bigd[lo]);
        }
        if (threadIdx.x < n) {  // kb and d of the deferred blooms were taken before any pair was updated
          w.bloom_k[big[threadIdx.x]] = bigkb[threadIdx.x] - bigd[threadIdx.x];
          w.bloom_d[big[threadIdx.x]] = 0;
        }
      }
      wing_grid_sync(&c->bar, epoch);
      lap(3);
      cs ^= 1;
    }
    if (!any) wing_grid_sync(&c->bar, epoch);  // (cannot happen: the minimum is selected) keeps the reset ordered
    // --- next level: compact the candidates (drop the peeled), minimum live support among them
    {
      const uint32_t nC = *(volatile uint32_t*)&c->cntC[cc];
      unsigned long long mn = ~0ull;
      for (uint64_t i0 = gt - ln; i0 < nC; i0 += nt) {
        const uint64_t i = i0 + ln;
        bool keep = false;
        uint32_t e = 0;
        if (i < nC) {
          e = __ldcg(Cand[cc] + i);
          keep = __ldcg(w.alive + e);
          if (keep) mn = min(mn, __ldcg(w.sup + e));
        }
        warp_append(keep, e, Cand[cc ^ 1], &c->cntC[cc ^ 1]);
      }
      mn = warp_min_u64(mn);
      if (ln == 0 && mn != ~0ull) atomicMin(&c->minC, mn);
    }
    wing_grid_sync(&c->bar, epoch);
    lap(0);
    const uint32_t nC2 = *(volatile uint32_t*)&c->cntC[cc ^ 1];
    const unsigned long long mnC = *(volatile unsigned long long*)&c->minC;
    if (nC2 == 0 || mnC > B) {
      // band exhausted: back to a full scan.  The barrier orders every thread's reads of the
      // counters before their reset; the scan phase does not touch them.
      wing_grid_sync(&c->bar, epoch);
      if (lead) {
        c->cntC[0] = 0;
        c->cntC[1] = 0;
        c->minC = ~0ull;
      }
      break;
    }
    k = mnC;  // > the level just finished: everything <= it was peeled
    cc ^= 1;
    {
      const uint32_t* CLs = Cand[cc];
      for (uint64_t i0 = gt - ln; i0 < nC2; i0 += nt) {
        const uint64_t i = i0 + ln;
        bool take = false;
        uint32_t e = 0;
        if (i < nC2) {
          e = __ldcg(CLs + i);
          take = __ldcg(w.sup + e) <= k;
        }
        warp_append(take, e, SX[0], &c->cnt[0]);
      }
    }
    wing_grid_sync(&c->bar, epoch);
    lap(1);
    if (lead) {  // every thread read them before the barrier above; the rounds do not touch them
      c->cntC[cc ^ 1] = 0;
      c->minC = ~0ull;
    }
    }  // levels of the band
  }
  if (lead) {
    c->levels = levels;
    c->rounds = rounds;
    for (int i = 0; i < 4; i++) c->clk[i] = clk[i];
  }
}

// θ back to the caller's CSR order (positions found as in k_edge_gather)
__global__ void k_wing_gather(uint32_t nX, uint64_t m, const uint64_t* __restrict__ offX,
                              const uint32_t* __restrict__ idxX, const uint32_t* __restrict__ rankX,
                              const uint32_t* __restrict__ rankY, const uint64_t* __restrict__ offXr,
                              const uint32_t* __restrict__ adjXr, const uint64_t* __restrict__ val,
                              uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nX;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (offX[mid] <= i) lo = mid; else hi = mid;
    }
    const uint32_t rx = rankX[lo], ry = rankY[idxX[i]];
    const uint64_t bx = offXr[rx];
    out[i] = val[bx + edge_lower_bound(adjXr + bx, (uint32_t)(offXr[rx + 1] - bx), ry)];
  }
}

}  // namespace pbng
