// kernels_cd.cuh — counting and coarse-grained decomposition (CD) kernels.
//
// Paper: Lakhotia, Kannan, Prasanna, arXiv 2110.12511 ("P:n" = PAPER.md line).
//   wedge aggregation / counting     P:369-391, Alg.1
//   CD tip peeling                   P:743-790, Alg.4, tip P:982-991
//   range determination              P:818-826, tip P:1387-1391
//   batch re-count
//   dynamic graph updates
#pragma once
#include "device_common.cuh"

namespace pbng {

// Per-warp / per-CTA hash capacities (slots are power-of-two; load factor <= 1/2).
constexpr uint32_t kWarpSlots = 1024;           // tier 0: one warp per u
constexpr uint32_t kWarpCap = kWarpSlots / 2;   // partners bound for tier 0
#ifndef PBNG_MID_LOG_SLOTS
#define PBNG_MID_LOG_SLOTS 13
#endif
constexpr uint32_t kLogCtaSlots = PBNG_MID_LOG_SLOTS;
constexpr uint32_t kCtaSlots = 1u << kLogCtaSlots;  // tier 1: one CTA per u
constexpr uint32_t kCtaCap = kCtaSlots / 2;          // partners bound for tier 1
constexpr uint32_t kWarpTierThreads = 256;
constexpr uint32_t kHeavyThreads = 512;
constexpr uint32_t kClassBig = 2048;            // classify: degree handled by a whole CTA
// Range histogram: 16-bit-style log-scale keys of the 64-bit support
// (exact below 256; 8 mantissa bits above), weighted by the static wedge work.
constexpr uint32_t kBins = 14336;
__host__ __device__ __forceinline__ uint32_t support_key(uint64_t s) {
  if (s < 256) return (uint32_t)s;
  if (s >> 63) return kBins - 1;  // (unreachable for real counts) keep the key inside the histogram
#ifdef __CUDA_ARCH__
  uint32_t e = 63 - __clzll((long long)s);
#else
  uint32_t e = 63 - __builtin_clzll(s);
#endif
  return 256 + (e - 8) * 256 + (uint32_t)((s >> (e - 8)) & 255);
}
// smallest support value mapped to key b (b <= kBins)
__host__ __device__ __forceinline__ uint64_t key_lo(uint32_t b) {
  if (b < 256) return b;
  uint32_t q = (b - 256) / 256, mnt = (b - 256) % 256, e = q + 8;
  if (e >= 64) return ~0ull;
  return ((uint64_t)(256 + mnt)) << (e - 8);
}

struct Counters {
  // reset every CD iteration (host memsets [0, offsetof(ntouched)))
  uint32_t nF;                   // frontier size (select)
  uint32_t ntier[3];             // tier list sizes (classify)
  uint32_t ticket[4];            // dynamic work tickets of the aggregation kernels
  uint32_t nbig;                 // classify: vertices left to k_classify_big
  uint32_t pad1;
  unsigned long long wedges;     // Σ wl over classified work (traversal, incl. u' = u)
  unsigned long long sel_wc;     // Σ wc over selected (range-target adaptation)
  // managed by the host loop
  uint32_t ntouched;             // touched V vertices (classify, CD)
  uint32_t pad0;
  unsigned long long live_wc;    // range pass: Σ wc over live
  unsigned long long live_n;     // range pass: live count
  unsigned long long max_live;   // range pass: 1 + largest live id
  // cumulative
  unsigned long long updates;    // C(w,2) decrements
  unsigned long long updates_live;  // ... of which to partners still live (counted with PBNG_OPT_STATS only)
  unsigned long long ld2_drop;   // compaction: decrease of Σ_v ld_v^2
  unsigned long long cum_wedges; // Σ of every classify's wedges
  unsigned long long cum_steps;  // Σ d_u of every traversed u ((u, v) steps)
  unsigned long long tier_wedges[3];  // Σ wl routed to each tier
  unsigned long long dbg[4];          // tier-2 internals: bitmap windows, overflows, dense passes, -
  unsigned long long prof[4];         // tier-2 clock64 of CTA thread 0: starts with tables, precompute, bitmap windows, dense passes
  unsigned long long prof2[4];        // tier-2: cycles / count of starts without tables, count of starts with tables, -
  unsigned long long hashc[4];        // tier 1: starts, starts split into groups, groups, starts passed on to tier 2
  unsigned long long prof3[8];        // tier-2 dense windows (PBNG_TRACE): cycles of sub-bound tables, marking, sweep;
                                      // entries, windows, Σ lists per pass; marking set-up cycles, marking loop cycles
};

// ---------------------------------------------------------------- init
// live degree of every v, and Σ_v d_v^2 (one-sided re-count cost, g10)
__global__ void k_init_v(uint32_t nV, const uint64_t* __restrict__ offV, uint32_t* __restrict__ ld,
                         unsigned long long* sum_d2) {
  unsigned long long acc = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nV; v += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t d = (uint32_t)(offV[v + 1] - offV[v]);
    ld[v] = d;
    acc += (unsigned long long)d * d;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && acc) atomicAdd(sum_d2, acc);
}

// wc[u] = Σ_{v ∈ N_u} d_v : static wedge work of peeling u (proxy 2; g5),
// and ∧_cnt = Σ_(u,v) min(d_u, d_v), the re-count cost.
__global__ void k_init_u(uint32_t nU, const uint64_t* __restrict__ offU, const uint32_t* __restrict__ adjU,
                         const uint64_t* __restrict__ offV, uint64_t* __restrict__ wc,
                         uint32_t* __restrict__ part, unsigned long long* sum_min) {
  const uint32_t ln = lane_id();
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long smin = 0;
  for (uint64_t u = gw; u < nU; u += nw) {
    uint64_t s = 0;
    const uint64_t du = offU[u + 1] - offU[u];
    for (uint64_t e = offU[u] + ln; e < offU[u + 1]; e += 32) {
      uint32_t v = adjU[e];
      const uint64_t d = offV[v + 1] - offV[v];
      s += d;
      smin += d < du ? d : du;
    }
    s = warp_sum(s);
    if (ln == 0) {
      wc[u] = s;
      part[u] = kUnassigned;
    }
  }
  smin = warp_sum(smin);
  if (ln == 0 && smin) atomicAdd(sum_min, smin);
}

// ---------------------------------------------------------------- classify
// For each listed u (or every unassigned u when list == nullptr) compute
// wl = Σ_{v∈N_u} ld[v] (wedges its traversal reads) and route it to a tier by
// the partner bound pb = wl - d_u.  Vertices that cannot decrement anybody
// (d_u < 2, pb == 0, or — peeling — exact support 0) are not traversed; in
// COUNT mode their support is written as 0 here.  Optionally tags every
// v ∈ N_u with the iteration's epoch (plain store; k_collect_touched lists
// them for the deletion pass).
// A warp takes 32 vertices and walks their edges as one flattened range
// (binary search over the lanes' inclusive degree scan), so every lane issues
// independent loads regardless of the degree mix.
template <int MODE>
__global__ void k_classify(uint32_t nU, const uint32_t* __restrict__ list, const uint32_t* __restrict__ count,
                           const uint64_t* __restrict__ offU, const uint32_t* __restrict__ adjU,
                           const uint32_t* __restrict__ ld, const uint32_t* __restrict__ part,
                           uint64_t* __restrict__ support, uint2* tier0, uint2* tier1, uint2* tier2,
                           uint2* bigq, uint32_t* vflag, uint32_t epoch, Counters* c, uint32_t hmax,
                           uint32_t dlim) {
  __shared__ unsigned long long s_acc[8][32];  // launched with 256 threads
  const uint32_t ln = lane_id(), wib = threadIdx.x >> 5;
  unsigned long long* acc = s_acc[wib & 7];
  const uint32_t n = list ? *count : nU;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long wsum = 0, ssum = 0, tw[3] = {0, 0, 0};
  // a warp takes G <= 32 vertices at a time: with fewer than 32 vertices per warp in
  // the batch (late CD iterations) G shrinks, so that every warp gets some and the
  // serial chain of dependent loads (adjU -> ld) per warp is as short as the batch allows
  const uint32_t G = n >= nw * 32 ? 32u : (uint32_t)max((unsigned long long)((n + nw - 1) / nw), 1ull);
  for (uint64_t b = gw * G; b < n; b += nw * G) {
    const uint64_t idx = b + ln;
    bool ok = ln < G && idx < n;
    const uint32_t u = ok ? (list ? list[idx] : (uint32_t)idx) : 0u;
    if (ok && !list && part[u] != kUnassigned) ok = false;
    const uint64_t e0 = ok ? offU[u] : 0, d0 = ok ? offU[u + 1] - e0 : 0;
    // hub vertices are summed by a whole CTA (k_classify_big)
    const bool big = d0 > kClassBig;
    warp_append2(big, make_uint2(u, 0), bigq, &c->nbig);
    if (big) ok = false;
    const uint64_t d = ok ? d0 : 0;
    acc[ln] = 0;
    // inclusive scan of degrees over the warp (64-bit: a warp may hold hubs)
    uint64_t incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, incl, o);
      if (ln >= (uint32_t)o) incl += y;
    }
    const uint64_t total = __shfl_sync(kFull, incl, 31);
    const uint64_t excl = incl - d;
    __syncwarp();
    for (uint64_t t0 = 0; t0 < total; t0 += 32) {
      const uint64_t t = t0 + ln;
      uint32_t j = 0;
#pragma unroll
      for (uint32_t s2 = 16; s2 > 0; s2 >>= 1) {
        const uint64_t y = __shfl_sync(kFull, incl, j + s2 - 1);
        if (y <= t) j += s2;
      }
      const uint64_t je = __shfl_sync(kFull, e0, j), jx = __shfl_sync(kFull, excl, j);
      const bool valid = t < total;
      unsigned long long val = 0;
      if (valid) {
        const uint32_t v = adjU[je + (t - jx)];
        val = ld[v];
        if (vflag) atomicAdd(&vflag[v], 1u);  // one more peeled entry in N_v
      }
      // segmented sum over lanes with the same vertex j (contiguous in lane order)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFull, val, o);
        const uint32_t yj = __shfl_up_sync(kFull, j, o);
        if (ln >= (uint32_t)o && yj == j) val += y;
      }
      const uint32_t nj = __shfl_down_sync(kFull, j, 1);
      if (valid && (ln == 31 || nj != j || t + 1 >= total)) acc[j] += val;
      __syncwarp();
    }
    __syncwarp();
    const uint64_t s = acc[ln];
    int tier = -1;
    uint32_t pb = 0;
    if (ok) {
      const uint64_t pb64 = s - d;  // u itself appears once in each of its lists
      bool work = d >= 2 && pb64 > 0;
      if (MODE == 1 && work) work = support[u] != 0;
      if (work) {
        pb = pb64 > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)pb64;
        tier = pb <= kWarpCap ? 0 : (pb <= hmax && d < dlim) ? 1 : 2;
        wsum += s;
        ssum += d;
        tw[tier] += s;
      } else if (MODE == 0) {
        support[u] = 0;
      }
    }
    const uint2 item = make_uint2(u, pb);
    warp_append2(tier == 0, item, tier0, &c->ntier[0]);
    warp_append2(tier == 1, item, tier1, &c->ntier[1]);
    warp_append2(tier == 2, item, tier2, &c->ntier[2]);
    __syncwarp();
  }
  // counters: warp sums, then one set of atomics per CTA (all of them hit one
  // cache line, so per-warp atomics from every warp would serialise in L2)
  __shared__ unsigned long long s_red[5][8];
  wsum = warp_sum(wsum);
  ssum = warp_sum(ssum);
  tw[0] = warp_sum(tw[0]);
  tw[1] = warp_sum(tw[1]);
  tw[2] = warp_sum(tw[2]);
  if (ln == 0) {
    s_red[0][wib] = wsum;
    s_red[1][wib] = ssum;
    s_red[2][wib] = tw[0];
    s_red[3][wib] = tw[1];
    s_red[4][wib] = tw[2];
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    unsigned long long s = 0;
    for (uint32_t w = 0; w < (blockDim.x >> 5); w++) s += s_red[threadIdx.x][w];
    if (s) {
      if (threadIdx.x == 0) {
        atomicAdd(&c->wedges, s);
        atomicAdd(&c->cum_wedges, s);
      } else if (threadIdx.x == 1) {
        atomicAdd(&c->cum_steps, s);
      } else {
        atomicAdd(&c->tier_wedges[threadIdx.x - 2], s);
      }
    }
  }
}

// The vertices k_classify deferred (degree > kClassBig): one CTA per vertex.
template <int MODE>
__global__ void __launch_bounds__(512) k_classify_big(const uint2* __restrict__ bigq, const Counters* cnt,
                                                     const uint64_t* __restrict__ offU,
                                                     const uint32_t* __restrict__ adjU,
                                                     const uint32_t* __restrict__ ld, uint64_t* __restrict__ support,
                                                     uint2* tier0, uint2* tier1, uint2* tier2, uint32_t* vflag,
                                                     uint32_t epoch,
                                                     Counters* c, uint32_t hmax, uint32_t dlim) {
  __shared__ unsigned long long s_part[16];
  const uint32_t n = cnt->nbig;
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint32_t u = bigq[i].x;
    const uint64_t e0 = offU[u], d = offU[u + 1] - e0;
    unsigned long long s = 0;
    for (uint64_t k = threadIdx.x; k < d; k += blockDim.x) {
      const uint32_t v = adjU[e0 + k];
      s += ld[v];
      if (vflag) atomicAdd(&vflag[v], 1u);
    }
    s = warp_sum(s);
    if (lane_id() == 0) s_part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      s = 0;
      for (uint32_t w = 0; w < (blockDim.x >> 5); w++) s += s_part[w];
      const uint64_t pb64 = s - d;
      bool work = d >= 2 && pb64 > 0;
      if (MODE == 1 && work) work = support[u] != 0;
      if (work) {
        const uint32_t pb = pb64 > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)pb64;
        const int tier = pb <= kWarpCap ? 0 : (pb <= hmax && d < dlim) ? 1 : 2;
        uint2* tl = tier == 0 ? tier0 : tier == 1 ? tier1 : tier2;
        tl[atomicAdd(&c->ntier[tier], 1u)] = make_uint2(u, pb);
        atomicAdd(&c->wedges, s);
        atomicAdd(&c->cum_wedges, s);
        atomicAdd(&c->cum_steps, (unsigned long long)d);
        atomicAdd(&c->tier_wedges[tier], s);
      } else if (MODE == 0) {
        support[u] = 0;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- aggregation
// MODE 0 (COUNT): support[u] = Σ_{u' unassigned, u' != u} C(w(u,u'),2)
// MODE 1 (PEEL):  for u in the frontier, every unassigned u' with w >= 2:
//                 support[u'] -= C(w(u,u'),2)   (tip batch update, P:987-991:
//                 updates from different frontier vertices touch disjoint
//                 butterflies, so they are summed atomically; no floor needed)
// MODE 2 (LINK):  for every member u of a tip level, every member u' with
//                 w(u,u') >= 2 (one butterfly {u,u'} at least) joins u's
//                 union-find set (k-tip components)
struct AggArgs {
  const uint64_t* __restrict__ offU;
  const uint32_t* __restrict__ adjU;
  const uint64_t* __restrict__ offV;
  const uint32_t* __restrict__ adjV;  // live adjacency (prefix ld[v] of each list)
  const uint32_t* __restrict__ ld;
  const uint32_t* __restrict__ part;
  uint64_t* support;
  const uint2* __restrict__ list;
  const uint32_t* __restrict__ count;
  uint32_t nU;
  uint32_t* ticket;      // dynamic scheduling counter (tiers 1-2)
  Counters* c;
  // vertex-priority counting (kernels_vp.cuh)
  const uint32_t* __restrict__ cutV;   // per v: live entries of N_v ranked above v (Alg.1 l.10)
  const uint32_t* __restrict__ cutU;   // per u: entries of N_u ranked above u
  // tier 2 (agg_win.cuh): per-CTA window-bound scratch
  uint32_t* win_bnd;
  uint64_t win_cap;
  uint32_t win_split;                  // window groups per tier-2 start (>1 for small batches)
  uint32_t win_pre;                    // starts with at most this many lists use precomputed window tables
  bool win_prof;                       // accumulate tier-2 phase clocks (PBNG_TRACE)
  uint32_t* cc;                        // LINK: union-find parents (k-tip components)
  const uint32_t* __restrict__ cut_e;  // LINK: per U-edge (u, v), members of N_v with id < u
  uint32_t idspace;                    // tier-2 windows cover partner ids [0, idspace) (COUNT, PEEL)
  // tier 1 (agg_hash.cuh): window-bound rows of long lists, degree-mass windows, count-field bits
  const uint32_t* __restrict__ rowid;
  const uint32_t* __restrict__ rows;
  const uint32_t* __restrict__ wb;
  uint32_t cb;
  uint2* tier2;                        // starts tier 1 passes on (a window above its capacity)
  uint32_t* ntier2;
  bool stats;                          // PEEL: also count decrements to live partners (A_live)
};

// Partner lists of the aggregation tiers: the live prefix of N_v (COUNT, PEEL),
// or only its members ranked before the start (LINK: a pair is linked once,
// from its larger id, so each wedge pair is walked once instead of twice)
template <int MODE>
__device__ __forceinline__ auto agg_lists(const AggArgs& a) {
  if constexpr (MODE == 2) {
    return PrefixLists{a.adjU, a.offV, a.cut_e};
  } else {
    return CdLists{a.adjU, a.offV, a.ld};
  }
}

template <int MODE>
__device__ __forceinline__ void emit(const AggArgs& a, uint32_t u, uint32_t k, uint32_t w, uint64_t& acc,
                                     unsigned long long& upd) {
  // PEEL skips the liveness test: a peeled partner's support is never read again
  // (selection, snapshots and FD only read live vertices), so decrementing it is
  // harmless and saves a random load per emitted pair.  With stats on, the
  // decrements that reach live partners are counted separately (bits 36..63 of
  // upd; flush_updates splits them): A_live of the roofline.
  PBNG_DCHECK(k < a.nU && (MODE == 0 || k != u));
  if (w >= 2 && (MODE == 1 || a.part[k] == kUnassigned)) {
    const uint64_t d = choose2(w);
    if (MODE == 0) {
      acc += d;
    } else if (MODE == 1) {
      red_add_u64(&a.support[k], 0ull - d);
      upd += (a.stats && a.part[k] == kUnassigned) ? (1ull << 36) + 1ull : 1ull;
    } else {
      cc_union(a.cc, u, k);  // u and k share a butterfly inside the level
    }
  }
}

// Per-thread update counts -> Counters (whole warp, converged): low 36 bits all
// decrements, high 28 bits the live ones; the fields are summed separately over
// the warp, so the split is exact while one thread's totals in one launch stay
// below 2^36 / 2^28 (a CD launch emits ~10^9 decrements over ~10^5 threads).
__device__ __forceinline__ void flush_updates(const AggArgs& a, unsigned long long upd) {
  const unsigned long long all = warp_sum(upd & ((1ull << 36) - 1)), live = warp_sum(upd >> 36);
  if (lane_id() == 0) {
    if (all) atomicAdd(&a.c->updates, all);
    if (live) atomicAdd(&a.c->updates_live, live);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kWarpTierThreads) k_agg_warp(AggArgs a) {
  extern __shared__ uint32_t sm[];
  const uint32_t w = threadIdx.x >> 5, ln = lane_id();
  uint32_t* keys = sm + w * (2 * kWarpSlots);
  uint32_t* vals = keys + kWarpSlots;
  for (uint32_t s = ln; s < kWarpSlots; s += 32) {
    keys[s] = kEmpty;
    vals[s] = 0;
  }
  __syncwarp();
  const uint32_t n = *a.count;
  const auto L = agg_lists<MODE>(a);
  unsigned long long upd = 0;
  const uint32_t wpb = blockDim.x >> 5;
  for (uint32_t i = blockIdx.x * wpb + w; i < n; i += gridDim.x * wpb) {
    const uint2 it = a.list[i];
    const uint32_t u = it.x;
    uint32_t logT = ceil_log2(2 * it.y);
    logT = logT < 5 ? 5 : logT;
    auto f = [&](bool ok, uint32_t x, uint64_t) {
      if (ok && x != u) hash_insert(keys, vals, logT, x);
    };
    warp_wedges(L, a.offU[u], a.offU[u + 1], a.adjV, f);
    __syncwarp();
    uint64_t acc = 0;
    const uint32_t T = 1u << logT;
    for (uint32_t s = ln; s < T; s += 32) {
      const uint32_t k = keys[s];
      if (k != kEmpty) {
        const uint32_t wv = vals[s];
        keys[s] = kEmpty;
        vals[s] = 0;
        emit<MODE>(a, u, k, wv, acc, upd);
      }
    }
    if (MODE == 0) {
      acc = warp_sum(acc);
      if (ln == 0) a.support[u] = acc;
    }
    __syncwarp();
  }
  if (MODE == 1) flush_updates(a, upd);
}

#include "agg_mid.cuh"
#include "agg_win.cuh"
#include "agg_hash.cuh"

// ---------------------------------------------------------------- range pass
// Partition start (Alg.4 l.5-8): snapshot ⋈^init = support for all
// live u and build the wedge-work-weighted histogram of current supports
// (find_range bins; tip bins keyed by support P:1387-1391).
__global__ void __launch_bounds__(1024) k_range_hist(uint32_t nU, const uint32_t* __restrict__ part,
                                                     const uint64_t* __restrict__ support,
                                                     const uint64_t* __restrict__ wc, uint64_t* __restrict__ init,
                                                     unsigned long long* ghist_w, uint32_t* ghist_n, Counters* c) {
  extern __shared__ unsigned long long hsm[];
  unsigned long long* hw = hsm;
  uint32_t* hn = (uint32_t*)(hsm + kBins);
  for (uint32_t b = threadIdx.x; b < kBins; b += blockDim.x) {
    hw[b] = 0;
    hn[b] = 0;
  }
  __syncthreads();
  unsigned long long tw = 0, tn = 0, mx = 0;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nU; u += (uint64_t)gridDim.x * blockDim.x) {
    if (part[u] != kUnassigned) continue;
    mx = u + 1;
    const uint64_t s = support[u];
    init[u] = s;
    const uint32_t k = support_key(s);
    const uint64_t w = wc[u];
    if (w) atomicAdd(&hw[k], (unsigned long long)w);
    atomicAdd(&hn[k], 1u);
    tw += w;
    tn++;
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < kBins; b += blockDim.x) {
    if (hn[b]) {
      atomicAdd(&ghist_n[b], hn[b]);
      if (hw[b]) atomicAdd(&ghist_w[b], hw[b]);
    }
  }
  tw = warp_sum(tw);
  tn = warp_sum(tn);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  if (lane_id() == 0 && tn) {
    atomicAdd(&c->live_wc, tw);
    atomicAdd(&c->live_n, tn);
    atomicMax(&c->max_live, mx);
  }
}

// ---------------------------------------------------------------- frontier
// activeSet = { live u : support[u] < bound }  (Alg.4 l.9/l.13),
// assigned to partition pid.  Warp ballots + block-wide scan give one global
// atomic per CTA tile for the compacted list.
__global__ void __launch_bounds__(256) k_select(uint32_t nU, uint32_t* __restrict__ part,
                                                const uint64_t* __restrict__ support,
                                                const uint64_t* __restrict__ wc, uint64_t bound, uint32_t pid,
                                                uint32_t* __restrict__ F, Counters* c) {
  __shared__ uint32_t s_scan[33];
  __shared__ uint32_t s_base;
  unsigned long long swc = 0;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x; b < nU; b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = b + threadIdx.x;
    bool sel = false;
    if (u < nU && part[u] == kUnassigned && support[u] < bound) sel = true;
    uint32_t total;
    const uint32_t r = block_excl_scan(sel ? 1u : 0u, s_scan, &total);
    if (total) {
      if (threadIdx.x == 0) s_base = atomicAdd(&c->nF, total);
      __syncthreads();
      if (sel) {
        F[s_base + r] = (uint32_t)u;
        part[u] = pid;
        swc += wc[u];
      }
      __syncthreads();
    }
  }
  __shared__ unsigned long long s_red[8];  // launched with 256 threads: one atomic per CTA
  swc = warp_sum(swc);
  if (lane_id() == 0) s_red[threadIdx.x >> 5] = swc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (uint32_t w = 0; w < (blockDim.x >> 5); w++) s += s_red[w];
    if (s) atomicAdd(&c->sel_wc, s);
  }
}

// ---------------------------------------------------------------- deletion
// Lazy deletion: vflag[v] counts the entries of N_v peeled since its last
// compaction.  A list is compacted now when it is short (< big), when at least
// 1/8 of its live prefix is peeled, or when forced (partition end: FD needs
// every list grouped by partition).  Stale entries in a live prefix are
// harmless to the aggregation (peeled partners are filtered when emitting).
__global__ void __launch_bounds__(256) k_collect_touched(uint32_t nV, uint32_t* __restrict__ vflag,
                                                         const uint32_t* __restrict__ ld, uint32_t big, bool force,
                                                         uint32_t* __restrict__ touched, Counters* c) {
  __shared__ uint32_t s_scan[33];
  __shared__ uint32_t s_base;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x; b < nV; b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = b + threadIdx.x;
    const uint32_t dead = v < nV ? vflag[v] : 0u;
    bool t = dead > 0;
    if (t && !force) {
      const uint32_t L = ld[v];
      t = L < big || (uint64_t)dead * 8 >= L;
    }
    if (t) vflag[v] = 0;
    uint32_t total;
    const uint32_t r = block_excl_scan(t ? 1u : 0u, s_scan, &total);
    if (total) {
      if (threadIdx.x == 0) s_base = atomicAdd(&c->ntouched, total);
      __syncthreads();
      if (t) touched[s_base + r] = (uint32_t)v;
      __syncthreads();
    }
  }
}

// Dynamic graph update: for every touched v, stable-partition
// the live prefix of N_v into [still live | newly peeled]; the peeled block is
// placed directly after the live prefix, so over the whole CD each N_v ends as
// [U_last | ... | U_1] — grouped by partition, which is the induced-subgraph
// layout FD needs.  Lists shorter than `big` use one warp,
// longer ones are chunked over CTAs (k_compact_plan / _count / _scan / _scatter).
__global__ void k_compact(const uint32_t* __restrict__ tv, const uint32_t* __restrict__ ntv,
                          const uint64_t* __restrict__ offV, uint32_t* adjL, uint32_t* tmp, uint32_t* ld,
                          const uint32_t* __restrict__ part, uint32_t big, Counters* c, uint32_t thr) {
  const uint32_t ln = lane_id();
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t n = *ntv;
  unsigned long long drop = 0;
  for (uint64_t i = gw; i < n; i += nw) {
    const uint32_t v = tv[i];
    const uint32_t L = ld[v];
    if (L >= big) continue;
    const uint64_t base = offV[v];
    for (uint32_t t = ln; t < L; t += 32) tmp[base + t] = adjL[base + t];
    __syncwarp();
    uint32_t lw = 0, dw = 0;
    for (uint32_t t0 = 0; t0 < L; t0 += 32) {
      const uint32_t t = t0 + ln;
      const bool ok = t < L;
      const uint32_t x = ok ? tmp[base + t] : 0u;
      const bool live = ok && part[x] > thr;
      const bool dead = ok && !live;
      const uint32_t ml = __ballot_sync(kFull, live), md = __ballot_sync(kFull, dead);
      if (live) adjL[base + lw + __popc(ml & lanemask_lt())] = x;
      if (dead) adjL[base + L - 1 - (dw + __popc(md & lanemask_lt()))] = x;
      lw += __popc(ml);
      dw += __popc(md);
    }
    PBNG_DCHECK(lw + dw == L);
    if (ln == 0) {
      ld[v] = lw;
      drop += (unsigned long long)L * L - (unsigned long long)lw * lw;
    }
    __syncwarp();
  }
  drop = warp_sum(drop);
  if (ln == 0 && drop) atomicAdd(&c->ld2_drop, drop);
}

// Lists of >= `big` entries are compacted by several CTAs: chunks of
// kCompChunk entries count their live entries (copying the chunk to tmp), a
// per-list scan places the chunks, and every chunk scatters its entries.
constexpr uint32_t kCompChunk = 4096;
constexpr uint32_t kCompThreads = 256;

// chunk tasks (touched index, chunk) for every touched list of >= big entries
__global__ void k_compact_plan(const uint32_t* __restrict__ tv, const uint32_t* __restrict__ ntv,
                               const uint32_t* __restrict__ ld, uint32_t big, uint2* __restrict__ tasks,
                               uint32_t* __restrict__ tbase, uint32_t* __restrict__ oldL, uint32_t* ntask) {
  const uint32_t n = *ntv;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t L = ld[tv[i]];
    oldL[i] = L;
    if (L < big) continue;
    const uint32_t nch = (L + kCompChunk - 1) / kCompChunk;
    const uint32_t b = atomicAdd(ntask, nch);
    tbase[i] = b;
    oldL[i] = L;
    for (uint32_t k = 0; k < nch; k++) tasks[b + k] = make_uint2(i, k);
  }
}

// per chunk: copy to tmp, count live entries -> cnt[task]
__global__ void __launch_bounds__(kCompThreads) k_compact_count(const uint2* __restrict__ tasks, const uint32_t* ntask,
                                                                const uint32_t* __restrict__ tv,
                                                                const uint32_t* __restrict__ oldL,
                                                                const uint64_t* __restrict__ offV,
                                                                const uint32_t* __restrict__ adjL, uint32_t* tmp,
                                                                const uint32_t* __restrict__ part, uint32_t* cnt,
                                                                uint32_t thr) {
  __shared__ uint32_t s_c;
  const uint32_t nt = *ntask;
  for (uint32_t t = blockIdx.x; t < nt; t += gridDim.x) {
    const uint2 tk = tasks[t];
    const uint64_t base = offV[tv[tk.x]];
    const uint32_t L = oldL[tk.x];
    const uint32_t a = tk.y * kCompChunk, b = min(L, a + kCompChunk);
    if (threadIdx.x == 0) s_c = 0;
    __syncthreads();
    uint32_t live = 0;
    for (uint32_t q = a + threadIdx.x; q < b; q += blockDim.x) {
      const uint32_t x = adjL[base + q];
      tmp[base + q] = x;
      live += part[x] > thr;
    }
    live = warp_sum(live);
    if (lane_id() == 0 && live) atomicAdd(&s_c, live);
    __syncthreads();
    if (threadIdx.x == 0) cnt[t] = s_c;
    __syncthreads();
  }
}

// per big list: exclusive scan of its chunk counts (in place), new live degree
__global__ void k_compact_scan(const uint32_t* __restrict__ tv, const uint32_t* __restrict__ ntv, uint32_t big,
                               const uint32_t* __restrict__ tbase, const uint32_t* __restrict__ oldL, uint32_t* cnt,
                               uint32_t* ld, Counters* c) {
  const uint32_t n = *ntv;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = tv[i];
    if (oldL[i] < big) continue;
    const uint32_t L = oldL[i], b = tbase[i], nch = (L + kCompChunk - 1) / kCompChunk;
    uint32_t run = 0;
    for (uint32_t k = 0; k < nch; k++) {
      const uint32_t x = cnt[b + k];
      cnt[b + k] = run;
      run += x;
    }
    ld[v] = run;
    atomicAdd(&c->ld2_drop, (unsigned long long)L * L - (unsigned long long)run * run);
  }
}

// per chunk: live entries to [base + live before), peeled ones after the new
// live prefix (this iteration's peeled group; order inside it is free)
__global__ void __launch_bounds__(kCompThreads) k_compact_scatter(const uint2* __restrict__ tasks,
                                                                  const uint32_t* ntask, const uint32_t* __restrict__ tv,
                                                                  const uint32_t* __restrict__ oldL,
                                                                  const uint32_t* __restrict__ tbase,
                                                                  const uint32_t* __restrict__ cnt,
                                                                  const uint64_t* __restrict__ offV,
                                                                  const uint32_t* __restrict__ ld, uint32_t* adjL,
                                                                  const uint32_t* __restrict__ tmp,
                                                                  const uint32_t* __restrict__ part, uint32_t thr) {
  constexpr uint32_t NW = kCompThreads / 32, SL = kCompChunk / NW;  // entries per warp slice
  __shared__ uint32_t s_w[NW];
  const uint32_t w = threadIdx.x >> 5, ln = lane_id();
  const uint32_t nt = *ntask;
  for (uint32_t t = blockIdx.x; t < nt; t += gridDim.x) {
    const uint2 tk = tasks[t];
    const uint32_t v = tv[tk.x];
    const uint64_t base = offV[v];
    const uint32_t L = oldL[tk.x], total = ld[v];
    const uint32_t a = tk.y * kCompChunk, b = min(L, a + kCompChunk);
    const uint32_t livepre = cnt[t];
    const uint32_t s0 = a + w * SL, s1 = min(b, s0 + SL);
    uint32_t lw = 0;
    for (uint32_t q = s0 + ln; q < s1; q += 32) lw += part[tmp[base + q]] > thr;
    lw = warp_sum(lw);
    if (ln == 0) s_w[w] = lw;
    __syncthreads();
    uint32_t lbefore = livepre;
    for (uint32_t k = 0; k < w; k++) lbefore += s_w[k];
    uint32_t dbefore = (s0 > b ? b : s0) - lbefore;  // peeled entries before this slice
    for (uint32_t q0 = s0; q0 < s1; q0 += 32) {
      const uint32_t q = q0 + ln;
      const bool ok = q < s1;
      const uint32_t x = ok ? tmp[base + q] : 0u;
      const bool live = ok && part[x] > thr;
      const bool dead = ok && !live;
      const uint32_t ml = __ballot_sync(kFull, live), md = __ballot_sync(kFull, dead);
      if (live) adjL[base + lbefore + __popc(ml & lanemask_lt())] = x;
      if (dead) adjL[base + total + dbefore + __popc(md & lanemask_lt())] = x;
      lbefore += __popc(ml);
      dbefore += __popc(md);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- validation
// PBNG_OPT_VALIDATE: offsets[0]=0, monotone, offsets[n]=m, indices < n_other.
__global__ void k_validate_csr(uint32_t n, uint64_t m, const uint64_t* __restrict__ off,
                               const uint32_t* __restrict__ idx, uint32_t n_other, uint32_t* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)n + 1 || i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i <= n) {
      const uint64_t o = off[i];
      if ((i == 0 && o != 0) || (i == n && o != m) || (i < n && off[i + 1] < o) || o > m) atomicOr(bad, 1u);
    }
    if (i < m && idx[i] >= n_other) atomicOr(bad, 2u);
  }
}

}  // namespace pbng
