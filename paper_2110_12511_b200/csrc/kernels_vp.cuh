// kernels_vp.cuh — vertex-priority per-vertex butterfly counting (Alg.1
// "pveBcnt"; Chiba-Nishizeki priority), restricted to
// the counts the tip decomposition needs (the peel side U).
//
// The graph is relabeled (kernels_relabel.cuh): ranks follow decreasing
// degree, ties put U before V, and every list is sorted by rank, so the wedges
// Alg.1 expands from a start (l.9-12: last ranked above both mid and start)
// are a PREFIX of each mid's list:
//   start u ∈ U, mid v ∈ N_u, last u' ∈ N_v with d_u' >= d_v and u' < u
//       -> the first cutV[v] entries of N_v, then only ids below u;
//   start v ∈ V, mid u ∈ N_v, last v' ∈ N_u with d_v' > d_u and v' < v
//       -> the first cutU[u] entries of N_u, then only ids below v.
// Per-vertex attribution (Alg.1 l.16-21):
//   start ∈ U: for every last with w >= 2, ⋈_start += C(w,2), ⋈_last += C(w,2);
//   start ∈ V: every mid u gets Σ over its wedges (u, v') of (w[v'] - 1).
// (The other attributions go to V vertices, whose counts are not needed.)
// Every butterfly is expanded from exactly one start (its top-ranked vertex is
// the last), for ANY total order, so counts are exact on the
// live subgraph as well: the §5.1 re-count reuses the priority
// of the original graph and skips peeled vertices.
#pragma once
#include "kernels_cd.cuh"

namespace pbng {

// start ∈ U: edge e of the start -> mid v, partner list = live N_v prefix
struct VpULists {
  const uint32_t* __restrict__ adjU;
  const uint64_t* __restrict__ offV;
  const uint32_t* __restrict__ cut;
  __device__ __forceinline__ void get(uint64_t e, uint64_t& base, uint32_t& len) const {
    const uint32_t v = adjU[e];
    base = offV[v];
    len = cut[v];
  }
  __device__ __forceinline__ uint32_t mid(uint64_t e) const { return adjU[e]; }
};
// start ∈ V: edge e of the start (live N_v) -> mid u, partner list = N_u prefix
struct VpVLists {
  const uint32_t* __restrict__ adjL;
  const uint64_t* __restrict__ offU;
  const uint32_t* __restrict__ cut;
  const uint32_t* __restrict__ part;
  __device__ __forceinline__ void get(uint64_t e, uint64_t& base, uint32_t& len) const {
    const uint32_t u = adjL[e];
    base = offU[u];
    len = part[u] == kUnassigned ? cut[u] : 0u;  // peeled mids are not in the live graph
  }
};

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* __restrict__ p, uint32_t n, uint32_t key) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// cutV[v] = live entries of N_v with rank < #{u : d_u >= d_v}  (u' ranked above mid v)
__global__ void k_vp_cut_v(uint32_t nV, const uint64_t* __restrict__ offV, const uint32_t* __restrict__ adjL,
                           const uint32_t* __restrict__ ld, const unsigned long long* __restrict__ binoffU,
                           uint32_t dmaxU, uint32_t* __restrict__ cutV) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nV; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = offV[v];
    const uint64_t d = offV[v + 1] - b;
    const uint32_t lim = d > dmaxU ? 0u : (uint32_t)binoffU[dmaxU - d + 1];
    cutV[v] = lower_bound_u32(adjL + b, ld[v], lim);
  }
}

// cutU[u] = entries of N_u with rank < #{v : d_v > d_u}  (v' ranked above mid u)
__global__ void k_vp_cut_u(uint32_t nU, const uint64_t* __restrict__ offU, const uint32_t* __restrict__ adjU,
                           const unsigned long long* __restrict__ binoffV, uint32_t dmaxV, uint32_t* __restrict__ cutU) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nU; u += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = offU[u];
    const uint64_t d = offU[u + 1] - b;
    const uint32_t lim = d >= dmaxV ? 0u : (uint32_t)binoffV[dmaxV - d];
    cutU[u] = lower_bound_u32(adjU + b, (uint32_t)d, lim);
  }
}

// Edge range of a start and its partner-list source.
template <int SIDE>
struct VpSide;
template <>
struct VpSide<0> {  // start ∈ U
  static __device__ __forceinline__ VpULists lists(const AggArgs& a) { return VpULists{a.adjU, a.offV, a.cutV}; }
  static __device__ __forceinline__ const uint32_t* partners(const AggArgs& a) { return a.adjV; }
  static __device__ __forceinline__ void range(const AggArgs& a, uint32_t x, uint64_t& e0, uint64_t& e1) {
    e0 = a.offU[x];
    e1 = a.offU[x + 1];
  }
};
template <>
struct VpSide<1> {  // start ∈ V
  static __device__ __forceinline__ VpVLists lists(const AggArgs& a) {
    return VpVLists{a.adjV, a.offU, a.cutU, a.part};
  }
  static __device__ __forceinline__ const uint32_t* partners(const AggArgs& a) { return a.adjU; }
  static __device__ __forceinline__ void range(const AggArgs& a, uint32_t x, uint64_t& e0, uint64_t& e1) {
    e0 = a.offV[x];
    e1 = e0 + a.ld[x];
  }
};

// Classify starts (SIDE 0: every live u < n; SIDE 1: every v < n) by the
// wedges their expansion reads, wl = Σ prefix lengths, into tier 0 (warp) /
// tier 1 (CTA).  A warp takes 32 starts and walks their edges flattened.
template <int SIDE>
__global__ void __launch_bounds__(256) k_vp_classify(uint32_t n, AggArgs a, uint2* tier0, uint2* tier1,
                                                     uint2* tier2, uint2* bigq, uint32_t hmax, uint32_t dlim) {
  __shared__ unsigned long long s_acc[8][32];
  const uint32_t ln = lane_id();
  unsigned long long* acc = s_acc[threadIdx.x >> 5];
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const auto L = VpSide<SIDE>::lists(a);
  unsigned long long wsum = 0, ssum = 0;
  for (uint64_t b = gw * 32; b < n; b += nw * 32) {
    const uint64_t idx = b + ln;
    bool ok = idx < n;
    const uint32_t x = (uint32_t)idx;
    if (SIDE == 0 && ok && a.part[x] != kUnassigned) ok = false;
    uint64_t e0 = 0, e1 = 0;
    if (ok) VpSide<SIDE>::range(a, x, e0, e1);
    // hub starts are summed by a whole CTA (k_vp_classify_big)
    const bool big = e1 - e0 > kClassBig;
    warp_append2(big, make_uint2(x, 0), bigq, &a.c->nbig);
    if (big) {
      ok = false;
      e1 = e0;
    }
    const uint64_t d = e1 - e0;
    uint64_t incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, incl, o);
      if (ln >= (uint32_t)o) incl += y;
    }
    const uint64_t total = __shfl_sync(kFull, incl, 31);
    const uint64_t excl = incl - d;
    acc[ln] = 0;
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
        uint64_t base;
        uint32_t len;
        L.get(je + (t - jx), base, len);
        val = len;
      }
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
    const unsigned long long mine = acc[ln];
    int tier = -1;
    uint32_t pb = 0;
    if (ok && mine) {
      pb = mine > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)mine;
      tier = pb <= kWarpCap ? 0 : (pb <= hmax && d < dlim) ? 1 : 2;
      wsum += mine;
      ssum += d;
    }
    const uint2 item = make_uint2(x, pb);
    warp_append2(tier == 0, item, tier0, &a.c->ntier[0]);
    warp_append2(tier == 1, item, tier1, &a.c->ntier[1]);
    warp_append2(tier == 2, item, tier2, &a.c->ntier[2]);
    __syncwarp();
  }
  wsum = warp_sum(wsum);
  ssum = warp_sum(ssum);
  if (ln == 0 && wsum) {
    atomicAdd(&a.c->wedges, wsum);
    atomicAdd(&a.c->cum_wedges, wsum);
    atomicAdd(&a.c->cum_steps, ssum);
  }
}

// The starts k_vp_classify deferred (more than kClassBig lists): one CTA each.
template <int SIDE>
__global__ void __launch_bounds__(512) k_vp_classify_big(AggArgs a, const uint2* __restrict__ bigq, uint2* tier0,
                                                         uint2* tier1, uint2* tier2, uint32_t hmax, uint32_t dlim) {
  __shared__ unsigned long long s_part[16];
  const uint32_t n = a.c->nbig;
  const auto L = VpSide<SIDE>::lists(a);
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint32_t x = bigq[i].x;
    uint64_t e0, e1;
    VpSide<SIDE>::range(a, x, e0, e1);
    unsigned long long s = 0;
    for (uint64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      uint64_t base;
      uint32_t len;
      L.get(e, base, len);
      s += len;
    }
    s = warp_sum(s);
    if (lane_id() == 0) s_part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      s = 0;
      for (uint32_t w = 0; w < (blockDim.x >> 5); w++) s += s_part[w];
      if (s) {
        const uint32_t pb = s > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)s;
        const int tier = pb <= kWarpCap ? 0 : (pb <= hmax && e1 - e0 < dlim) ? 1 : 2;
        uint2* tl = tier == 0 ? tier0 : tier == 1 ? tier1 : tier2;
        tl[atomicAdd(&a.c->ntier[tier], 1u)] = make_uint2(x, pb);
        atomicAdd(&a.c->wedges, s);
        atomicAdd(&a.c->cum_wedges, s);
        atomicAdd(&a.c->cum_steps, (unsigned long long)(e1 - e0));
      }
    }
    __syncthreads();
  }
}

// Tier 0: one warp per start, per-warp open-addressing table of w[last].
template <int SIDE>
__global__ void __launch_bounds__(kWarpTierThreads) k_vp_agg_warp(AggArgs a) {
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
  const auto L = VpSide<SIDE>::lists(a);
  const uint32_t* __restrict__ partner = VpSide<SIDE>::partners(a);
  const uint32_t wpb = blockDim.x >> 5;
  for (uint32_t i = blockIdx.x * wpb + w; i < n; i += gridDim.x * wpb) {
    const uint2 it = a.list[i];
    const uint32_t x = it.x;
    uint32_t logT = ceil_log2(2 * it.y);
    logT = logT < 5 ? 5 : logT;
    uint64_t e0, e1;
    VpSide<SIDE>::range(a, x, e0, e1);
    auto f = [&](bool ok, uint32_t y, uint64_t) {
      if (ok && y < x) hash_insert(keys, vals, logT, y);
    };
    warp_wedges(L, e0, e1, partner, f);
    __syncwarp();
    if (SIDE == 1) {
      // pass 2 (Alg.1 l.20-21): mid u gets Σ (w[last] - 1) over its wedges
      auto f2 = [&](bool ok, uint32_t y, uint64_t e) {
        unsigned long long val = 0;
        if (ok && y < x) val = hash_lookup(keys, vals, logT, y) - 1u;
        const uint64_t key = ok ? e : ~0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long yv = __shfl_up_sync(kFull, val, o);
          const uint64_t ky = __shfl_up_sync(kFull, key, o);
          if (ln >= (uint32_t)o && ky == key) val += yv;
        }
        const uint64_t kn = __shfl_down_sync(kFull, key, 1);
        if (ok && (ln == 31 || kn != key) && val) red_add_u64(&a.support[a.adjV[e]], val);
      };
      warp_wedges(L, e0, e1, partner, f2);
      __syncwarp();
    }
    uint64_t acc = 0;
    const uint32_t T = 1u << logT;
    for (uint32_t s = ln; s < T; s += 32) {
      const uint32_t k = keys[s];
      if (k != kEmpty) {
        const uint32_t wv = vals[s];
        keys[s] = kEmpty;
        vals[s] = 0;
        if (SIDE == 0 && wv >= 2 && a.part[k] == kUnassigned) {
          const uint64_t d = choose2(wv);
          red_add_u64(&a.support[k], d);
          acc += d;
        }
      }
    }
    if (SIDE == 0) {
      acc = warp_sum(acc);
      if (ln == 0 && acc) red_add_u64(&a.support[x], acc);
    }
    __syncwarp();
  }
}

// pass-2 hook of range_agg_one for V starts: mid (adjL[e]) += Σ (w - 1)
struct VpPass2 {
  static constexpr bool kOn = true;
  const uint32_t* adjL;
  uint64_t* support;
  __device__ __forceinline__ void operator()(uint64_t e, unsigned long long cs) const {
    red_add_u64(&support[adjL[e]], cs);
  }
};

// Middle tier: one CTA per start, shared-memory hash table (agg_mid.cuh).
template <int SIDE>
__global__ void __launch_bounds__(kMidThreads, kMidCtas) k_vp_agg_mid(AggArgs a) {
  extern __shared__ __align__(16) unsigned char msm[];
  MidSmem& S = *reinterpret_cast<MidSmem*>(msm);
  __shared__ uint32_t s_nlong, s_t;
  __shared__ unsigned long long s_acc;
  for (uint32_t i = threadIdx.x; i < kCtaSlots; i += blockDim.x) {
    S.keys[i] = kEmpty;
    S.vals[i] = 0;
  }
  const uint32_t n = *a.count;
  const auto L = VpSide<SIDE>::lists(a);
  const uint32_t* __restrict__ partner = VpSide<SIDE>::partners(a);
  for (;;) {
    if (threadIdx.x == 0) {
      s_t = atomicAdd(a.ticket, 1u);
      s_acc = 0;
    }
    __syncthreads();
    const uint32_t i = s_t;
    if (i >= n) break;
    const uint2 it = a.list[i];
    const uint32_t x = it.x;
    uint64_t e0, e1;
    VpSide<SIDE>::range(a, x, e0, e1);
    auto keep = [x](uint32_t y) { return y < x; };
    if (SIDE == 0) {
      uint64_t acc = 0;
      auto out = [&](uint32_t k, uint32_t w) {
        if (w >= 2 && a.part[k] == kUnassigned) {
          const uint64_t d = choose2(w);
          red_add_u64(&a.support[k], d);
          acc += d;
        }
      };
      mid_agg_one(L, e0, e1, partner, it.y, S, &s_nlong, keep, out);
      acc = warp_sum(acc);
      if (lane_id() == 0 && acc) atomicAdd(&s_acc, (unsigned long long)acc);
      __syncthreads();
      if (threadIdx.x == 0 && s_acc) red_add_u64(&a.support[x], s_acc);
    } else {
      auto out = [](uint32_t, uint32_t) {};
      mid_agg_one(L, e0, e1, partner, it.y, S, &s_nlong, keep, out, VpPass2{a.adjV, a.support});
    }
    __syncthreads();
  }
}

// Tier 1 for starts in U: packed hash tables over degree-mass windows
// (agg_hash.cuh); C(w,2) to every last below the start and to the start.
__global__ void __launch_bounds__(kHashThreads, kHashCtas) k_vp_agg_hash(AggArgs a) {
  extern __shared__ __align__(16) unsigned char hsm_[];
  HashSmem& S = *reinterpret_cast<HashSmem*>(hsm_);
  hash_tier<3>(a, VpSide<0>::lists(a), S);
}

// Tier 2: one CTA per start, window bitmap over segments (agg_win.cuh).
template <int SIDE>
__global__ void __launch_bounds__(kWinThreads, kWinCtas) k_vp_agg_win(AggArgs a) {
  extern __shared__ __align__(16) unsigned char wsm[];
  WinSmem& S = *reinterpret_cast<WinSmem*>(wsm);
  __shared__ WinShared sh;
  for (uint32_t i = threadIdx.x; i < kWinBitWords; i += blockDim.x) S.bits[i] = 0;
  for (uint32_t i = threadIdx.x; i < kWinDupSlots; i += blockDim.x) S.dup[i] = kEmptySlot;
  uint32_t* bnd = a.win_bnd + (uint64_t)blockIdx.x * a.win_cap;
  const uint32_t G = a.win_split;
  const uint64_t n = (uint64_t)*a.count * G;
  const auto L = VpSide<SIDE>::lists(a);
  const uint32_t* __restrict__ partner = VpSide<SIDE>::partners(a);
  for (;;) {
    if (threadIdx.x == 0) {
      sh.t = atomicAdd(a.ticket, 1u);
      sh.acc = 0;
    }
    __syncthreads();
    const uint32_t t = sh.t;
    if (t >= n) break;
    const uint32_t x = a.list[t / G].x;
    uint64_t e0, e1;
    VpSide<SIDE>::range(a, x, e0, e1);
    if (SIDE == 0) {
      uint64_t acc = 0;
      auto out = [&](uint32_t k, uint32_t wv) {
        if (a.part[k] == kUnassigned) {
          const uint64_t d = choose2(wv);
          red_add_u64(&a.support[k], d);
          acc += d;
        }
      };
      win_agg_one(L, e0, e1, 0xFFFFFFFFu, x, t % G, G, partner, S, sh, bnd, a.win_pre, out, a.c, false);
      acc = warp_sum(acc);
      if (lane_id() == 0 && acc) atomicAdd(&sh.acc, (unsigned long long)acc);
      __syncthreads();
      if (threadIdx.x == 0 && sh.acc) red_add_u64(&a.support[x], sh.acc);
    } else {
      auto out = [&](uint32_t, uint32_t) {};
      win_agg_one(L, e0, e1, 0xFFFFFFFFu, x, t % G, G, partner, S, sh, bnd, a.win_pre, out, a.c, false,
                  VpPass2{a.adjV, a.support});
    }
    __syncthreads();
  }
}

}  // namespace pbng
