// agg_mid.cuh — middle aggregation tier: one CTA per vertex whose partner
// bound exceeds a warp table (kWarpCap) but fits one shared-memory hash table
// (kCtaCap).  The wedges u -> v -> u' are walked by cta_wedges (warp-chunked
// lists, CTA-strided long lists) and w(u, u') counted in an open-addressing
// table; the sweep emits every partner once.  No window passes: the cost is
// one table insert per wedge plus one sweep of the table.
#pragma once
// (included inside namespace pbng by kernels_cd.cuh)

constexpr uint64_t kEmptySlot = 0xFFFFFFFF00000000ull;  // empty (key << 32 | count) slot
constexpr uint32_t kDupProbe = 32;                     // probe limit of the tier-2 repeat table

// No second pass (CD peel / one-sided count); vertex-priority counting with
// starts in V supplies VpPass2 (kernels_vp.cuh).
struct NoPass2 {
  static constexpr bool kOn = false;
  __device__ void operator()(uint64_t, unsigned long long) const {}
};

#ifndef PBNG_MID_THREADS
#define PBNG_MID_THREADS 512
#endif
#ifndef PBNG_MID_CTAS
#define PBNG_MID_CTAS 2
#endif
constexpr uint32_t kMidThreads = PBNG_MID_THREADS;
constexpr uint32_t kMidCtas = PBNG_MID_CTAS;  // resident CTAs per SM

struct MidSmem {
  uint32_t keys[kCtaSlots];
  uint32_t vals[kCtaSlots];
  uint16_t used[kCtaCap];               // slots taken, in insertion order (sweep list)
  uint32_t s_long[kMidThreads];
  uint32_t s_pre[kMidThreads];
  unsigned long long s_base[kMidThreads];
  uint32_t s_scan[33];
  uint32_t nused;
};

// Aggregate w over the wedges of one start (lists e in [e0, e1)), keeping
// partners x with keep(x); then, if pass2 is on, walk the wedges again and
// call pass2(e, Σ (w - 1)) per list; finally emit(k, w) for every partner.
// The walk flattens the start's entries over the whole CTA; the sweep visits
// only the slots taken.  Call with the whole CTA; the table is empty on entry
// and on exit.
template <class L, class Keep, class Emit, class Pass2 = NoPass2>
__device__ __forceinline__ void mid_agg_one(const L& lists, uint64_t e0, uint64_t e1,
                                            const uint32_t* __restrict__ partner, uint32_t pb, MidSmem& S,
                                            uint32_t* s_nlong, const Keep& keep, Emit& emit,
                                            const Pass2& pass2 = Pass2()) {
  const uint32_t ln = lane_id();
  uint32_t logT = ceil_log2(2 * pb);
  logT = logT < 5 ? 5 : (logT > kLogCtaSlots ? kLogCtaSlots : logT);
  if (threadIdx.x == 0) S.nused = 0;
  __syncthreads();
  auto f = [&](bool ok, uint32_t x, uint64_t) {
    const uint32_t sl = ok && keep(x) ? hash_insert_new(S.keys, S.vals, logT, x) : 0xFFFFFFFFu;
    const bool fresh = sl != 0xFFFFFFFFu;
    const uint32_t m = __ballot_sync(kFull, fresh);
    if (m) {
      const uint32_t leader = __ffs(m) - 1;
      uint32_t base = 0;
      if (ln == leader) base = atomicAdd(&S.nused, (uint32_t)__popc(m));
      base = __shfl_sync(kFull, base, leader);
      if (fresh) S.used[base + __popc(m & lanemask_lt())] = (uint16_t)sl;
    }
  };
  cta_flat_wedges(lists, e0, e1, partner, S.s_pre, S.s_base, S.s_scan, S.s_long, s_nlong, f);
  if (Pass2::kOn) {
    auto f2 = [&](bool ok, uint32_t x, uint64_t e) {
      unsigned long long val = 0;
      if (ok && keep(x)) val = hash_lookup(S.keys, S.vals, logT, x) - 1u;
      const uint64_t key = ok ? e : ~0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long yv = __shfl_up_sync(kFull, val, o);
        const uint64_t ky = __shfl_up_sync(kFull, key, o);
        if (ln >= (uint32_t)o && ky == key) val += yv;
      }
      const uint64_t kn = __shfl_down_sync(kFull, key, 1);
      if (ok && (ln == 31 || kn != key) && val) pass2(e, val);
    };
    cta_flat_wedges(lists, e0, e1, partner, S.s_pre, S.s_base, S.s_scan, S.s_long, s_nlong, f2);
  }
  const uint32_t nu = S.nused;
  for (uint32_t i = threadIdx.x; i < nu; i += blockDim.x) {
    const uint32_t s = S.used[i];
    const uint32_t k = S.keys[s];
    const uint32_t w = S.vals[s];
    S.keys[s] = kEmpty;
    S.vals[s] = 0;
    emit(k, w);
  }
  __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(kMidThreads, kMidCtas) k_agg_mid(AggArgs a) {
  extern __shared__ __align__(16) unsigned char msm[];
  MidSmem& S = *reinterpret_cast<MidSmem*>(msm);
  __shared__ uint32_t s_nlong, s_t;
  __shared__ unsigned long long s_acc;
  for (uint32_t i = threadIdx.x; i < kCtaSlots; i += blockDim.x) {
    S.keys[i] = kEmpty;
    S.vals[i] = 0;
  }
  const uint32_t n = *a.count;
  const auto L = agg_lists<MODE>(a);
  unsigned long long upd = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      s_t = atomicAdd(a.ticket, 1u);
      s_acc = 0;
    }
    __syncthreads();
    const uint32_t i = s_t;
    if (i >= n) break;
    const uint2 it = a.list[i];
    const uint32_t u = it.x;
    uint64_t acc = 0;
    auto keep = [u](uint32_t x) { return x != u; };
    auto out = [&](uint32_t k, uint32_t w) { emit<MODE>(a, u, k, w, acc, upd); };
    mid_agg_one(L, a.offU[u], a.offU[u + 1], a.adjV, it.y, S, &s_nlong, keep, out);
    if (MODE == 0) {
      acc = warp_sum(acc);
      if (lane_id() == 0 && acc) atomicAdd(&s_acc, (unsigned long long)acc);
      __syncthreads();
      if (threadIdx.x == 0) a.support[u] = s_acc;
    }
    __syncthreads();
  }
  if (MODE == 1) flush_updates(a, upd);
}
