// device_common.cuh — warp/CTA primitives shared by the PBNG kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pbng {

// Checked builds (-DPBNG_CHECK=1, tests/test_gpu_checked.py): PBNG_DCHECK(c)
// records the source line of the first failed condition in g_check_line
// (no trap: the kernel runs on, the host turns the record into an error after
// the call).  Stands in for compute-sanitizer memcheck, which this pool does
// not allow: the checks guard the shared-memory table / bitmap indices, the
// partner and support indices of every emitted update, and the list bounds of
// compaction and FD.  Compiled out (constant false) in the product build.
#ifndef PBNG_CHECK
#define PBNG_CHECK 0
#endif
__device__ unsigned int g_check_line;
#define PBNG_DCHECK(c)                                                       \
  do {                                                                       \
    if (PBNG_CHECK && !(c)) atomicCAS(&::pbng::g_check_line, 0u, (unsigned)__LINE__); \
  } while (0)

constexpr uint32_t kUnassigned = 0xFFFFFFFFu;  // part[u] of a vertex not yet peeled
constexpr uint32_t kEmpty = 0xFFFFFFFFu;       // empty hash key
constexpr unsigned kFull = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint64_t choose2(uint64_t w) { return w * (w - 1) / 2; }

__device__ __forceinline__ uint32_t ceil_log2(uint32_t x) { return x <= 1 ? 0 : 32 - __clz(x - 1); }

// fire-and-forget 64-bit add (wraps: adding 2^64 - d subtracts d)
__device__ __forceinline__ void red_add_u64(uint64_t* p, uint64_t v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t y = __shfl_xor_sync(kFull, v, o);
    v = y < v ? y : v;
  }
  return v;
}

// Warp-aggregated append: every lane with `pred` writes `val` to list[slot]
// with one atomic per warp.  All 32 lanes must be converged.
__device__ __forceinline__ void warp_append(bool pred, uint32_t val, uint32_t* list, uint32_t* counter) {
  uint32_t m = __ballot_sync(kFull, pred);
  if (!m) return;
  uint32_t leader = __ffs(m) - 1, base = 0;
  if (lane_id() == leader) base = atomicAdd(counter, (uint32_t)__popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (pred) list[base + __popc(m & lanemask_lt())] = val;
}
__device__ __forceinline__ void warp_append2(bool pred, uint2 val, uint2* list, uint32_t* counter) {
  uint32_t m = __ballot_sync(kFull, pred);
  if (!m) return;
  uint32_t leader = __ffs(m) - 1, base = 0;
  if (lane_id() == leader) base = atomicAdd(counter, (uint32_t)__popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (pred) list[base + __popc(m & lanemask_lt())] = val;
}

// Open-addressing (linear probing) table in shared memory: key u' -> w count.
// Keys never change once set until the table is swept, so a non-empty plain
// read is final; an empty read is resolved by CAS.
__device__ __forceinline__ void hash_insert(uint32_t* keys, uint32_t* vals, uint32_t logT, uint32_t k) {
  const uint32_t mask = (1u << logT) - 1;
  uint32_t h = (k * 0x9E3779B1u) >> (32 - logT);
  for (uint32_t probes = 0;; probes++) {
    PBNG_DCHECK(probes <= mask);  // the table is never full
    uint32_t cur = ((volatile uint32_t*)keys)[h];
    if (cur == k) break;
    if (cur == kEmpty) {
      cur = atomicCAS(&keys[h], kEmpty, k);
      if (cur == kEmpty || cur == k) break;
    }
    h = (h + 1) & mask;
  }
  atomicAdd(&vals[h], 1u);
}

// Add c occurrences of k (open addressing as hash_insert).
__device__ __forceinline__ void hash_add(uint32_t* keys, uint32_t* vals, uint32_t logT, uint32_t k, uint32_t c) {
  const uint32_t mask = (1u << logT) - 1;
  uint32_t h = (k * 0x9E3779B1u) >> (32 - logT);
  for (;;) {
    uint32_t cur = ((volatile uint32_t*)keys)[h];
    if (cur == k) break;
    if (cur == kEmpty) {
      cur = atomicCAS(&keys[h], kEmpty, k);
      if (cur == kEmpty || cur == k) break;
    }
    h = (h + 1) & mask;
  }
  atomicAdd(&vals[h], c);
}

// hash_insert that also reports the slot when k was new (else 0xFFFFFFFF).
__device__ __forceinline__ uint32_t hash_insert_new(uint32_t* keys, uint32_t* vals, uint32_t logT, uint32_t k) {
  const uint32_t mask = (1u << logT) - 1;
  uint32_t h = (k * 0x9E3779B1u) >> (32 - logT);
  uint32_t fresh = 0xFFFFFFFFu;
  for (;;) {
    uint32_t cur = ((volatile uint32_t*)keys)[h];
    if (cur == k) break;
    if (cur == kEmpty) {
      cur = atomicCAS(&keys[h], kEmpty, k);
      if (cur == kEmpty) {
        fresh = h;
        break;
      }
      if (cur == k) break;
    }
    h = (h + 1) & mask;
  }
  atomicAdd(&vals[h], 1u);
  return fresh;
}

// Count stored for k by hash_insert (0 if absent).
__device__ __forceinline__ uint32_t hash_lookup(const uint32_t* keys, const uint32_t* vals, uint32_t logT, uint32_t k) {
  const uint32_t mask = (1u << logT) - 1;
  uint32_t h = (k * 0x9E3779B1u) >> (32 - logT);
  for (;;) {
    const uint32_t cur = keys[h];
    if (cur == k) return vals[h];
    if (cur == kEmpty) return 0;
    h = (h + 1) & mask;
  }
}

// ---- partner-list sources ---------------------------------------------------
// For edge index e of u (offU[u] <= e < offU[u+1]) give the absolute start of
// the partner list in adjV and its length.
struct CdLists {  // CD: live prefix of N_v (dynamic deletion keeps it compact)
  const uint32_t* __restrict__ adjU;
  const uint64_t* __restrict__ offV;
  const uint32_t* __restrict__ ld;
  __device__ __forceinline__ void get(uint64_t e, uint64_t& base, uint32_t& len) const {
    uint32_t v = adjU[e];
    base = offV[v];
    len = ld[v];
  }
  __device__ __forceinline__ uint32_t mid(uint64_t e) const { return adjU[e]; }
};
struct PrefixLists {  // k-tip level retrieval: the part of N_v ranked before the start
  const uint32_t* __restrict__ adjU;
  const uint64_t* __restrict__ offV;
  const uint32_t* __restrict__ cut;  // per U-edge (u, v): members of N_v with id < u
  __device__ __forceinline__ void get(uint64_t e, uint64_t& base, uint32_t& len) const {
    uint32_t v = adjU[e];
    base = offV[v];
    len = cut[e];
  }
  __device__ __forceinline__ uint32_t mid(uint64_t e) const { return adjU[e]; }
};
struct FdLists {  // FD: the segment N_v ∩ U_i of the partition's induced subgraph G_i
  const uint32_t* __restrict__ adjU;
  const uint64_t* __restrict__ offV;
  const uint64_t* __restrict__ seg;  // per U-edge: lo | hi << 32, relative to offV[v]
  __device__ __forceinline__ void get(uint64_t e, uint64_t& base, uint32_t& len) const {
    uint32_t v = adjU[e];
    uint64_t s = seg[e];
    base = offV[v] + (uint32_t)s;
    len = (uint32_t)(s >> 32) - (uint32_t)s;
  }
};

// ---- wedge enumeration ------------------------------------------------------
// One warp walks the partner lists of up to 32 consecutive edges [we0, we1) of
// one u.  f(ok, u', e) is called warp-convergently (ok = lane holds an entry;
// e = edge index of the list the entry came from).
//   len >= longlim          : deferred to the CTA (index appended to s_long)
//   32 <= len < longlim     : whole warp strides the list (coalesced)
//   len < 32                : flattened over the warp with a shuffle binary
//                             search of the inclusive length scan
template <class L, class F>
__device__ __forceinline__ void warp_chunk(const L& lists, uint64_t we0, uint64_t we1,
                                           const uint32_t* __restrict__ adjV, uint32_t longlim,
                                           uint32_t* s_long, uint32_t* s_nlong, uint64_t chunk0, F& f) {
  const uint32_t ln = lane_id();
  const uint64_t e = we0 + ln;
  uint64_t base = 0;
  uint32_t len = 0;
  if (e < we1) lists.get(e, base, len);
  if (len >= longlim) {
    uint32_t slot = atomicAdd(s_nlong, 1u);
    s_long[slot] = (uint32_t)(e - chunk0);
    len = 0;
  }
  uint32_t mid = __ballot_sync(kFull, len >= 32);
  while (mid) {
    const int j = __ffs(mid) - 1;
    mid &= mid - 1;
    const uint64_t b = __shfl_sync(kFull, base, j);
    const uint32_t l = __shfl_sync(kFull, len, j);
    const uint64_t ej = we0 + j;
    for (uint32_t t0 = 0; t0 < l; t0 += 32) {
      const uint32_t t = t0 + ln;
      const bool ok = t < l;
      const uint32_t x = ok ? adjV[b + t] : 0u;
      f(ok, x, ej);
    }
  }
  const uint32_t slen = len >= 32 ? 0u : len;
  uint32_t incl = slen;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (ln >= (uint32_t)o) incl += y;
  }
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  const uint32_t excl = incl - slen;
  for (uint32_t t0 = 0; t0 < total; t0 += 32) {
    const uint32_t t = t0 + ln;
    uint32_t j = 0;
#pragma unroll
    for (uint32_t s = 16; s > 0; s >>= 1) {
      uint32_t y = __shfl_sync(kFull, incl, j + s - 1);
      if (y <= t) j += s;
    }
    const uint32_t ex = __shfl_sync(kFull, excl, j);
    const uint64_t b = __shfl_sync(kFull, base, j);
    const bool ok = t < total;
    const uint32_t x = ok ? adjV[b + (t - ex)] : 0u;
    f(ok, x, we0 + j);
  }
}

template <class L, class F>
__device__ __forceinline__ void warp_wedges(const L& lists, uint64_t e0, uint64_t e1,
                                            const uint32_t* __restrict__ adjV, F& f) {
  for (uint64_t c = e0; c < e1; c += 32)
    warp_chunk(lists, c, c + 32 < e1 ? c + 32 : e1, adjV, 0xFFFFFFFFu, nullptr, nullptr, 0, f);
}

// Whole CTA walks all partner lists of one u.  Neighbours are taken in chunks
// of blockDim; each warp takes 32 of them (warp_chunk); lists of length
// >= blockDim are then walked by the whole CTA, one at a time.
// s_long must hold blockDim entries.  Contains __syncthreads: call uniformly.
template <class L, class F>
__device__ __forceinline__ void cta_wedges(const L& lists, uint64_t e0, uint64_t e1,
                                           const uint32_t* __restrict__ adjV, uint32_t* s_long,
                                           uint32_t* s_nlong, F& f) {
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t CH = blockDim.x;
  for (uint64_t c = e0; c < e1; c += CH) {
    const uint64_t ce = c + CH < e1 ? c + CH : e1;
    if (threadIdx.x == 0) *s_nlong = 0;
    __syncthreads();
    const uint64_t we0 = c + 32ull * w;
    if (we0 < ce) warp_chunk(lists, we0, we0 + 32 < ce ? we0 + 32 : ce, adjV, CH, s_long, s_nlong, c, f);
    __syncthreads();
    const uint32_t nl = *s_nlong;
    for (uint32_t i = 0; i < nl; i++) {
      uint64_t base;
      uint32_t len;
      const uint64_t ei = c + s_long[i];
      lists.get(ei, base, len);
      for (uint32_t t0 = 0; t0 < len; t0 += CH) {
        const uint32_t t = t0 + threadIdx.x;
        const bool ok = t < len;
        const uint32_t x = ok ? adjV[base + t] : 0u;
        f(ok, x, ei);
      }
    }
    __syncthreads();
  }
}

// Whole CTA walks all partner lists of one start with the entries flattened
// over the threads (one list per thread for the length scan, so at most
// blockDim lists; more fall back to cta_wedges).  Every thread takes entries
// t, t + blockDim, ... and finds its list by binary search over the scanned
// lengths, so a start with a few medium lists keeps every warp busy.
// f(ok, x, e) is called CTA-convergently.  Contains __syncthreads.
template <class L, class F>
__device__ __forceinline__ void cta_flat_wedges(const L& lists, uint64_t e0, uint64_t e1,
                                                const uint32_t* __restrict__ adjV, uint32_t* s_pre,
                                                unsigned long long* s_base, uint32_t* s_scan, uint32_t* s_long,
                                                uint32_t* s_nlong, F& f);

// Block-wide exclusive scan of one uint32 per thread (blockDim multiple of 32,
// <= 1024).  s_warp: 33 uint32 of shared memory.  Returns the exclusive prefix;
// *total receives the block sum.  Contains __syncthreads.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* s_warp, uint32_t* total) {
  const uint32_t ln = lane_id(), w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (ln >= (uint32_t)o) incl += y;
  }
  if (ln == 31) s_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t v = ln < nw ? s_warp[ln] : 0u;
    uint32_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(kFull, vi, o);
      if (ln >= (uint32_t)o) vi += y;
    }
    if (ln < nw) s_warp[ln] = vi - v;
    if (ln == 31) s_warp[32] = vi;  // nw <= 32: lane 31 holds the grand total
  }
  __syncthreads();
  uint32_t res = s_warp[w] + incl - x;
  *total = s_warp[32];
  __syncthreads();
  return res;
}

template <class L, class F>
__device__ __forceinline__ void cta_flat_wedges(const L& lists, uint64_t e0, uint64_t e1,
                                                const uint32_t* __restrict__ adjV, uint32_t* s_pre,
                                                unsigned long long* s_base, uint32_t* s_scan, uint32_t* s_long,
                                                uint32_t* s_nlong, F& f) {
  const uint64_t d = e1 - e0;
  if (d > blockDim.x) {
    cta_wedges(lists, e0, e1, adjV, s_long, s_nlong, f);
    return;
  }
  uint64_t base = 0;
  uint32_t len = 0;
  if (threadIdx.x < d) lists.get(e0 + threadIdx.x, base, len);
  uint32_t total;
  const uint32_t pre = block_excl_scan(len, s_scan, &total);
  if (threadIdx.x < d) {
    s_pre[threadIdx.x] = pre;
    s_base[threadIdx.x] = base;
  }
  __syncthreads();
  const uint32_t nd = (uint32_t)d;
  for (uint32_t t0 = 0; t0 < total; t0 += blockDim.x) {
    const uint32_t t = t0 + threadIdx.x;
    const bool ok = t < total;
    uint32_t lo = 0, hi = nd;  // largest j with s_pre[j] <= t
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_pre[mid] <= t) lo = mid; else hi = mid;
    }
    const uint32_t x = ok ? adjV[s_base[lo] + (t - s_pre[lo])] : 0u;
    f(ok, x, e0 + lo);
  }
  __syncthreads();
}

// Union-find over ids for butterfly connectivity (k-tip components, Def. 2
// P:451-459).  parent[x] <= x always holds: a root is hooked only under a
// smaller root, so the root of a set is its smallest id and any ancestor read
// by a racing find is still a valid (smaller) parent.
__device__ __forceinline__ uint32_t cc_find(uint32_t* parent, uint32_t x) {
  volatile uint32_t* p = parent;
  uint32_t y = p[x];
  while (y != x) {
    const uint32_t z = p[y];
    if (z != y) p[x] = z;  // path halving
    x = y;
    y = z;
  }
  return x;
}

__device__ __forceinline__ void cc_union(uint32_t* parent, uint32_t a, uint32_t b) {
  for (;;) {
    a = cc_find(parent, a);
    b = cc_find(parent, b);
    if (a == b) return;
    if (a < b) {
      const uint32_t t = a;
      a = b;
      b = t;
    }
    if (atomicCAS(&parent[a], a, b) == a) return;  // else a was hooked meanwhile: retry
  }
}

}  // namespace pbng
