// kernels_relabel.cuh — priority relabeling of both vertex sides (Alg.1 l.2-5,
// P:399-406): vertices are renumbered per side in decreasing order of degree
// and every adjacency list is rewritten in the new labels and sorted, so that
//   * vertex-priority counting (Alg.1 l.10) can stop each list walk
//     at a prefix, and
//   * every other kernel keeps its precondition of id-sorted lists.
// The whole decomposition then runs on the relabeled graph (tip numbers are
// invariant under relabeling, Lemma 1) and θ is gathered back.
//
// Order among equal degrees is whatever the scatter atomics produce: any total
// order gives exact counts, so results are deterministic
// while the wedge counters may differ by a little between runs.
#pragma once
#include "device_common.cuh"

namespace pbng {

constexpr uint32_t kSortSmall = 32;    // lists <= this: per-thread register network
constexpr uint32_t kSortTile = 4096;   // lists <= this: one CTA bitonic sort in smem
constexpr uint32_t kSortThreads = 512;

// ---------------------------------------------------------------- scan
// Exclusive scan of a uint64 array in place: tiles of kScanTile, tile sums,
// one-CTA scan of the tile sums, add-back.
constexpr uint32_t kScanThreads = 1024;
constexpr uint32_t kScanItems = 4;
constexpr uint32_t kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint64_t block_excl_scan64(uint64_t x, uint64_t* s_warp, uint64_t* total) {
  const uint32_t ln = lane_id(), w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(kFull, incl, o);
    if (ln >= (uint32_t)o) incl += y;
  }
  if (ln == 31) s_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    const uint64_t v = ln < nw ? s_warp[ln] : 0ull;
    uint64_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, vi, o);
      if (ln >= (uint32_t)o) vi += y;
    }
    if (ln < nw) s_warp[ln] = vi - v;
    if (ln == 31) s_warp[32] = vi;
  }
  __syncthreads();
  const uint64_t r = s_warp[w] + incl - x;
  *total = s_warp[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(uint64_t n, uint64_t* a, uint64_t* tsum) {
  __shared__ uint64_t s_warp[33];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint64_t x[kScanItems], s = 0;
#pragma unroll
  for (uint32_t k = 0; k < kScanItems; k++) {
    x[k] = base + k < n ? a[base + k] : 0ull;
    s += x[k];
  }
  uint64_t tot;
  uint64_t run = block_excl_scan64(s, s_warp, &tot);
#pragma unroll
  for (uint32_t k = 0; k < kScanItems; k++) {
    if (base + k < n) a[base + k] = run;
    run += x[k];
  }
  if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_top(uint32_t ntiles, uint64_t* tsum) {
  __shared__ uint64_t s_warp[33];
  uint64_t carry = 0;
  for (uint32_t c = 0; c < ntiles; c += kScanThreads) {
    const uint32_t i = c + threadIdx.x;
    const uint64_t x = i < ntiles ? tsum[i] : 0ull;
    uint64_t tot;
    const uint64_t r = block_excl_scan64(x, s_warp, &tot);
    if (i < ntiles) tsum[i] = carry + r;
    carry += tot;
  }
}

__global__ void k_scan_add(uint64_t n, uint64_t* a, const uint64_t* __restrict__ tsum) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] += tsum[i / kScanTile];
}

// ---------------------------------------------------------------- degree order
__global__ void k_deg_max(uint32_t n, const uint64_t* __restrict__ off, unsigned long long* dmax) {
  unsigned long long mx = 0;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = off[x + 1] - off[x];
    mx = d > mx ? d : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(kFull, mx, o);
    mx = y > mx ? y : mx;
  }
  if (lane_id() == 0 && mx) atomicMax(dmax, mx);
}

// bins keyed by r = dmax - d (descending degree): cnt[r] (vertices), edg[r] (edges)
__global__ void k_deg_hist(uint32_t n, const uint64_t* __restrict__ off, uint32_t dmax,
                           unsigned long long* cnt, unsigned long long* edg) {
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x; b < n; b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = b + threadIdx.x;
    const bool ok = x < n;
    const uint32_t d = ok ? (uint32_t)(off[x + 1] - off[x]) : 0u;
    const uint32_t key = ok ? dmax - d : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(kFull, key);
    if (ok && lane_id() == (uint32_t)(__ffs(peers) - 1)) {
      const uint32_t c = __popc(peers);
      atomicAdd(&cnt[key], (unsigned long long)c);
      atomicAdd(&edg[key], (unsigned long long)c * d);
    }
  }
}

// rank[x] = position of x in decreasing-degree order; inv[rank] = x.
// binoff = exclusive scan of cnt (first rank of each degree).
__global__ void k_rank_scatter(uint32_t n, const uint64_t* __restrict__ off, uint32_t dmax,
                               const unsigned long long* __restrict__ binoff, unsigned int* cursor,
                               uint32_t* __restrict__ rank, uint32_t* __restrict__ inv) {
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x; b < n; b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = b + threadIdx.x;
    const bool ok = x < n;
    const uint32_t d = ok ? (uint32_t)(off[x + 1] - off[x]) : 0u;
    const uint32_t key = ok ? dmax - d : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(kFull, key);
    const uint32_t leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (ok && lane_id() == leader) base = atomicAdd(&cursor[key], (uint32_t)__popc(peers));
    base = __shfl_sync(kFull, base, leader);
    if (ok) {
      const uint32_t r = (uint32_t)binoff[key] + base + __popc(peers & lanemask_lt());
      rank[x] = r;
      inv[r] = (uint32_t)x;
    }
  }
}

// offsets of the relabeled CSR: rank i of degree d starts at
// edgoff[key] + (i - binoff[key]) * d  (all lists of one degree are contiguous)
__global__ void k_rank_offsets(uint32_t n, uint64_t m, const uint32_t* __restrict__ inv,
                               const uint64_t* __restrict__ off, uint32_t dmax,
                               const unsigned long long* __restrict__ binoff,
                               const unsigned long long* __restrict__ edgoff, uint64_t* __restrict__ offN) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (i == n) {
      offN[n] = m;
      continue;
    }
    const uint32_t x = inv[i];
    const uint64_t d = off[x + 1] - off[x];
    const uint32_t key = dmax - (uint32_t)d;
    offN[i] = edgoff[key] + (i - binoff[key]) * d;
  }
}

// adjN[offN[i] + k] = rank_other[adj[off[inv[i]] + k]]  (unsorted).  A warp
// takes 32 consecutive ranks and walks their edges as one flattened range;
// ranks < nbig (the longest lists) are left to k_relabel_fill_big.
__global__ void k_relabel_fill(uint32_t n, uint32_t nbig, const uint32_t* __restrict__ inv,
                               const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                               const uint64_t* __restrict__ offN, const uint32_t* __restrict__ rank_other,
                               uint32_t* __restrict__ adjN) {
  const uint32_t ln = lane_id();
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t b = nbig + gw * 32; b < n; b += nw * 32) {
    const uint64_t i = b + ln;
    const bool ok = i < n;
    const uint64_t src = ok ? off[inv[i]] : 0ull;
    const uint64_t dst = ok ? offN[i] : 0ull;
    const uint32_t d = ok ? (uint32_t)(offN[i + 1] - dst) : 0u;
    uint32_t incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (ln >= (uint32_t)o) incl += y;
    }
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - d;
    for (uint32_t t0 = 0; t0 < total; t0 += 32) {
      const uint32_t t = t0 + ln;
      uint32_t j = 0;
#pragma unroll
      for (uint32_t s = 16; s > 0; s >>= 1) {
        const uint32_t y = __shfl_sync(kFull, incl, j + s - 1);
        if (y <= t) j += s;
      }
      const uint64_t js = __shfl_sync(kFull, src, j), jd = __shfl_sync(kFull, dst, j);
      const uint32_t jx = __shfl_sync(kFull, excl, j);
      if (t < total) adjN[jd + (t - jx)] = rank_other[adj[js + (t - jx)]];
    }
  }
}

__global__ void k_relabel_fill_big(uint32_t nbig, const uint32_t* __restrict__ inv, const uint64_t* __restrict__ off,
                                   const uint32_t* __restrict__ adj, const uint64_t* __restrict__ offN,
                                   const uint32_t* __restrict__ rank_other, uint32_t* __restrict__ adjN) {
  for (uint32_t i = blockIdx.x; i < nbig; i += gridDim.x) {
    const uint64_t src = off[inv[i]], dst = offN[i], d = offN[i + 1] - dst;
    for (uint64_t k = threadIdx.x; k < d; k += blockDim.x) adjN[dst + k] = rank_other[adj[src + k]];
  }
}

// ---------------------------------------------------------------- segmented sort
// Lists of the relabeled CSR are sorted by size class (ranks are in decreasing
// degree order, so each class is a contiguous rank range):
//   d <= 32       one thread per list, bitonic network in registers
//   d <= 4096     one CTA per list, bitonic sort in shared memory
//   d >  4096     4096-element chunks sorted like the previous class, then
//                 merge passes (merge-path tiles) doubling the run length
template <uint32_t N>
__device__ __forceinline__ void reg_bitonic(uint32_t (&x)[N]) {
#pragma unroll
  for (uint32_t k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (uint32_t i = 0; i < N; i++) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const uint32_t a = x[i], b = x[l];
          const bool sw = up ? (a > b) : (a < b);
          x[i] = sw ? b : a;
          x[l] = sw ? a : b;
        }
      }
    }
  }
}

template <uint32_t N>
__device__ __forceinline__ void sort_small_list(uint32_t* __restrict__ p, uint32_t d) {
  uint32_t x[N];
#pragma unroll
  for (uint32_t k = 0; k < N; k++) x[k] = k < d ? p[k] : 0xFFFFFFFFu;
  reg_bitonic<N>(x);
#pragma unroll
  for (uint32_t k = 0; k < N; k++)
    if (k < d) p[k] = x[k];
}

// ranks [r0, n) all have degree <= 32
__global__ void k_sort_small(uint32_t r0, uint32_t n, const uint64_t* __restrict__ offN, uint32_t* adjN) {
  for (uint64_t i = r0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = offN[i];
    const uint32_t d = (uint32_t)(offN[i + 1] - s);
    if (d <= 1) continue;
    if (d <= 4) sort_small_list<4>(adjN + s, d);
    else if (d <= 8) sort_small_list<8>(adjN + s, d);
    else if (d <= 16) sort_small_list<16>(adjN + s, d);
    else sort_small_list<32>(adjN + s, d);
  }
}

// One CTA sorts one segment of <= kSortTile entries in shared memory.
// Segments: ranks [r0, r1) (whole lists) then `ntask` explicit (start, len) chunks.
__global__ void __launch_bounds__(kSortThreads) k_sort_tile(uint32_t r0, uint32_t r1, const uint64_t* __restrict__ offN,
                                                            const ulonglong2* __restrict__ tasks, uint32_t ntask,
                                                            uint32_t* adjN) {
  __shared__ uint32_t s[kSortTile];
  const uint32_t nseg = (r1 - r0) + ntask;
  for (uint32_t t = blockIdx.x; t < nseg; t += gridDim.x) {
    uint64_t st;
    uint32_t d;
    if (t < r1 - r0) {
      st = offN[r0 + t];
      d = (uint32_t)(offN[r0 + t + 1] - st);
    } else {
      const ulonglong2 tk = tasks[t - (r1 - r0)];
      st = tk.x;
      d = (uint32_t)tk.y;
    }
    uint32_t N = 32;
    while (N < d) N <<= 1;
    for (uint32_t k = threadIdx.x; k < N; k += blockDim.x) s[k] = k < d ? adjN[st + k] : 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t k = 2; k <= N; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
          const uint32_t l = i ^ j;
          if (l > i) {
            const bool up = (i & k) == 0;
            const uint32_t a = s[i], b = s[l];
            if (up ? (a > b) : (a < b)) {
              s[i] = b;
              s[l] = a;
            }
          }
        }
        __syncthreads();
      }
    }
    for (uint32_t k = threadIdx.x; k < d; k += blockDim.x) adjN[st + k] = s[k];
    __syncthreads();
  }
}

// Merge pass: every task is one output tile of kSortTile entries of one list
// (x = list start, y = list length | tile index << 32); runs of length `run`
// are merged pairwise src -> dst.  Each thread locates its first output on the
// merge path by binary search and then merges sequentially.
constexpr uint32_t kMergePer = kSortTile / kSortThreads;  // outputs per thread
__global__ void __launch_bounds__(kSortThreads) k_merge_pass(const ulonglong2* __restrict__ tasks, uint32_t ntask,
                                                             uint64_t run, const uint32_t* __restrict__ src,
                                                             uint32_t* __restrict__ dst) {
  for (uint32_t t = blockIdx.x; t < ntask; t += gridDim.x) {
    const ulonglong2 tk = tasks[t];
    const uint64_t ls = tk.x, len = tk.y & 0xFFFFFFFFull, tile = tk.y >> 32;
    const uint64_t o0 = tile * kSortTile + (uint64_t)threadIdx.x * kMergePer;  // first output (list-relative)
    if (o0 >= len) continue;
    const uint64_t ps = (o0 / (2 * run)) * (2 * run);  // start of this run pair
    const uint64_t na = min(run, len - ps);
    const uint64_t nb = ps + run < len ? min(run, len - ps - run) : 0;
    const uint32_t* A = src + ls + ps;
    const uint32_t* B = A + na;
    const uint64_t k = o0 - ps;
    // merge path: i + j = k, A[i-1] <= B[j] and B[j-1] < A[i]
    uint64_t lo = k > nb ? k - nb : 0, hi = k < na ? k : na;
    while (lo < hi) {
      const uint64_t i = (lo + hi) >> 1;
      const uint64_t j = k - i;
      if (A[i] <= B[j - 1]) lo = i + 1; else hi = i;
    }
    uint64_t i = lo, j = k - lo;
    uint32_t* D = dst + ls + ps + k;
    const uint64_t cnt = min((uint64_t)kMergePer, na + nb - k);
    for (uint64_t q = 0; q < cnt; q++) {
      const bool takeA = j >= nb || (i < na && A[i] <= B[j]);
      D[q] = takeA ? A[i++] : B[j++];
    }
  }
}

// dst <- src for every task tile (copy back after a merge pass)
__global__ void k_copy_tiles(const ulonglong2* __restrict__ tasks, uint32_t ntask, const uint32_t* __restrict__ src,
                             uint32_t* __restrict__ dst) {
  for (uint32_t t = blockIdx.x; t < ntask; t += gridDim.x) {
    const ulonglong2 tk = tasks[t];
    const uint64_t ls = tk.x, len = tk.y & 0xFFFFFFFFull, tile = tk.y >> 32;
    const uint64_t a = tile * kSortTile, b = min(a + kSortTile, len);
    for (uint64_t q = a + threadIdx.x; q < b; q += blockDim.x) dst[ls + q] = src[ls + q];
  }
}

// θ / supports / plan outputs back to the caller's labels: out[x] = in[rank[x]]
template <class T>
__global__ void k_gather(uint32_t n, const uint32_t* __restrict__ rank, const T* __restrict__ in, T* __restrict__ out) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x)
    out[x] = in[rank[x]];
}

}  // namespace pbng
