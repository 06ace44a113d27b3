// kernels_edge.cuh — per-edge butterfly counting (Alg.1 "pveBcnt", per-edge
// part): ⋈_e = number of butterflies of G that
// contain edge e (notation table).
//
// Vertex-priority expansion as in kernels_vp.cuh: ranks follow decreasing
// degree (U before V on ties), lists are sorted by rank, so the lasts Alg.1
// expands from a start (l.11: last ranked above both mid and start) are a
// PREFIX of each mid's list — the first cutM[mid] entries (ranked above mid),
// cut again at the start's own id.  Starts run on both sides, one launch
// sequence per side (start side S, mid side M):
//   pass 1  wedge_count[last] += 1 over every wedge (mid, last)   (l.9-13)
//   pass 2  for every wedge with c = wedge_count[last] >= 2:       (l.27-30)
//             ⋈_(start,mid) += c - 1   -> accS[position of mid in N_start]
//             ⋈_(mid,last)  += c - 1   -> accM[position of last in N_mid]
// Every butterfly is expanded from exactly one start (the vertex opposite its
// top-ranked vertex), for any total order, so the sums are exact.  An edge is
// stored twice (in the U and the V CSR); its count is accU[p] + accV[q], with
// p / q its positions in the two relabeled CSRs, gathered into the caller's
// CSR order by k_edge_gather.
//
// Tiers by the start's wedge bound pb = Σ_mid cutM[mid]:
//   W  cap <= kEdgeWarpPb    warp per start, per-warp smem hash (512 slots)
//   C  cap <= kEdgeCtaPb     CTA per start, CTA smem hash (8192 slots)
//   D  larger                persistent CTA per start: dense counters over the
//                            last ids (< start id) in shared memory when the
//                            start id is below kEdgeDenseSmem, else a 16384-slot
//                            shared hash when cap <= 2·kEdgeCtaPb, else dense
//                            counters in a per-CTA global array cleared by a
//                            third walk
// with pb the start's exact wedge count and cap = min(pb, start id) the most
// distinct lasts it can see.  Hash tables keep a list of their filled slots,
// so clearing costs the start's distinct lasts.
// Inside every tier a warp walks 32 mids at a time, their prefixes flattened
// over the lanes (inclusive scan of the prefix lengths, owner lane found by a
// 5-step shuffle search), so short and long prefixes keep all lanes busy; the
// per-(start,mid) sums of pass 2 are combined in shared memory and written
// once per mid (the start owns that entry in this launch).
#pragma once
#include "device_common.cuh"

namespace pbng {

#ifndef PBNG_EDGE_WARP_PB
#define PBNG_EDGE_WARP_PB 256
#endif
#ifndef PBNG_EDGE_CTA_PB
#define PBNG_EDGE_CTA_PB 4096
#endif
#ifndef PBNG_EDGE_DENSE_SMEM
#define PBNG_EDGE_DENSE_SMEM 49152
#endif
constexpr uint32_t kEdgeWarpPb = PBNG_EDGE_WARP_PB;  // test builds lower the tier bounds
constexpr uint32_t kEdgeWarpLog = 9;          // 512 slots per warp: 5 CTAs of 8 warps per SM
constexpr uint32_t kEdgeWarpThreads = 256;
constexpr uint32_t kEdgeCtaPb = PBNG_EDGE_CTA_PB;
constexpr uint32_t kEdgeCtaLog = 13;          // 8192 slots (+ filled-slot list): two CTAs per SM
constexpr uint32_t kEdgeCtaThreads = 512;
constexpr uint32_t kEdgeDenseSmem = PBNG_EDGE_DENSE_SMEM;  // dense smem counters (192 KB)
constexpr uint32_t kEdgeDenseThreads = 1024;
constexpr uint32_t kEdgeBigLog = 14;          // tier-D shared hash: 16384 slots, <= 8192 keys
constexpr uint32_t kEdgeBigCap = PBNG_EDGE_CTA_PB * 2;
// shared words of the tier-D tables (dense counters or hash + filled list)
constexpr uint32_t kEdgeDenseWords = kEdgeDenseSmem > 2 * (1u << kEdgeBigLog) + kEdgeBigCap
                                         ? kEdgeDenseSmem : 2 * (1u << kEdgeBigLog) + kEdgeBigCap;

struct EdgeArgs {
  uint32_t nS;
  const uint64_t* __restrict__ offS;  // start-side CSR (relabeled)
  const uint32_t* __restrict__ adjS;
  const uint64_t* __restrict__ offM;  // mid-side CSR (relabeled)
  const uint32_t* __restrict__ adjM;
  const uint32_t* __restrict__ cutM;  // entries of N_mid ranked above mid
  uint64_t* accS;                     // per start-side CSR position
  uint64_t* accM;                     // per mid-side CSR position
  uint2* q;                           // tier queues: q[t * nS + i] = (start, cap)
  uint32_t* nq;                       // [3] queue lengths, [3] tier-D ticket
  unsigned long long* wedges;         // Alg.1 wedges expanded (pass 1), may be null
  uint32_t* plen;                     // per start-side edge: prefix length (written by k_edge_classify)
  uint32_t* dense;                    // tier-D global counters, nS per CTA
};

__device__ __forceinline__ uint32_t edge_lower_bound(const uint32_t* __restrict__ p, uint32_t n, uint32_t key) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// wedge-count tables: add one occurrence / read / clear
// open addressing with a list of the slots filled, so that clearing costs the
// distinct keys, not the table size
struct EdgeHash {
  static constexpr bool kRewalk = false;
  uint32_t* keys;
  uint32_t* vals;
  uint32_t* list;  // filled slots (at most the table's key cap)
  uint32_t* n;
  uint32_t logT;
  __device__ __forceinline__ void add(uint32_t k) {
    const uint32_t f = hash_insert_new(keys, vals, logT, k);
    if (f != 0xFFFFFFFFu) list[atomicAdd(n, 1u)] = f;
  }
  __device__ __forceinline__ uint32_t get(uint32_t k) const { return hash_lookup(keys, vals, logT, k); }
  __device__ __forceinline__ void clear(uint32_t) {}
  __device__ __forceinline__ void reset(uint32_t tid, uint32_t nt) {
    const uint32_t c = *(volatile uint32_t*)n;
    for (uint32_t j = tid; j < c; j += nt) {
      const uint32_t f = list[j];
      keys[f] = kEmpty;
      vals[f] = 0;
    }
  }
};
struct EdgeDenseSmem {
  static constexpr bool kRewalk = false;
  uint32_t* cnt;
  __device__ __forceinline__ void add(uint32_t k) { atomicAdd(&cnt[k], 1u); }
  __device__ __forceinline__ uint32_t get(uint32_t k) const { return cnt[k]; }
  __device__ __forceinline__ void clear(uint32_t) {}
};
struct EdgeDenseGlobal {
  static constexpr bool kRewalk = true;
  uint32_t* cnt;
  __device__ __forceinline__ void add(uint32_t k) { atomicAdd(&cnt[k], 1u); }
  __device__ __forceinline__ uint32_t get(uint32_t k) const { return __ldcg(&cnt[k]); }
  __device__ __forceinline__ void clear(uint32_t k) { __stcg(&cnt[k], 0u); }
};

// One warp walks mids [g0 + 32*wi, e1) in groups of 32 (stride 32*nw) of start s.
// PASS 1: count; PASS 2: attribute c - 1; PASS 3: clear (global dense only).
// s_sum: 32 u64 of this warp's shared scratch.  Returns the wedges walked.
template <int PASS, class Tab>
__device__ __forceinline__ uint64_t edge_walk(const EdgeArgs& a, uint32_t s, uint64_t e0, uint64_t e1, uint32_t wi,
                                              uint32_t nw, Tab& t, unsigned long long* s_sum) {
  const uint32_t ln = lane_id();
  uint64_t walked = 0;
  for (uint64_t g = e0 + 32ull * wi; g < e1; g += 32ull * nw) {
    const uint64_t e = g + ln;
    uint32_t len = 0;
    uint64_t base = 0;
    if (e < e1) {
      len = a.plen[e];  // ranked above mid and below s (k_edge_classify)
      if (len) base = a.offM[a.adjS[e]];
    }
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (ln >= (uint32_t)o) incl += y;
    }
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - len;
    if (PASS == 2) {
      s_sum[ln] = 0;
      __syncwarp();
    }
    walked += total;
    for (uint32_t kb = 0; kb < total; kb += 32) {
      const uint32_t k = kb + ln;
      // owner = number of lanes whose inclusive end is <= k
      uint32_t pos = 0;
#pragma unroll
      for (uint32_t step = 16; step > 0; step >>= 1) {
        const uint32_t y = __shfl_sync(kFull, incl, pos + step - 1);
        if (y <= k) pos += step;
      }
      const uint32_t owner = pos > 31 ? 31 : pos;
      const uint32_t oex = __shfl_sync(kFull, excl, owner);
      const uint64_t ob = __shfl_sync(kFull, base, owner);
      if (k < total) {
        const uint64_t f = ob + (k - oex);
        const uint32_t last = a.adjM[f];
        PBNG_DCHECK(last < s);
        if (PASS == 1) t.add(last);
        if (PASS == 2) {
          const uint32_t c = t.get(last);
          PBNG_DCHECK(c >= 1);
          if (c >= 2) {
            red_add_u64(a.accM + f, (uint64_t)(c - 1));
            atomicAdd(&s_sum[owner], (unsigned long long)(c - 1));
          }
        }
        if (PASS == 3) t.clear(last);
      }
    }
    if (PASS == 2) {
      __syncwarp();
      if (e < e1 && s_sum[ln]) a.accS[e] += s_sum[ln];  // entry e belongs to this start only
      __syncwarp();
    }
  }
  return walked;
}

// Same passes with the whole CTA flattened over the wedges: mids are taken
// blockDim at a time (one per thread: prefix length by binary search, block
// scan), then every thread takes wedges t, t + blockDim, ... of the chunk and
// finds its mid by binary search over the scanned lengths, so a start with a
// few long prefixes keeps every warp busy.  Pass-2 sums per mid are combined
// in shared memory and added to accS once per mid.  Contains __syncthreads.
struct EdgeCtaScratch {
  uint32_t pre[kEdgeDenseThreads];
  unsigned long long base[kEdgeDenseThreads];
  unsigned long long sum[kEdgeDenseThreads];
  uint32_t scan[33];
};
template <int PASS, class Tab>
__device__ __forceinline__ uint64_t edge_walk_cta(const EdgeArgs& a, uint32_t s, Tab& t, EdgeCtaScratch& sc) {
  const uint64_t e0 = a.offS[s], e1 = a.offS[s + 1];
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  uint64_t walked = 0;
  for (uint64_t c = e0; c < e1; c += nt) {
    const uint32_t nd = (uint32_t)(e1 - c < nt ? e1 - c : nt);
    uint32_t len = 0;
    uint64_t base = 0;
    if (tid < nd) {
      len = a.plen[c + tid];
      if (len) base = a.offM[a.adjS[c + tid]];
    }
    uint32_t total;
    const uint32_t pre = block_excl_scan(len, sc.scan, &total);
    if (tid < nd) {
      sc.pre[tid] = pre;
      sc.base[tid] = base;
      if (PASS == 2) sc.sum[tid] = 0;
    }
    __syncthreads();
    walked += total;
    for (uint32_t k = tid; k < total; k += nt) {
      uint32_t lo = 0, hi = nd;  // largest j with pre[j] <= k
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sc.pre[mid] <= k) lo = mid; else hi = mid;
      }
      const uint64_t f = sc.base[lo] + (k - sc.pre[lo]);
      const uint32_t last = a.adjM[f];
      PBNG_DCHECK(last < s);
      if (PASS == 1) t.add(last);
      if (PASS == 2) {
        const uint32_t cw = t.get(last);
        if (cw >= 2) {
          red_add_u64(a.accM + f, (uint64_t)(cw - 1));
          atomicAdd(&sc.sum[lo], (unsigned long long)(cw - 1));
        }
      }
      if (PASS == 3) t.clear(last);
    }
    __syncthreads();
    if (PASS == 2 && tid < nd && sc.sum[tid]) a.accS[c + tid] += sc.sum[tid];
  }
  return walked;
}

template <class Tab>
__device__ __forceinline__ uint64_t edge_start_cta(const EdgeArgs& a, uint32_t s, Tab& t, EdgeCtaScratch& sc) {
  const uint64_t walked = edge_walk_cta<1>(a, s, t, sc);
  __syncthreads();
  edge_walk_cta<2>(a, s, t, sc);
  __syncthreads();
  if (Tab::kRewalk) {
    edge_walk_cta<3>(a, s, t, sc);
    __syncthreads();
  }
  return walked;
}

// Route every start by its exact Alg.1 wedge count pb = Σ_mid |prefix(mid, s)|
// (warp per start, lanes over mids, one binary search per mid, whose result
// is kept in plen for the walks); the table a start needs holds at most
// cap = min(pb, s) distinct lasts (ids below s).
__global__ void __launch_bounds__(256) k_edge_classify(EdgeArgs a) {
  const uint32_t ln = lane_id();
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t x = gw; x < a.nS; x += nw) {
    const uint64_t e0 = a.offS[x], e1 = a.offS[x + 1];
    if (e1 - e0 < 2 || x == 0) continue;  // a butterfly needs two mids and a last below x
    uint64_t pb = 0;
    for (uint64_t e = e0 + ln; e < e1; e += 32) {
      const uint32_t mid = a.adjS[e];
      const uint32_t len = edge_lower_bound(a.adjM + a.offM[mid], a.cutM[mid], (uint32_t)x);
      a.plen[e] = len;
      pb += len;
    }
    pb = warp_sum(pb);
    if (ln == 0 && pb >= 2) {
      const uint64_t cap = pb < x ? pb : x;
      const uint32_t t = cap <= kEdgeWarpPb ? 0 : (cap <= kEdgeCtaPb ? 1 : 2);
      const uint32_t i = atomicAdd(&a.nq[t], 1u);
      a.q[(uint64_t)t * a.nS + i] = make_uint2((uint32_t)x, (uint32_t)(cap < 0xFFFFFFFFull ? cap : 0xFFFFFFFFull));
    }
  }
}

struct WarpSync {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

// the three passes of one start over a table; `sync` is the barrier of the
// group walking the start (warp or CTA)
template <class Tab, class Sync>
__device__ __forceinline__ uint64_t edge_start(const EdgeArgs& a, uint32_t s, uint32_t wi, uint32_t nw, Tab& t,
                                               unsigned long long* s_sum, Sync sync) {
  const uint64_t e0 = a.offS[s], e1 = a.offS[s + 1];
  const uint64_t walked = edge_walk<1>(a, s, e0, e1, wi, nw, t, s_sum);
  sync();
  edge_walk<2>(a, s, e0, e1, wi, nw, t, s_sum);
  sync();
  if (Tab::kRewalk) {
    edge_walk<3>(a, s, e0, e1, wi, nw, t, s_sum);
    sync();
  }
  return walked;
}

// Tier W: warp per start.
__global__ void __launch_bounds__(kEdgeWarpThreads) k_edge_warp(EdgeArgs a) {
  extern __shared__ uint32_t sm[];
  __shared__ unsigned long long s_sum[kEdgeWarpThreads / 32][32];
  __shared__ uint32_t s_n[kEdgeWarpThreads / 32];
  const uint32_t w = threadIdx.x >> 5, ln = lane_id();
  const uint32_t T = 1u << kEdgeWarpLog;
  uint32_t* base = sm + w * (2 * T + kEdgeWarpPb);
  EdgeHash h{base, base + T, base + 2 * T, &s_n[w], kEdgeWarpLog};
  for (uint32_t i = ln; i < T; i += 32) {
    h.keys[i] = kEmpty;
    h.vals[i] = 0;
  }
  if (ln == 0) s_n[w] = 0;
  __syncwarp();
  const uint32_t n = a.nq[0];
  uint64_t walked = 0;
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + w; i < n; i += gridDim.x * (blockDim.x >> 5)) {
    walked += edge_start(a, a.q[i].x, 0, 1, h, s_sum[w], WarpSync());
    h.reset(ln, 32);
    __syncwarp();
    if (ln == 0) s_n[w] = 0;
    __syncwarp();
  }
  if (a.wedges && ln == 0 && walked) atomicAdd(a.wedges, (unsigned long long)walked);
}

// Tier C: CTA per start.
__global__ void __launch_bounds__(kEdgeCtaThreads) k_edge_cta(EdgeArgs a) {
  extern __shared__ uint32_t sm[];
  __shared__ uint32_t s_n;
  const uint32_t T = 1u << kEdgeCtaLog;
  EdgeCtaScratch& sc = *reinterpret_cast<EdgeCtaScratch*>(sm + 2 * T + kEdgeCtaPb);
  EdgeHash h{sm, sm + T, sm + 2 * T, &s_n, kEdgeCtaLog};
  for (uint32_t i = threadIdx.x; i < T; i += blockDim.x) {
    h.keys[i] = kEmpty;
    h.vals[i] = 0;
  }
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  const uint32_t n = a.nq[1];
  uint64_t walked = 0;
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    walked += edge_start_cta(a, a.q[(uint64_t)a.nS + i].x, h, sc);  // every thread sees the total
    h.reset(threadIdx.x, blockDim.x);
    __syncthreads();
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
  }
  if (a.wedges && threadIdx.x == 0 && walked) atomicAdd(a.wedges, (unsigned long long)walked);
}

// Tier D: persistent CTAs take starts by ticket.  Lasts are ids below s:
//   s <= kEdgeDenseSmem        dense counters in shared memory over [0, s)
//   cap <= kEdgeBigCap         CTA hash of 2^kEdgeBigLog slots in shared memory
//   otherwise                  dense counters in this CTA's global array,
//                              cleared by a third walk
__global__ void __launch_bounds__(kEdgeDenseThreads) k_edge_dense(EdgeArgs a) {
  extern __shared__ uint32_t sm[];
  __shared__ uint32_t s_i, s_n;
  const uint32_t n = a.nq[2];
  EdgeCtaScratch& sc = *reinterpret_cast<EdgeCtaScratch*>(sm + kEdgeDenseWords);
  uint32_t* gcnt = a.dense + (uint64_t)blockIdx.x * a.nS;
  const uint32_t TB = 1u << kEdgeBigLog;
  EdgeHash h{sm, sm + TB, sm + 2 * TB, &s_n, kEdgeBigLog};
  bool hash_ready = false;
  uint64_t walked = 0;
  for (;;) {
    if (threadIdx.x == 0) s_i = atomicAdd(&a.nq[3], 1u);
    __syncthreads();
    const uint32_t i = s_i;
    __syncthreads();
    if (i >= n) break;
    const uint2 qe = a.q[2ull * a.nS + i];
    const uint32_t s = qe.x;
    if (s <= kEdgeDenseSmem) {
      EdgeDenseSmem t{sm};
      for (uint32_t j = threadIdx.x; j < s; j += blockDim.x) sm[j] = 0;
      hash_ready = false;
      __syncthreads();
      walked += edge_start_cta(a, s, t, sc);
    } else if (qe.y <= kEdgeBigCap) {
      if (!hash_ready) {
        for (uint32_t j = threadIdx.x; j < TB; j += blockDim.x) {
          h.keys[j] = kEmpty;
          h.vals[j] = 0;
        }
        if (threadIdx.x == 0) s_n = 0;
        hash_ready = true;
        __syncthreads();
      }
      walked += edge_start_cta(a, s, h, sc);
      h.reset(threadIdx.x, blockDim.x);
      __syncthreads();
      if (threadIdx.x == 0) s_n = 0;
      __syncthreads();
    } else {
      EdgeDenseGlobal t{gcnt};
      walked += edge_start_cta(a, s, t, sc);
    }
  }
  if (a.wedges && threadIdx.x == 0 && walked) atomicAdd(a.wedges, (unsigned long long)walked);
}

// ⋈_e in the caller's CSR order of the output side: caller edge i = (x, y)
// with x = row of i (offsets of the output side), y = idx[i]; its positions
// in the relabeled CSRs are found by binary search in the sorted lists.
__global__ void k_edge_gather(uint32_t nX, uint64_t m, const uint64_t* __restrict__ offX,
                              const uint32_t* __restrict__ idxX, const uint32_t* __restrict__ rankX,
                              const uint32_t* __restrict__ rankY, const uint64_t* __restrict__ offXr,
                              const uint32_t* __restrict__ adjXr, const uint64_t* __restrict__ offYr,
                              const uint32_t* __restrict__ adjYr, const uint64_t* __restrict__ accX,
                              const uint64_t* __restrict__ accY, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nX;  // row: last x with offX[x] <= i
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (offX[mid] <= i) lo = mid; else hi = mid;
    }
    const uint32_t rx = rankX[lo], ry = rankY[idxX[i]];
    const uint64_t bx = offXr[rx], by = offYr[ry];
    const uint64_t p = bx + edge_lower_bound(adjXr + bx, (uint32_t)(offXr[rx + 1] - bx), ry);
    const uint64_t q = by + edge_lower_bound(adjYr + by, (uint32_t)(offYr[ry + 1] - by), rx);
    PBNG_DCHECK(adjXr[p] == ry && adjYr[q] == rx);
    out[i] = accX[p] + accY[q];
  }
}

}  // namespace pbng
