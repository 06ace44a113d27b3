// kernels_fd.cuh — fine-grained decomposition (FD) kernels.
//
// Paper: arXiv 2110.12511 ("P:n" = PAPER.md line).
//   FD principle: peel each partition independently from ⋈^init
//   tip FD on the induced subgraph G_i = (U_i, V), edge in exactly one
//   LPT work estimate = wedges of G_i with both endpoints in U_i
//   dynamic task allocation (threads pop partition ids)
// Each partition is peeled level-synchronously inside one CTA: the level
// k = max(k, min live support); every live vertex with support <= k gets
// θ = k and is peeled in the same round (equal to sequential BUP on G_i,
// Alg.2 P:508-531 with the max(θ, ·) floor; exact supports need no clamp).
#pragma once
#include "kernels_cd.cuh"

namespace pbng {

constexpr uint32_t kFdThreads = 512;
#ifndef PBNG_FD_WARP_SLOTS
#define PBNG_FD_WARP_SLOTS 512
#endif
#ifndef PBNG_FD_CTA_SLOTS
#define PBNG_FD_CTA_SLOTS 16384
#endif
constexpr uint32_t kFdWarpSlots = PBNG_FD_WARP_SLOTS;  // per-warp table (light vertices)
constexpr uint32_t kFdWarpCap = kFdWarpSlots / 2;
constexpr uint32_t kFdCtaSlots = PBNG_FD_CTA_SLOTS;    // CTA table (medium vertices)
constexpr uint32_t kFdCtaCap = kFdCtaSlots / 2;
constexpr uint32_t kFdLogCtaSlots = 31 - __builtin_clz(PBNG_FD_CTA_SLOTS);
constexpr uint64_t kFdWarpWork = 1u << 15;  // wedges above which a vertex goes to the whole CTA

// ---------------------------------------------------------------- membership
// A vertex with ⋈^init = 0 is in no butterfly of its partition's subgraph: its
// tip number is 0 (θ <= support) and peeling it decrements nobody, so it is
// settled here (θ = 0, peeled) and kept out of the FD member lists.
// pcount[p]: FD members of p (⋈^init > 0); pall[p]: every vertex of p (the
// partner ids of a partition's wedges are drawn from these, which bounds the
// distinct partners of any member)
__global__ void k_part_count(uint32_t nU, const uint32_t* __restrict__ part, const uint64_t* __restrict__ init,
                             uint32_t nparts, uint32_t* pcount, uint32_t* pall) {
  extern __shared__ uint32_t hc[];
  for (uint32_t i = threadIdx.x; i < 2 * nparts; i += blockDim.x) hc[i] = 0;
  __syncthreads();
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nU; u += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = part[u];
    atomicAdd(&hc[nparts + p], 1u);
    if (init[u]) atomicAdd(&hc[p], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nparts; i += blockDim.x) {
    if (hc[i]) atomicAdd(&pcount[i], hc[i]);
    if (hc[nparts + i]) atomicAdd(&pall[i], hc[nparts + i]);
  }
}

// members grouped by partition: members[poff[p] ..) (order inside a group is free)
__global__ void k_part_scatter(uint32_t nU, const uint32_t* __restrict__ part, const uint64_t* __restrict__ init,
                               const uint32_t* __restrict__ poff, uint32_t* pcur, uint32_t* members,
                               uint32_t* __restrict__ state, uint64_t* __restrict__ theta) {
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x; b < nU; b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = b + threadIdx.x;
    bool ok = u < nU;
    if (ok && init[u] == 0) {
      state[u] = 3;
      theta[u] = 0;
      ok = false;
    }
    const uint32_t p = ok ? part[u] : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(kFull, p);
    if (ok) {
      const uint32_t leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (lane_id() == leader) base = atomicAdd(&pcur[p], (uint32_t)__popc(peers));
      base = __shfl_sync(peers, base, leader);
      members[poff[p] + base + __popc(peers & lanemask_lt())] = (uint32_t)u;
    }
  }
}

// first index i in [0, n) of a list sorted by part descending with
// part[list[i]] <= p (strict: < p); n if none.
__device__ __forceinline__ uint32_t desc_bound(const uint32_t* __restrict__ list, uint32_t n,
                                               const uint32_t* __restrict__ part, uint32_t p, bool strict) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint32_t q = part[list[mid]];
    if (strict ? q < p : q <= p) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// For every U-edge (u, v): the segment N_v ∩ U_part[u] of the partition-ordered
// list (seg = lo | hi << 32), and the LPT work estimate
// work[p] = Σ_{u∈U_p} Σ_{v∈N_u} |N_v ∩ U_p| = Σ_v |N_v ∩ U_p|^2  (g13).
// Also counts the vertices whose FD partner bound exceeds the CTA table
// (*nheavy), which decides whether FD needs its dense-counter slots.
__global__ void k_fd_seg(uint32_t nU, const uint64_t* __restrict__ offU, const uint32_t* __restrict__ adjU,
                         const uint64_t* __restrict__ offV, const uint32_t* __restrict__ adjL,
                         const uint32_t* __restrict__ part, uint32_t nparts, uint64_t* __restrict__ seg,
                         unsigned long long* work, uint32_t* nheavy) {
  extern __shared__ unsigned long long sw[];
  for (uint32_t i = threadIdx.x; i < nparts; i += blockDim.x) sw[i] = 0;
  __syncthreads();
  const uint32_t ln = lane_id();
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = gw; u < nU; u += nw) {
    const uint32_t p = part[u];
    unsigned long long acc = 0;
    for (uint64_t e = offU[u] + ln; e < offU[u + 1]; e += 32) {
      const uint32_t v = adjU[e];
      const uint64_t b = offV[v];
      const uint32_t n = (uint32_t)(offV[v + 1] - b);
      const uint32_t lo = desc_bound(adjL + b, n, part, p, false);
      const uint32_t hi = desc_bound(adjL + b, n, part, p, true);
      seg[e] = (uint64_t)lo | ((uint64_t)hi << 32);
      acc += hi - lo;
    }
    acc = warp_sum(acc);
    if (ln == 0 && acc) {
      atomicAdd(&sw[p], acc);
      const uint64_t d = offU[u + 1] - offU[u];
      if (acc - d > kFdCtaCap) atomicAdd(nheavy, 1u);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nparts; i += blockDim.x)
    if (sw[i]) atomicAdd(&work[i], sw[i]);
}

// ---------------------------------------------------------------- FD peel
// One CTA peels one partition level-synchronously (equal to sequential BUP):
//   level advance: k = max(k, min live support); every live vertex with
//                  support <= k is selected (θ = k);
//   cascade:       the selected vertices' wedges decrement their partners;
//                  a partner whose support drops to <= k ("crosser") is
//                  selected in the next round at the same level.
// Crossers are detected by the decrement itself (old > k >= new), so cascade
// rounds cost O(selected).  Level advances scan a candidate BAND holding every
// live vertex with support <= T; T is re-chosen from a histogram when the band
// empties so that the band holds a small share of the partition.
struct FdArgs {
  uint32_t nU;
  const uint64_t* __restrict__ offU;
  const uint32_t* __restrict__ adjU;
  const uint64_t* __restrict__ offV;
  const uint32_t* __restrict__ adjL;
  const uint64_t* __restrict__ seg;
  const uint32_t* __restrict__ poff;
  const uint32_t* __restrict__ pall;   // vertices per partition (distinct-partner bound)
  const uint32_t* __restrict__ order;  // partition ids, decreasing work (LPT)
  uint32_t nparts;
  uint32_t* ticket;
  uint32_t* members;  // per partition: vertices outside the band (compacted at refills)
  uint32_t* cand;     // per partition: band, two buffers (cand, cand2)
  uint32_t* cand2;
  uint32_t* sel;      // per partition: selected vertices, two buffers (sel, sel2)
  uint32_t* sel2;
  uint32_t* selpb;    // partner bound per selected vertex (0 = nothing to update)
  uint32_t* bigl;     // indices (into sel) of selected vertices handled by the whole CTA
  uint64_t* s;        // FD supports, initialised to ⋈^init
  uint32_t* state;    // 0 = member, 1 = band, 2 = selected next round, 3 = peeled
  uint64_t* theta;
  uint32_t* slot_cnt;
  uint32_t* slot_touch;
  uint32_t* slot_dup;
  unsigned long long* wedges;
  unsigned long long* updates;
  uint32_t* rounds_max;
  unsigned long long* ptrace;  // optional: per partition {rounds, wedges, cycles, members} (PBNG_TRACE)
};

struct FdBand {            // shared-memory view of the partition being peeled
  uint32_t* cand;          // current band buffer (partition slice)
  uint32_t* next;          // buffer receiving this round's crossers (partition slice)
  uint32_t nc;             // band entries (grows when decrements cross T)
  uint32_t nx;             // crossers appended this round
  unsigned long long T;    // band threshold
  unsigned long long k;    // level
};

// s[x] -= C(w,2) for a live partition member x; crossers (new <= k) are queued
// for the next round, members whose support drops to <= T join the band.
__device__ __forceinline__ void fd_emit(const FdArgs& a, uint32_t x, uint32_t w, unsigned long long& upd,
                                        FdBand& band) {
  if (w < 2) return;
  const uint32_t st = a.state[x];
  if (st == 3) return;
  const uint64_t d = choose2(w);
  const uint64_t nv = atomicAdd((unsigned long long*)&a.s[x], (unsigned long long)(0ull - d)) - d;
  upd++;
  if (st == 2) return;
  if (nv <= band.k) {
    if (atomicCAS(&a.state[x], st, 2u) == st || (st == 0 && atomicCAS(&a.state[x], 1u, 2u) == 1u))
      band.next[atomicAdd(&band.nx, 1u)] = x;
  } else if (st == 0 && nv <= band.T && atomicCAS(&a.state[x], 0u, 1u) == 0u) {
    band.cand[atomicAdd(&band.nc, 1u)] = x;
  }
}

__global__ void __launch_bounds__(kFdThreads, 1) k_fd(FdArgs a) {
  extern __shared__ uint32_t sm[];
  const uint32_t w = threadIdx.x >> 5, ln = lane_id(), nw = blockDim.x >> 5;
  uint32_t* wkeys = sm + w * (2 * kFdWarpSlots);
  uint32_t* wvals = wkeys + kFdWarpSlots;
  uint32_t* ckeys = sm + nw * (2 * kFdWarpSlots);
  uint32_t* cvals = ckeys + kFdCtaSlots;
  uint32_t* s_long = cvals + kFdCtaSlots;
  __shared__ uint32_t s_nlong, s_ntouch, s_ndup, s_t, s_nbig, s_n0, s_n1;
  __shared__ unsigned long long s_min;
  __shared__ uint32_t s_hist[65];
  __shared__ uint32_t s_pre[kFdThreads];
  __shared__ unsigned long long s_base[kFdThreads];
  __shared__ uint32_t s_scan[33];
  __shared__ FdBand band;
  for (uint32_t i = threadIdx.x; i < nw * 2 * kFdWarpSlots; i += blockDim.x) sm[i] = (i / kFdWarpSlots) % 2 == 0 ? kEmpty : 0u;
  for (uint32_t i = threadIdx.x; i < kFdCtaSlots; i += blockDim.x) {
    ckeys[i] = kEmpty;
    cvals[i] = 0;
  }
  uint32_t* hcnt = a.slot_cnt + (uint64_t)blockIdx.x * a.nU;
  uint32_t* htouch = a.slot_touch + (uint64_t)blockIdx.x * a.nU;
  uint32_t* hdup = a.slot_dup + (uint64_t)blockIdx.x * a.nU;
  const FdLists L{a.adjU, a.offV, a.seg};
  unsigned long long wedges = 0, upd = 0, steps = 0;
  uint32_t rounds_max = 0;
  __syncthreads();
  for (;;) {
    if (threadIdx.x == 0) s_t = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const uint32_t t = s_t;
    __syncthreads();
    if (t >= a.nparts) break;
    const uint32_t p = a.order[t];
    const uint32_t lo = a.poff[p];
    uint32_t* mem = a.members + lo;
    uint32_t* cbuf[2] = {a.cand + lo, a.cand2 + lo};
    uint32_t* sbuf[2] = {a.sel + lo, a.sel2 + lo};
    uint32_t* selpb = a.selpb + lo;
    uint32_t* bigl = a.bigl + lo;
    uint32_t nrest = a.poff[p + 1] - lo;
    const uint32_t psz = a.pall[p] ? a.pall[p] - 1 : 0;
    uint32_t cb = 0, sb = 0;  // current band / selection buffers
    uint32_t rounds = 0;
    const long long t_start = clock64();
    if (threadIdx.x == 0) {
      band.cand = cbuf[0];
      band.next = sbuf[1];
      band.nc = 0;
      band.nx = 0;
      band.T = 0;
      band.k = 0;
    }
    __syncthreads();
    long long ph[4] = {0, 0, 0, 0}, tph = clock64();  // trace: selection, bounds, light, heavy
    for (;;) {
      uint32_t nsel = band.nx;
      uint32_t* sel;
      if (nsel) {
        // ---- cascade round: this level's crossers (already off the band)
        sb ^= 1;
        sel = sbuf[sb];
        for (uint32_t j = threadIdx.x; j < nsel; j += blockDim.x) {
          const uint32_t u = sel[j];
          a.state[u] = 3;
          a.theta[u] = band.k;
        }
      } else {
        // ---- level advance
        uint32_t nc = band.nc;
        if (nc == 0) {
          // band refill: members' minimum m; T from a log histogram of s - m so
          // that about max(1024, nrest/32) members enter; the rest is compacted
          if (threadIdx.x == 0) {
            s_min = ~0ull;
            s_n0 = 0;
          }
          for (uint32_t i = threadIdx.x; i < 65; i += blockDim.x) s_hist[i] = 0;
          __syncthreads();
          uint64_t mn = ~0ull;
          for (uint32_t j = threadIdx.x; j < nrest; j += blockDim.x) {
            const uint32_t u = mem[j];
            if (a.state[u] == 0) {
              const uint64_t v = a.s[u];
              mn = v < mn ? v : mn;
            }
          }
          mn = warp_min_u64(mn);
          if (ln == 0) atomicMin(&s_min, (unsigned long long)mn);
          __syncthreads();
          const uint64_t m = s_min;
          if (m == ~0ull) break;  // partition done
          for (uint32_t j = threadIdx.x; j < nrest; j += blockDim.x) {
            const uint32_t u = mem[j];
            if (a.state[u] == 0) {
              const uint64_t dlt = a.s[u] - m;
              atomicAdd(&s_hist[dlt ? 64 - __clzll((long long)dlt) : 0], 1u);
            }
          }
          __syncthreads();
          const uint32_t target = nrest / 32 > 1024 ? nrest / 32 : 1024;
          uint32_t cum = 0, bb = 0;
          for (; bb < 64; bb++) {
            cum += s_hist[bb];
            if (cum >= target) break;
          }
          const uint64_t span = bb >= 64 ? ~0ull : (bb == 0 ? 0ull : ((1ull << bb) - 1));
          const uint64_t T = span > ~0ull - m ? ~0ull : m + span;
          uint32_t* cur = cbuf[cb];
          for (uint32_t j0 = 0; j0 < nrest; j0 += blockDim.x) {
            const uint32_t j = j0 + threadIdx.x;
            const uint32_t u = j < nrest ? mem[j] : 0u;
            const bool lv = j < nrest && a.state[u] == 0;
            const bool in = lv && a.s[u] <= T;
            if (in) a.state[u] = 1;
            __syncthreads();  // every read of this tile precedes the in-place writes below
            warp_append(in, u, cur, &band.nc);
            warp_append(lv && !in, u, mem, &s_n0);  // in-place: writes trail reads
            __syncthreads();
          }
          nrest = s_n0;
          if (threadIdx.x == 0) band.T = T;
          __syncthreads();
          nc = band.nc;
        }
        // level k = max(k, min support over the band) — every live vertex with
        // support <= T is in the band, so this is the live minimum
        uint32_t* cur = cbuf[cb];
        if (threadIdx.x == 0) s_min = ~0ull;
        __syncthreads();
        {
          uint64_t mn = ~0ull;
          for (uint32_t j = threadIdx.x; j < nc; j += blockDim.x) {
            const uint32_t u = cur[j];
            if (a.state[u] == 1) {
              const uint64_t v = a.s[u];
              mn = v < mn ? v : mn;
            }
          }
          mn = warp_min_u64(mn);
          if (ln == 0) atomicMin(&s_min, (unsigned long long)mn);
        }
        __syncthreads();
        if (s_min == ~0ull) {  // only stale entries left in the band: refill
          if (threadIdx.x == 0) band.nc = 0;
          __syncthreads();
          continue;
        }
        const uint64_t kk = s_min > band.k ? s_min : band.k;
        // select {band : support <= k} (θ = k); the rest moves to the other band buffer
        sel = sbuf[sb];
        uint32_t* oth = cbuf[cb ^ 1];
        if (threadIdx.x == 0) {
          s_n0 = 0;
          s_n1 = 0;
        }
        __syncthreads();
        for (uint32_t j0 = 0; j0 < nc; j0 += blockDim.x) {
          const uint32_t j = j0 + threadIdx.x;
          const uint32_t u = j < nc ? cur[j] : 0u;
          const bool lv = j < nc && a.state[u] == 1;
          const bool sl = lv && a.s[u] <= kk;
          if (sl) {
            a.state[u] = 3;
            a.theta[u] = kk;
          }
          warp_append(sl, u, sel, &s_n0);
          warp_append(lv && !sl, u, oth, &s_n1);
        }
        __syncthreads();
        nsel = s_n0;
        cb ^= 1;
        if (threadIdx.x == 0) {
          band.k = kk;
          band.cand = oth;
          band.nc = s_n1;
        }
        if (nsel == 0) {  // only stale entries were left: refill next time
          __syncthreads();
          continue;
        }
      }
      rounds++;
      __syncthreads();  // every thread has read band.nx / band.nc of this round
      if (a.ptrace) {
        const long long now = clock64();
        ph[0] += now - tph;
        tph = now;
      }
      if (threadIdx.x == 0) {
        band.next = sbuf[sb ^ 1];
        band.nx = 0;
        s_nbig = 0;
      }
      __syncthreads();
      // (3) partner bound of each selected vertex inside G_p
      for (uint32_t j = w; j < nsel; j += nw) {
        const uint32_t u = sel[j];
        const uint64_t e0 = a.offU[u], e1 = a.offU[u + 1];
        if (a.s[u] == 0) {  // in no butterfly with a live vertex: decrements nobody
          if (ln == 0) selpb[j] = 0;
          continue;
        }
        uint64_t wl = 0;
        for (uint64_t e = e0 + ln; e < e1; e += 32) {
          uint64_t b;
          uint32_t len;
          L.get(e, b, len);
          wl += len;
        }
        wl = warp_sum(wl);
        if (ln == 0) {
          const uint64_t d = e1 - e0;
          uint64_t pb = wl - d;  // u appears once in each of its segments
          uint32_t r = 0;
          if (d >= 2 && pb > 0 && a.s[u] != 0) {
            if (pb > psz) pb = psz;  // partners are other vertices of this partition
            r = (uint32_t)pb;
            wedges += wl;
            steps += d;
          }
          // whole-CTA work, step (5): big tables, or long walks a single warp would
          // serialise (flagged in the top bit)
          const bool big = r > kFdWarpCap || (r && wl > kFdWarpWork);
          selpb[j] = big ? (r | 0x80000000u) : r;
          if (big) bigl[atomicAdd(&s_nbig, 1u)] = j;
        }
      }
      __syncthreads();
      if (a.ptrace) {
        const long long now = clock64();
        ph[1] += now - tph;
        tph = now;
      }
      // (4) light: one warp per vertex, per-warp table
      for (uint32_t j = w; j < nsel; j += nw) {
        const uint32_t pb = selpb[j];
        if (pb == 0 || (pb & 0x80000000u)) continue;
        const uint32_t u = sel[j];
        uint32_t logT = ceil_log2(2 * pb);
        logT = logT < 5 ? 5 : logT;
        auto f = [&](bool ok, uint32_t x, uint64_t) {
          if (ok && x != u) hash_insert(wkeys, wvals, logT, x);
        };
        warp_wedges(L, a.offU[u], a.offU[u + 1], a.adjL, f);
        __syncwarp();
        for (uint32_t s = ln; s < (1u << logT); s += 32) {
          const uint32_t key = wkeys[s];
          if (key != kEmpty) {
            const uint32_t wv = wvals[s];
            wkeys[s] = kEmpty;
            wvals[s] = 0;
            fd_emit(a, key, wv, upd, band);
          }
        }
        __syncwarp();
      }
      __syncthreads();
      if (a.ptrace) {
        const long long now = clock64();
        ph[2] += now - tph;
        tph = now;
      }
      // (5) medium / heavy: whole CTA per vertex
      const uint32_t nbig = s_nbig;
      for (uint32_t bj = 0; bj < nbig; bj++) {
        const uint32_t j = bigl[bj];
        const uint32_t pb = selpb[j] & 0x7FFFFFFFu;
        const uint32_t u = sel[j];
        if (pb <= kFdWarpCap) {
          // few distinct partners but a long walk: every warp counts its share of
          // the entries in its own table (no cross-warp contention on hot keys),
          // then the warp tables are summed into the CTA table
          uint32_t logT = ceil_log2(2 * pb);
          logT = logT < 5 ? 5 : logT;
          auto f = [&](bool ok, uint32_t x, uint64_t) {
            if (ok && x != u) hash_insert(wkeys, wvals, logT, x);
          };
          cta_flat_wedges(L, a.offU[u], a.offU[u + 1], a.adjL, s_pre, s_base, s_scan, s_long, &s_nlong, f);
          for (uint32_t s = ln; s < (1u << logT); s += 32) {
            const uint32_t key = wkeys[s];
            if (key != kEmpty) {
              const uint32_t c = wvals[s];
              wkeys[s] = kEmpty;
              wvals[s] = 0;
              hash_add(ckeys, cvals, logT, key, c);
            }
          }
          __syncthreads();
          for (uint32_t s = threadIdx.x; s < (1u << logT); s += blockDim.x) {
            const uint32_t key = ckeys[s];
            if (key != kEmpty) {
              const uint32_t wv = cvals[s];
              ckeys[s] = kEmpty;
              cvals[s] = 0;
              fd_emit(a, key, wv, upd, band);
            }
          }
          __syncthreads();
        } else if (pb <= kFdCtaCap) {
          uint32_t logT = ceil_log2(2 * pb);
          logT = logT > kFdLogCtaSlots ? kFdLogCtaSlots : logT;
          auto f = [&](bool ok, uint32_t x, uint64_t) {
            if (ok && x != u) hash_insert(ckeys, cvals, logT, x);
          };
          cta_flat_wedges(L, a.offU[u], a.offU[u + 1], a.adjL, s_pre, s_base, s_scan, s_long, &s_nlong, f);
          for (uint32_t s = threadIdx.x; s < (1u << logT); s += blockDim.x) {
            const uint32_t key = ckeys[s];
            if (key != kEmpty) {
              const uint32_t wv = cvals[s];
              ckeys[s] = kEmpty;
              cvals[s] = 0;
              fd_emit(a, key, wv, upd, band);
            }
          }
          __syncthreads();
        } else {
          if (threadIdx.x == 0) {
            s_ntouch = 0;
            s_ndup = 0;
          }
          __syncthreads();
          auto f = [&](bool ok, uint32_t x, uint64_t) {
            bool first = false, second = false;
            if (ok && x != u) {
              const uint32_t old = atomicAdd(&hcnt[x], 1u);
              first = old == 0;
              second = old == 1;
            }
            uint32_t m = __ballot_sync(kFull, first);
            if (m) {
              uint32_t base = 0;
              const uint32_t leader = __ffs(m) - 1;
              if (ln == leader) base = atomicAdd(&s_ntouch, (uint32_t)__popc(m));
              base = __shfl_sync(kFull, base, leader);
              if (first) htouch[base + __popc(m & lanemask_lt())] = x;
            }
            m = __ballot_sync(kFull, second);
            if (m) {
              uint32_t base = 0;
              const uint32_t leader = __ffs(m) - 1;
              if (ln == leader) base = atomicAdd(&s_ndup, (uint32_t)__popc(m));
              base = __shfl_sync(kFull, base, leader);
              if (second) hdup[base + __popc(m & lanemask_lt())] = x;
            }
          };
          cta_flat_wedges(L, a.offU[u], a.offU[u + 1], a.adjL, s_pre, s_base, s_scan, s_long, &s_nlong, f);
          const uint32_t nd = s_ndup, nt = s_ntouch;
          for (uint32_t q = threadIdx.x; q < nd; q += blockDim.x) {
            const uint32_t key = hdup[q];
            fd_emit(a, key, hcnt[key], upd, band);
          }
          __syncthreads();
          for (uint32_t q = threadIdx.x; q < nt; q += blockDim.x) hcnt[htouch[q]] = 0;
          __syncthreads();
        }
      }
      __syncthreads();
      if (a.ptrace) {
        const long long now = clock64();
        ph[3] += now - tph;
        tph = now;
      }
    }
    rounds_max = rounds > rounds_max ? rounds : rounds_max;
    if (a.ptrace && threadIdx.x == 0) {
      a.ptrace[8 * p + 0] = rounds;
      a.ptrace[8 * p + 1] = clock64() - t_start;
      a.ptrace[8 * p + 3] = a.poff[p + 1] - lo;
      for (int q = 0; q < 4; q++) a.ptrace[8 * p + 4 + q] = ph[q];
    }
  }
  wedges = warp_sum(wedges);
  upd = warp_sum(upd);
  steps = warp_sum(steps);
  if (ln == 0) {
    if (wedges) atomicAdd(a.wedges, wedges);
    if (upd) atomicAdd(a.updates, upd);
    if (steps) atomicAdd(a.wedges + 2, steps);
  }
  if (threadIdx.x == 0) atomicMax(a.rounds_max, rounds_max);
}

}  // namespace pbng

namespace pbng {

// ---------------------------------------------------------------- FD on the grid
// A partition whose FD work is far above the average but whose members are few
// (the densest core, highest tip numbers) would keep one SM busy long after the
// others finished.  It is peeled instead in host-driven rounds that use every
// SM: the same level-synchronous rule (level k = max(k, min live support);
// peel every live member with support <= k), with the wedges of the selected
// members spread over all CTAs and w counted per (selected, member) pair in
// shared memory, indexed by the member's position in the partition.
constexpr uint32_t kGridCnt = 36864;  // (selected x members) counters per CTA (144 KB)
constexpr uint32_t kGridMaxMembers = 4096;
constexpr uint32_t kGridThreads = 512;

// lpos[members[i]] = i
__global__ void k_fdg_pos(const uint32_t* __restrict__ members, uint32_t n, uint32_t* __restrict__ lpos) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) lpos[members[i]] = i;
}

// One CTA: select up to maxsel live members with support <= k (θ = k), and the
// prefix of their degrees.  ctl = {level, nsel, total edges}.
__global__ void __launch_bounds__(1024) k_fdg_select(const uint32_t* __restrict__ members, uint32_t n,
                                                     const uint64_t* __restrict__ offU, uint64_t* s,
                                                     uint32_t* state, uint64_t* theta, uint32_t maxsel,
                                                     uint32_t* sel, uint64_t* selpre, unsigned long long* ctl) {
  __shared__ unsigned long long s_min;
  __shared__ uint32_t s_n, s_scan[33];
  if (threadIdx.x == 0) {
    s_min = ~0ull;
    s_n = 0;
  }
  __syncthreads();
  uint64_t mn = ~0ull;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t u = members[i];
    if (state[u] == 0) mn = s[u] < mn ? s[u] : mn;
  }
  mn = warp_min_u64(mn);
  if (lane_id() == 0) atomicMin(&s_min, (unsigned long long)mn);
  __syncthreads();
  if (s_min == ~0ull) {
    if (threadIdx.x == 0) ctl[1] = 0;
    return;
  }
  const uint64_t k = s_min > ctl[0] ? s_min : ctl[0];
  for (uint32_t i0 = 0; i0 < n; i0 += blockDim.x) {
    const uint32_t i = i0 + threadIdx.x;
    const uint32_t u = i < n ? members[i] : 0u;
    bool take = i < n && state[u] == 0 && s[u] <= k;
    const uint32_t m = __ballot_sync(kFull, take);
    uint32_t base = 0;
    const uint32_t leader = m ? __ffs(m) - 1 : 0;
    if (m && lane_id() == leader) base = atomicAdd(&s_n, (uint32_t)__popc(m));
    base = __shfl_sync(kFull, base, leader);
    const uint32_t slot = base + __popc(m & lanemask_lt());
    if (take && slot < maxsel) {
      sel[slot] = u;
      state[u] = 3;
      theta[u] = k;
    }
  }
  __syncthreads();
  const uint32_t ns = s_n < maxsel ? s_n : maxsel;
  // degree prefix of the selected members (ns <= blockDim)
  const uint32_t d = threadIdx.x < ns ? (uint32_t)(offU[sel[threadIdx.x] + 1] - offU[sel[threadIdx.x]]) : 0u;
  uint32_t tot;
  const uint32_t pre = block_excl_scan(d, s_scan, &tot);
  if (threadIdx.x < ns) selpre[threadIdx.x] = pre;
  if (threadIdx.x == 0) {
    selpre[ns] = tot;
    ctl[0] = k;
    ctl[1] = ns;
    ctl[2] = tot;
  }
}

// All CTAs: w(selected j, member l) over the selected members' wedges inside G_p.
__global__ void __launch_bounds__(kGridThreads) k_fdg_agg(const uint32_t* __restrict__ sel, const uint64_t* __restrict__ selpre,
                                                          uint32_t nsel, uint32_t psz, const uint64_t* __restrict__ offU,
                                                          const uint32_t* __restrict__ adjU,
                                                          const uint64_t* __restrict__ offV,
                                                          const uint64_t* __restrict__ seg,
                                                          const uint32_t* __restrict__ adjL,
                                                          const uint32_t* __restrict__ lpos,
                                                          const uint32_t* __restrict__ state, uint32_t* gcnt,
                                                          unsigned long long* wedges) {
  extern __shared__ uint32_t cnt[];
  __shared__ uint64_t s_pre[1025];
  const uint32_t nc = nsel * psz;
  for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) cnt[i] = 0;
  for (uint32_t i = threadIdx.x; i <= nsel; i += blockDim.x) s_pre[i] = selpre[i];
  __syncthreads();
  const uint64_t total = s_pre[nsel];
  const FdLists L{adjU, offV, seg};
  unsigned long long wl = 0;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nsel;  // selected member j: s_pre[j] <= t < s_pre[j + 1]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_pre[mid] <= t) lo = mid; else hi = mid;
    }
    const uint32_t u = sel[lo];
    uint64_t base;
    uint32_t len;
    L.get(offU[u] + (t - s_pre[lo]), base, len);
    wl += len;
    for (uint32_t q = 0; q < len; q++) {
      const uint32_t x = adjL[base + q];
      if (x == u) continue;
      const uint32_t l = lpos[x];
      if (l != 0xFFFFFFFFu && state[x] == 0) atomicAdd(&cnt[lo * psz + l], 1u);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x)
    if (cnt[i]) atomicAdd(&gcnt[i], cnt[i]);
  wl = warp_sum(wl);
  if (lane_id() == 0 && wl) atomicAdd(wedges, wl);
}

// Apply the decrements C(w, 2) of this round and clear the counters.
__global__ void k_fdg_apply(uint32_t nc, uint32_t psz, const uint32_t* __restrict__ members, uint32_t* gcnt, uint64_t* s,
                            unsigned long long* updates) {
  unsigned long long upd = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    const uint32_t w = gcnt[i];
    if (!w) continue;
    gcnt[i] = 0;
    if (w >= 2) {
      atomicAdd((unsigned long long*)&s[members[i % psz]], (unsigned long long)(0ull - choose2(w)));
      upd++;
    }
  }
  upd = warp_sum(upd);
  if (lane_id() == 0 && upd) atomicAdd(updates, upd);
}

}  // namespace pbng
