// kernels_level.cuh — retrieval of one level of the k-tip hierarchy from the
// tip numbers ("any level of the k-tip hierarchy can be quickly
// retrieved" from θ).  The level is the subgraph induced on
// U_k = {u : θ_u >= k} and all of V (Def. 2, V(H) = V(G)); its
// k-tips are the classes of U_k under butterfly connectivity: u ~ u' when
// they share >= 2 neighbours (one butterfly).  Those pairs are found by the
// LINK mode of the aggregation tiers (kernels_cd.cuh); these kernels mark the
// members, initialise the union-find and turn roots into canonical labels.
#pragma once
#include "kernels_cd.cuh"

namespace pbng {

constexpr uint32_t kLevelOut = 0u;  // part[] of a non-member (any value != kUnassigned)

// caller id x -> internal id rank[x]: membership, singleton sets, label slots
__global__ void k_level_mark(uint32_t n, const uint32_t* __restrict__ rank, const uint64_t* __restrict__ tip,
                             uint64_t k, uint32_t* __restrict__ part, uint32_t* __restrict__ cc,
                             uint32_t* __restrict__ minlab) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = rank[x];
    part[i] = tip[x] >= k ? kUnassigned : kLevelOut;
    cc[i] = i;
    minlab[i] = 0xFFFFFFFFu;
  }
}

// per U-edge (u, v) of a member u: position of u in the member prefix of N_v
// (lists are sorted by internal id and stay sorted under deletion), i.e. the
// number of members of N_v with a smaller id.  Edge-parallel; u by binary
// search over offU.
__global__ void k_level_cut(uint32_t nU, uint64_t m, const uint64_t* __restrict__ offU,
                            const uint32_t* __restrict__ adjU, const uint64_t* __restrict__ offV,
                            const uint32_t* __restrict__ adjL, const uint32_t* __restrict__ ld,
                            const uint32_t* __restrict__ part, uint32_t* __restrict__ cut) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nU;  // largest u with offU[u] <= e
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (offU[mid] <= e) lo = mid; else hi = mid;
    }
    const uint32_t u = lo;
    uint32_t c = 0;
    if (part[u] == kUnassigned) {
      const uint32_t v = adjU[e];
      const uint32_t* p = adjL + offV[v];
      uint32_t a = 0, b = ld[v];
      while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if (p[mid] < u) a = mid + 1; else b = mid;
      }
      c = a;
    }
    cut[e] = c;
  }
}

// smallest caller id of every set, stored at its root
__global__ void k_level_minlab(uint32_t n, const uint32_t* __restrict__ rank, const uint32_t* __restrict__ part,
                               uint32_t* cc, uint32_t* minlab) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = rank[x];
    if (part[i] == kUnassigned) atomicMin(&minlab[cc_find(cc, i)], (uint32_t)x);
  }
}

// out[x] = smallest caller id of x's k-tip, or 0xFFFFFFFF outside the level;
// ncomp counts the members that label their own k-tip
__global__ void k_level_label(uint32_t n, const uint32_t* __restrict__ rank, const uint32_t* __restrict__ part,
                              uint32_t* cc, const uint32_t* __restrict__ minlab, uint32_t* __restrict__ out,
                              uint32_t* ncomp) {
  uint32_t own = 0;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = rank[x];
    uint32_t lab = 0xFFFFFFFFu;
    if (part[i] == kUnassigned) {
      lab = minlab[cc_find(cc, i)];
      own += lab == (uint32_t)x;
    }
    out[x] = lab;
  }
  own = warp_sum(own);
  if (lane_id() == 0 && own) atomicAdd(ncomp, own);
}

}  // namespace pbng
