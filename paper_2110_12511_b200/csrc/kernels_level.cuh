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
