// ubench_smem.cu — shared-memory operation throughput on this GPU (B200), for the
// choice of per-wedge aggregation primitive: atomicOr / atomicAdd / atomicCAS /
// plain LDS on random words, and a full packed-hash insert (CAS + add, linear
// probing) at several load factors.  One CTA of 1024 threads per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_smem scripts/ubench_smem.cu && ./ubench_smem
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kWords = 32768;  // 128 KB
constexpr int kIters = 2048;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  return x;
}

template <int OP>
__global__ void __launch_bounds__(1024, 1) k_op(uint32_t* out, uint32_t seed) {
  extern __shared__ uint32_t w[];
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) w[i] = 0;
  __syncthreads();
  uint32_t acc = 0;
  const uint32_t base = (blockIdx.x * 1024u + threadIdx.x) * kIters + seed;
#pragma unroll 4
  for (int it = 0; it < kIters; it++) {
    const uint32_t x = mix(base + it);
    const uint32_t o = x & (kWords - 1);
    if (OP == 0) acc += atomicOr(&w[o], 1u << (x >> 27));
    else if (OP == 1) atomicAdd(&w[o], 1u);
    else if (OP == 2) acc += atomicCAS(&w[o], 0u, x | 1u);
    else if (OP == 3) acc += w[o];
    else if (OP == 4) atomicOr(&w[o], 1u << (x >> 27));  // no return
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// packed hash insert: T slots, keys drawn from a pool of `distinct` ids so that the
// table reaches load distinct/T; slot = (x + 1) << 7 | count
__global__ void __launch_bounds__(1024, 1) k_hash(uint32_t* out, uint32_t seed, uint32_t T, uint32_t distinct) {
  extern __shared__ uint32_t w[];
  for (int i = threadIdx.x; i < (int)T; i += blockDim.x) w[i] = 0;
  __syncthreads();
  const uint32_t base = (blockIdx.x * 1024u + threadIdx.x) * kIters + seed;
  for (int it = 0; it < kIters / 8; it++) {
    const uint32_t x = mix(base + it) % distinct;
    const uint32_t key = (x + 1u) << 7;
    uint32_t h = __umulhi(x * 0x9E3779B1u, T);
    for (;;) {
      const uint32_t old = atomicCAS(&w[h], 0u, key | 1u);
      if (old == 0u) break;
      if ((old >> 7) == x + 1u) {
        atomicAdd(&w[h], 1u);
        break;
      }
      if (++h == T) h = 0;
    }
  }
  if (w[threadIdx.x] == 0x12345678u) out[0] = 1;
}

// same with read-before-CAS probing (plain LDS until key or empty)
__global__ void __launch_bounds__(1024, 1) k_hash_rd(uint32_t* out, uint32_t seed, uint32_t T, uint32_t distinct) {
  extern __shared__ uint32_t w[];
  for (int i = threadIdx.x; i < (int)T; i += blockDim.x) w[i] = 0;
  __syncthreads();
  const uint32_t base = (blockIdx.x * 1024u + threadIdx.x) * kIters + seed;
  for (int it = 0; it < kIters / 8; it++) {
    const uint32_t x = mix(base + it) % distinct;
    const uint32_t key = (x + 1u) << 7;
    uint32_t h = __umulhi(x * 0x9E3779B1u, T);
    for (;;) {
      uint32_t cur = ((volatile uint32_t*)w)[h];
      if (cur == 0u) {
        cur = atomicCAS(&w[h], 0u, key | 1u);
        if (cur == 0u) break;
      }
      if ((cur >> 7) == x + 1u) {
        atomicAdd(&w[h], 1u);
        break;
      }
      if (++h == T) h = 0;
    }
  }
  if (w[threadIdx.x] == 0x12345678u) out[0] = 1;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  uint32_t* out;
  cudaMalloc(&out, 4);
  const size_t smem = kWords * 4;
  cudaFuncSetAttribute(k_op<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_op<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_op<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_op<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_op<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_hash, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_hash_rd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"atomicOr_ret", "atomicAdd_noret", "atomicCAS", "lds", "atomicOr_noret"};
  std::printf("{\"sms\": %d, \"clock_khz\": %d", nsm, clk);
  for (int op = 0; op < 5; op++) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
      cudaEventRecord(a);
      switch (op) {
        case 0: k_op<0><<<nsm, 1024, smem>>>(out, rep); break;
        case 1: k_op<1><<<nsm, 1024, smem>>>(out, rep); break;
        case 2: k_op<2><<<nsm, 1024, smem>>>(out, rep); break;
        case 3: k_op<3><<<nsm, 1024, smem>>>(out, rep); break;
        case 4: k_op<4><<<nsm, 1024, smem>>>(out, rep); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best) best = ms;
    }
    const double per = (double)nsm * 1024 * kIters / (best * 1e-3);
    std::printf(", \"%s_per_sm_clk\": %.3f", names[op], per / nsm / (clk * 1e3));
  }
  const uint32_t T = 22528;
  const double loads[] = {0.25, 0.5, 0.67, 0.8};
  for (int v = 0; v < 2; v++)
    for (double ld : loads) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(a);
        if (v == 0) k_hash<<<nsm, 1024, smem>>>(out, rep, T, (uint32_t)(ld * T));
        else k_hash_rd<<<nsm, 1024, smem>>>(out, rep, T, (uint32_t)(ld * T));
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
      }
      const double per = (double)nsm * 1024 * (kIters / 8) / (best * 1e-3);
      std::printf(", \"hash%s_load%.2f_per_sm_clk\": %.3f", v ? "_rd" : "", ld, per / nsm / (clk * 1e3));
    }
  std::printf("}\n");
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
