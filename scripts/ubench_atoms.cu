// ubench_atoms.cu — measured shared-memory atomic throughput on this GPU, the
// per-wedge operation of the aggregation kernels (one atomicOr / atomicAdd on a
// 32-bit shared word per wedge).  Used as the "smem atomics" roofline in bench.py.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_atoms scripts/ubench_atoms.cu
//   ./ubench_atoms  -> one JSON line
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kWords = 32768;  // 128 KB, as the aggregation bitmap
constexpr int kIters = 4096;

// Every lane hits a different word each step (spread addresses, stride 33 words
// across lanes so no two lanes share a bank line pattern), like ids of a sorted
// partner list mapped into a window bitmap.
template <int OP>
__global__ void __launch_bounds__(1024, 1) k_atoms(uint32_t* out, uint32_t seed) {
  extern __shared__ uint32_t w[];
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) w[i] = 0;
  __syncthreads();
  uint32_t x = (threadIdx.x * 2654435761u) ^ seed, acc = 0;
  for (int it = 0; it < kIters; it++) {
    x = x * 1664525u + 1013904223u;
    const uint32_t o = (x >> 8) & (kWords * 32 - 1);
    const uint32_t bit = 1u << (o & 31);
    if (OP == 0) acc += atomicOr(&w[o >> 5], bit) & bit;
    else if (OP == 1) acc += atomicAdd(&w[o >> 5], 1u);
    else acc += w[o >> 5];  // plain LDS
  }
  if (acc == 0xFFFFFFFFu) out[0] = acc;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  uint32_t* out;
  cudaMalloc(&out, 4);
  const size_t smem = kWords * 4;
  cudaFuncSetAttribute(k_atoms<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_atoms<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_atoms<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double rate[3];
  for (int op = 0; op < 3; op++) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; rep++) {
      cudaEventRecord(a);
      if (op == 0) k_atoms<0><<<nsm, 1024, smem>>>(out, rep);
      if (op == 1) k_atoms<1><<<nsm, 1024, smem>>>(out, rep);
      if (op == 2) k_atoms<2><<<nsm, 1024, smem>>>(out, rep);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best) best = ms;
    }
    rate[op] = (double)nsm * 1024 * kIters / (best * 1e-3);
  }
  std::printf("{\"sms\": %d, \"clock_khz\": %d, \"smem_atomic_or_per_s\": %.4e, \"smem_atomic_add_per_s\": %.4e, "
              "\"smem_lds_per_s\": %.4e, \"per_sm_per_clk_or\": %.4f}\n",
              nsm, clk, rate[0], rate[1], rate[2], rate[0] / nsm / (clk * 1e3));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
