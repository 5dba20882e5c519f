// Dependent random 4-byte reads through a random cyclic list of 2^28 nodes
// (the list-ranking walk's access pattern, as rand_read_perm.cu) under each
// cudaLimitMaxL2FetchGranularity setting: how many DRAM bytes one random
// successor read costs, and how fast the chase runs.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/l2_fetch_gran scripts/micro/l2_fetch_gran.cu
#include <cuda_runtime.h>
#include <thrust/device_ptr.h>
#include <thrust/random.h>
#include <thrust/sequence.h>
#include <thrust/shuffle.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__global__ void chase(const uint32_t* __restrict__ succ, uint32_t n, int steps, uint32_t* sink) {
  uint32_t cur = (uint32_t)((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 2654435761ull % n);
  for (int s = 0; s < steps; ++s) cur = ld_cg(succ + cur);
  if (cur == 0xffffffffu) *sink = cur;
}

__global__ void link(const uint32_t* __restrict__ order, uint32_t n, uint32_t* __restrict__ succ) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    succ[order[i]] = order[(i + 1) % n];
}

int main() {
  const uint32_t n = 1u << 28;
  uint32_t *succ, *order, *sink;
  cudaMalloc(&succ, (size_t)n * 4);
  cudaMalloc(&order, (size_t)n * 4);
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  thrust::device_ptr<uint32_t> o(order);
  thrust::sequence(o, o + n);
  thrust::shuffle(o, o + n, thrust::default_random_engine(42));
  link<<<sms * 8, 256>>>(order, n, succ);
  cudaDeviceSynchronize();
  size_t def = 0;
  cudaDeviceGetLimit(&def, cudaLimitMaxL2FetchGranularity);
  printf("default cudaLimitMaxL2FetchGranularity = %zu\n", def);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t g : {(size_t)32, (size_t)64, (size_t)128, def}) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    for (int bps : {4, 16}) {
      const int bl = sms * bps, threads = 128, st = 2048 * 16 / bps;
      chase<<<bl, threads>>>(succ, n, st, sink);
      cudaEventRecord(a);
      chase<<<bl, threads>>>(succ, n, st, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("limit %3zu (set %s, reads back %3zu)  %2d blocks/SM: %7.3f ms  %6.2f G dependent reads/s\n", g,
             cudaGetErrorString(e), got, bps, ms, (double)bl * threads * st / ms / 1e6);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
