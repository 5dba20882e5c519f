// Throughput of 64-bit global atomicAdd on ONE address (the list-ranking
// walk's chunk and sublist counters) when 303K threads each issue one every
// few microseconds, vs. spread over many addresses.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/atomic_rate scripts/micro/atomic_rate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

template <bool AGG>
__global__ void hammer(unsigned long long* ctr, int per_thread, int spread) {
  unsigned long long acc = 0;
  unsigned long long* p = ctr + (spread > 1 ? ((blockIdx.x * blockDim.x + threadIdx.x) % spread) * 32 : 0);
  for (int i = 0; i < per_thread; ++i) acc += atomicAdd(p, 1ull);  // result used: a dependent claim
  if (acc == 0x1234567) ctr[1] = acc;
}

int main() {
  unsigned long long* ctr;
  cudaMalloc(&ctr, 1 << 20);
  cudaMemset(ctr, 0, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int spread : {1, 2, 8, 64, 4096}) {
    const int blocks = sms * 16, threads = 128, per = 32;
    hammer<false><<<blocks, threads>>>(ctr, per, spread);
    cudaEventRecord(a);
    hammer<false><<<blocks, threads>>>(ctr, per, spread);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double n = (double)blocks * threads * per;
    printf("addresses %5d: %8.3f ms for %.1fM atomics = %7.2f G atomics/s\n", spread, ms, n / 1e6, n / ms / 1e6);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
