// Dependent random 4-byte reads through a TRULY random cyclic permutation of
// 2^28 nodes (the list-ranking walk's access pattern), next to the affine
// permutation of rand_read.cu (succ[i] = a*i + b mod n), whose chains keep a
// regular spacing between threads and are kinder to DRAM than a random list.
// Same geometry: 148 SMs x 16 blocks x 128 threads, 256 steps per thread.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/rand_read_perm scripts/micro/rand_read_perm.cu
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

// succ[order[i]] = order[i+1]: one cycle through all n nodes in random order
__global__ void link(const uint32_t* __restrict__ order, uint32_t n, uint32_t* __restrict__ succ) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    succ[order[i]] = order[(i + 1) % n];
}

__global__ void make_affine(uint32_t* succ, uint32_t n, uint32_t a) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    succ[i] = (uint32_t)((i * (uint64_t)a + 12345u) & (n - 1));
}

int main() {
  const uint32_t n = 1u << 28;
  uint32_t *succ, *order, *sink;
  cudaMalloc(&succ, (size_t)n * 4);
  cudaMalloc(&order, (size_t)n * 4);
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 128, blocks = sms * 16, steps = 256;
  const double reads = (double)threads * blocks * steps;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int kind = 0; kind < 2; ++kind) {
    if (kind == 0) {
      make_affine<<<sms * 8, 256>>>(succ, n, 2654435761u | 1u);
    } else {
      thrust::device_ptr<uint32_t> o(order);
      thrust::sequence(o, o + n);
      thrust::shuffle(o, o + n, thrust::default_random_engine(42));
      link<<<sms * 8, 256>>>(order, n, succ);
    }
    cudaDeviceSynchronize();
    // the same number of reads spread over fewer, longer chains
    for (int bps : {16, 8, 6, 4, 3}) {
      const int bl = sms * bps, st = (int)(reads / ((double)bl * threads));
      chase<<<bl, threads>>>(succ, n, st, sink);
      cudaEventRecord(a);
      chase<<<bl, threads>>>(succ, n, st, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%-22s %6d chains x %5d steps: %7.3f ms  %6.2f G dependent reads/s\n",
             kind == 0 ? "affine permutation" : "random cyclic list", bl * threads, st, ms,
             (double)bl * threads * st / ms / 1e6);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
