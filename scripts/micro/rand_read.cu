// Random dependent 4-byte reads (the list-ranking walk): DRAM bytes per read
// under different load flavours and L2 fetch-granularity limits.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/rand_read scripts/micro/rand_read.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) {
  uint32_t v; asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}
__device__ __forceinline__ uint32_t ld_cv(const uint32_t* p) {
  uint32_t v; asm volatile("ld.global.cv.u32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}
__device__ __forceinline__ uint32_t ld_ef(const uint32_t* p, uint64_t pol) {
  uint32_t v; asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol)); return v;
}
__device__ __forceinline__ uint32_t ld_nc_na(const uint32_t* p) {
  uint32_t v; asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}

// each thread chases a pseudo-random chain: next = succ[cur] (succ is a random cyclic permutation)
__global__ void chase(const uint32_t* __restrict__ succ, uint32_t n, int steps, int mode, uint32_t* sink) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint32_t cur = (uint32_t)((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 2654435761ull % n);
  for (int s = 0; s < steps; ++s) {
    const uint32_t* p = succ + cur;
    cur = mode == 0 ? ld_cg(p) : mode == 1 ? ld_cv(p) : mode == 2 ? ld_ef(p, pol) : ld_nc_na(p);
  }
  if (cur == 0xffffffffu) *sink = cur;
}

__global__ void make_perm(uint32_t* succ, uint32_t n, uint32_t a) {
  // succ[i] = (i * a + 1) mod n with a odd, n a power of two: one long cycle-ish permutation
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    succ[i] = (uint32_t)((i * (uint64_t)a + 12345u) & (n - 1));
}

int main() {
  const uint32_t n = 1u << 28;  // 1 GiB of uint32
  uint32_t *succ, *sink;
  cudaMalloc(&succ, (size_t)n * 4);
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  make_perm<<<sms * 8, 256>>>(succ, n, 2654435761u | 1u);
  cudaDeviceSynchronize();
  const int threads = 128, blocks = sms * 16, steps = 256;
  const double reads = (double)threads * blocks * steps;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t gran : {0, 32, 64, 128}) {
    if (gran) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    for (int mode = 0; mode < 4; ++mode) {
      chase<<<blocks, threads>>>(succ, n, steps, mode, sink);
      cudaEventRecord(a);
      chase<<<blocks, threads>>>(succ, n, steps, mode, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("granularity limit %3zu mode %d (%s): %7.3f ms  %6.2f G reads/s\n", got, mode,
             mode == 0 ? "ld.cg" : mode == 1 ? "ld.cv" : mode == 2 ? "ld.cg evict_first" : "ld.nc no_allocate", ms,
             reads / ms / 1e6);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
