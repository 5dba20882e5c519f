// Random-gather sector accounting: which load flavour moves how many sectors per 4-byte random read.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int MODE>
__global__ void gather(const int* __restrict__ a, int* __restrict__ out, uint32_t n, uint32_t mask) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t j = hash(i) & mask;
  int v;
  if (MODE == 0) v = __ldg(a + j);
  else if (MODE == 1) asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(a + j));
  else if (MODE == 2) asm volatile("ld.global.s32 %0, [%1];" : "=r"(v) : "l"(a + j));
  else if (MODE == 3) asm volatile("ld.global.cv.s32 %0, [%1];" : "=r"(v) : "l"(a + j));
  else asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(a + j));
  out[i] = v;
}
// dependent chains: each thread follows a random chain of `steps` loads
template <int MODE>
__global__ void chase(const int* __restrict__ a, int* __restrict__ out, uint32_t nthreads, int steps) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nthreads) return;
  int cur = (int)(hash(i) & 0x0fffffff);
  for (int s = 0; s < steps; ++s) {
    int v;
    if (MODE == 0) v = __ldg(a + cur);
    else asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(a + cur));
    cur = v;
  }
  out[i] = cur;
}
// random 8-byte writes (the list-ranking walk's (sublist, offset) store)
template <int MODE>
__global__ void scatter8(unsigned long long* __restrict__ a, uint32_t m, uint32_t mask) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  uint32_t j = hash(i * 3 + 1) & mask;
  if (MODE == 0) a[j] = i;
  else asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(a + j), "l"((unsigned long long)i) : "memory");
}
__global__ void init(int* a, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = (int)(hash(i * 7 + 1) & (n - 1));
}
int main(int argc, char** argv) {
  const uint32_t n = 1u << 28, m = 1u << 26;
  if (argc > 1) {  // cudaLimitMaxL2FetchGranularity: bytes fetched from DRAM per L2 miss
    const size_t g = (size_t)atoi(argv[1]);
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    printf("L2 fetch granularity request %zu -> %s, now %zu\n", g, cudaGetErrorString(e), got);
  }
  int *a, *o;
  cudaMalloc(&a, (size_t)n * 4); cudaMalloc(&o, (size_t)m * 4);
  init<<<4096, 256>>>(a, n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
#define RUN(M) gather<M><<<m / 256, 256>>>(a, o, m, n - 1); cudaEventRecord(e0); gather<M><<<m / 256, 256>>>(a, o, m, n - 1); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); printf("gather mode %d: %.3f ms, %.2f G loads/s\n", M, ms, m / ms / 1e6);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4)
  const uint32_t nt = 1u << 20; const int steps = 256;
#define CH(M) chase<M><<<nt / 256, 256>>>(a, o, nt, steps); cudaEventRecord(e0); chase<M><<<nt / 256, 256>>>(a, o, nt, steps); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); printf("chase mode %d: %.3f ms, %.2f G loads/s\n", M, ms, (double)nt * steps / ms / 1e6);
  CH(0) CH(1)
  // scatter: 2^26 random 8-B writes into a 1 GiB array (2^27 u64 slots)
#define SC(M) scatter8<M><<<m / 256, 256>>>((unsigned long long*)a, m, (n / 2) - 1); cudaEventRecord(e0); scatter8<M><<<m / 256, 256>>>((unsigned long long*)a, m, (n / 2) - 1); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); printf("scatter8 mode %d: %.3f ms, %.2f G writes/s\n", M, ms, m / ms / 1e6);
  SC(0) SC(1)
  return 0;
}
