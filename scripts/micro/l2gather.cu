// L2-resident random-gather rate on B200: how many random 8-byte reads per
// second can the SMs issue against an 8 MB array (SpMV's x vector) that lives
// in L2?  This is the bound of the SpMV product phase (one x gather per nnz).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2gather l2gather.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// MODE 0: __ldg; 1: ld.global.nc.L1::no_allocate; 2: ld.global.cg (L2 only)
// Each thread does U independent gathers per iteration, indices precomputed
// in a streamed int32 array (like col_idx) or hashed (no index stream).
template <int MODE, bool IDX, int U, bool VAL = false>
__global__ void __launch_bounds__(256) gather(const double* __restrict__ x, const int* __restrict__ idx,
                                              double* __restrict__ out, uint32_t n, uint32_t mask,
                                              const double* __restrict__ val = nullptr) {
  const uint32_t stride = gridDim.x * blockDim.x * U;
  double acc = 0.0;
  for (uint32_t base = (blockIdx.x * blockDim.x) * U + threadIdx.x; base < n; base += stride) {
    int j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = base + u * blockDim.x;
      j[u] = IDX ? (k < n ? __ldg(idx + k) : 0) : (int)(hash(k) & mask);
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0) v[u] = __ldg(x + j[u]);
      else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[u]) : "l"(x + j[u]));
      else asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v[u]) : "l"(x + j[u]));
    }
    if (VAL) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = base + u * blockDim.x;
        if (k < n) v[u] *= __ldg(val + k);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;  // keep the loads alive
}

__global__ void init(double* x, int* idx, uint32_t nx, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i < nx) x[i] = i * 0.5;
    idx[i] = (int)(hash(i * 3 + 7) % nx);
  }
}

int main() {
  const uint32_t nx = 1u << 20;   // 8 MB of f64
  const uint32_t n = 1u << 24;    // 16M gathers (the SpMV config's nnz)
  double *x, *o;
  int* idx;
  double* val;
  cudaMalloc(&val, (size_t)n * 8);
  cudaMemset(val, 0, (size_t)n * 8);
  cudaMalloc(&x, (size_t)nx * 8);
  cudaMalloc(&o, 64);
  cudaMalloc(&idx, (size_t)n * 4);
  init<<<4096, 256>>>(x, idx, nx, n);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
#define RUNV(M, I, U, G, V)                                                                 \
  {                                                                                         \
    const int grid = sms * G;                                                               \
    for (int r = 0; r < 3; ++r) gather<M, I, U, V><<<grid, 256>>>(x, idx, o, n, nx - 1, val); \
    cudaEventRecord(e0);                                                                    \
    for (int r = 0; r < 10; ++r) gather<M, I, U, V><<<grid, 256>>>(x, idx, o, n, nx - 1, val); \
    cudaEventRecord(e1);                                                                    \
    cudaEventSynchronize(e1);                                                               \
    cudaEventElapsedTime(&ms, e0, e1);                                                      \
    ms /= 10;                                                                               \
    printf("mode %d idx %d val %d U %2d ctas/SM %d: %8.2f us  %7.1f G gathers/s  %6.2f gathers/clk/SM (1.965 GHz)\n", \
           M, (int)I, (int)V, U, G, ms * 1e3, n / ms / 1e6, n / (ms * 1e-3) / sms / 1.965e9);       \
  }
#define RUN(M, I, U, G) RUNV(M, I, U, G, false)
  RUN(0, false, 8, 8) RUN(1, false, 8, 8) RUN(2, false, 8, 8)
  RUN(0, true, 8, 1) RUN(0, true, 8, 2) RUN(0, true, 4, 2) RUN(0, true, 2, 2) RUN(0, true, 16, 1)
  RUNV(0, true, 8, 8, true) RUNV(0, true, 16, 4, true) RUNV(0, true, 8, 2, true) RUNV(0, true, 4, 8, true)
  RUN(0, true, 8, 8) RUN(1, true, 8, 8) RUN(2, true, 8, 8)
  RUN(0, true, 16, 4) RUN(1, true, 16, 4) RUN(0, true, 4, 8) RUN(1, true, 16, 8)
  // L1 capacity left for in-flight misses: pad each CTA with unused dynamic smem
#define RUNS(M, U, G, SM)                                                                   \
  {                                                                                         \
    const int grid = sms * G;                                                               \
    cudaFuncSetAttribute(gather<M, true, U, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM); \
    for (int r = 0; r < 3; ++r) gather<M, true, U, false><<<grid, 256, SM>>>(x, idx, o, n, nx - 1, val); \
    cudaEventRecord(e0);                                                                    \
    for (int r = 0; r < 10; ++r) gather<M, true, U, false><<<grid, 256, SM>>>(x, idx, o, n, nx - 1, val); \
    cudaEventRecord(e1);                                                                    \
    cudaEventSynchronize(e1);                                                               \
    cudaEventElapsedTime(&ms, e0, e1);                                                      \
    ms /= 10;                                                                               \
    printf("mode %d U %2d ctas/SM %d smem/CTA %6d: %8.2f us  %6.2f gathers/clk/SM\n", M, U, G, SM, ms * 1e3, \
           n / (ms * 1e-3) / sms / 1.965e9);                                                \
  }
  // explicit carveout (percent of the unified L1/smem given to shared memory), kernel uses no smem
#define RUNC(M, U, PCT)                                                                     \
  {                                                                                         \
    const int grid = sms;                                                                   \
    cudaFuncSetAttribute(gather<M, true, U, false>, cudaFuncAttributePreferredSharedMemoryCarveout, PCT); \
    for (int r = 0; r < 3; ++r) gather<M, true, U, false><<<grid, 256>>>(x, idx, o, n, nx - 1, val); \
    cudaEventRecord(e0);                                                                    \
    for (int r = 0; r < 10; ++r) gather<M, true, U, false><<<grid, 256>>>(x, idx, o, n, nx - 1, val); \
    cudaEventRecord(e1);                                                                    \
    cudaEventSynchronize(e1);                                                               \
    cudaEventElapsedTime(&ms, e0, e1);                                                      \
    ms /= 10;                                                                               \
    printf("mode %d U %2d carveout %3d%%: %8.2f us  %6.2f gathers/clk/SM\n", M, U, PCT, ms * 1e3, \
           n / (ms * 1e-3) / sms / 1.965e9);                                                \
  }
  {
    const int pcts[] = {0, 4, 7, 13, 25, 39, 50, 52, 64, 75, 77, 86, 90, 100};
    for (int p : pcts) { RUNC(0, 8, p) }
  }
  {
    const int sizes[] = {0, 16384, 32768, 49152, 65536, 81920, 102400, 131072, 163840, 196608, 225000};
    for (int sz : sizes) { RUNS(0, 8, 1, sz) }
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
