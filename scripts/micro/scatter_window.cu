// Random 8-byte stores confined to a sliding window (the list-ranking
// bucketed scatter): DRAM bytes per store vs window size.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/scatter_window scripts/micro/scatter_window.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// entry i targets window (i / per_win), random slot inside it
__global__ void scatter(int64_t* out, int64_t n, int64_t win, int hint) {
  uint64_t keep;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w0 = (i / win) * win;
    const int64_t t = w0 + (int64_t)(mix((uint64_t)i) % (uint64_t)win);
    if (hint) asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(out + t), "l"(i), "l"(keep) : "memory");
    else out[t] = i;
  }
}

// the same, but slot = a permutation inside the window (every slot written once)
__global__ void scatter_perm(int64_t* out, int64_t n, int64_t win) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w0 = (i / win) * win, k = i - w0;
    const int64_t t = w0 + (int64_t)(((uint64_t)k * 2654435761ull + 12345) % (uint64_t)win);
    if (t < n) out[t] = i;
  }
}

int main() {
  const int64_t n = 1ll << 28;
  int64_t* out;
  cudaMalloc(&out, n * 8);
  cudaMemset(out, 0, n * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int64_t wins[] = {1ll << 17, 1ll << 19, 1ll << 20, 1ll << 21, 1ll << 22, 1ll << 24, n};
  for (int mode = 0; mode < 2; ++mode)
    for (int64_t w : wins) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 2) scatter_perm<<<sms * 8, 256>>>(out, n, w);
        else scatter<<<sms * 8, 256>>>(out, n, w, mode);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("mode %d window %9lld entries (%6.1f MB): %7.3f ms  %6.2f G stores/s\n", mode, (long long)w,
                        w * 8 / 1e6, ms, n / ms / 1e6);
      }
    }
  return 0;
}
