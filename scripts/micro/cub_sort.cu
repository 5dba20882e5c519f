// CUB's DeviceRadixSort::SortPairs (the CUDA 12.9 toolkit's onesweep) on the
// sort workload's shape — u32 keys + u32 payload, 2^28 uniform random keys —
// as the library baseline next to libhb200's hb_sort (profiles/micro_cub_sort_r02.txt).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/cub_sort scripts/micro/cub_sort.cu
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__global__ void fill(uint32_t* k, uint32_t* v, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + i * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    k[i] = (uint32_t)(z ^ (z >> 31));
    v[i] = (uint32_t)i;
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int lg : {24, 26, 28, 29}) {
    const size_t n = (size_t)1 << lg;
    uint32_t *k0, *k1, *v0, *v1;
    cudaMalloc(&k0, n * 4);
    cudaMalloc(&k1, n * 4);
    cudaMalloc(&v0, n * 4);
    cudaMalloc(&v1, n * 4);
    void* tmp = nullptr;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int64_t)n);
    cudaMalloc(&tmp, tb);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f, sum = 0;
    const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
      fill<<<sms * 8, 256>>>(k0, v0, n, 12345 + r);
      cudaEventRecord(a);
      cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int64_t)n);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 2) {
        sum += ms;
        best = ms < best ? ms : best;
      }
    }
    printf("cub SortPairs u32+u32 n=2^%d: mean %.3f ms (best %.3f) = %.1f Gkeys/s  temp %.1f MB\n", lg, sum / reps, best,
           n / (sum / reps) / 1e6, tb / 1e6);
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(tmp);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
