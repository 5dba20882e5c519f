// Random 8-byte gathers from distributed shared memory: can a thread-block
// cluster hold a slice of SpMV's x vector in its CTAs' shared memory and
// serve part of the gathers without the L2 request path (~0.9 requests/clk/SM,
// l2gather.cu)?  Each CTA of a CL-CTA cluster holds SLOT doubles; every
// thread issues random loads: a fraction P/16 through ld.shared::cluster to
// the owning CTA, the rest as L2-resident global gathers from an 8 MB array.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dsmem_gather dsmem_gather.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int U>
__global__ void __launch_bounds__(256) dsmem_gather(const double* __restrict__ x, uint32_t nx_mask, uint32_t slot,
                                                    uint32_t iters, int p16, double* out) {
  extern __shared__ double xs[];
  cg::cluster_group cl = cg::this_cluster();
  for (uint32_t i = threadIdx.x; i < slot; i += blockDim.x) xs[i] = (double)i;
  cl.sync();
  const uint32_t csize = cl.num_blocks();
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (uint32_t it = 0; it < iters; ++it) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t h = hash(tid * 7919u + it * 131u + u);
      if ((int)(h & 15) < p16) {
        const uint32_t r = (h >> 4) % csize, off = (h >> 12) % slot;
        const double* remote = cl.map_shared_rank(xs, r);
        v[u] = remote[off];
      } else {
        v[u] = __ldg(x + ((h >> 4) & nx_mask));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  cl.sync();  // no CTA may exit while others read its shared memory
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const uint32_t nx = 1u << 20;
  double *x, *o;
  cudaMalloc(&x, (size_t)nx * 8);
  cudaMalloc(&o, 64);
  cudaMemset(x, 0, (size_t)nx * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto kern = dsmem_gather<8>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cl : {1, 2, 4, 8, 16}) {
    for (int kb : {64, 100, 180}) {
      const size_t smem = (size_t)kb * 1024;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int p16 : {0, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        const int occ = kb <= 64 ? 3 : kb <= 100 ? 2 : 1;
        const int grid = (sms * occ * 4 + cl - 1) / cl * cl;  // ~4 waves
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const uint32_t iters = 128, slot = (uint32_t)(smem / 8);
        cudaError_t err = cudaLaunchKernelEx(&cfg, kern, (const double*)x, nx - 1, slot, iters, p16, o);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) err = cudaLaunchKernelEx(&cfg, kern, (const double*)x, nx - 1, slot, iters, p16, o);
        cudaEventRecord(e1);
        cudaError_t e2 = cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 5;
        const double loads = (double)grid * 256 * iters * 8;
        printf("cluster %2d smem %3d KB dsmem %5.1f%%: %8.2f us  %5.2f loads/clk/SM  (%s %s)\n", cl, kb,
               100.0 * p16 / 16, ms * 1e3, loads / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(err),
               cudaGetErrorString(e2));
      }
    }
  }
  return 0;
}
