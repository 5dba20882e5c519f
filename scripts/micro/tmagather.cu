// TMA gather4 rate: can the TMA unit add random-gather throughput on top of
// the LSU path (~0.9 L2 requests/clk/SM, l2gather.cu)?  x (8 MB f64) is viewed
// as a 2-D tensor of 16-byte rows {2 doubles}; one
// cp.async.bulk.tensor.2d...tile::gather4 fetches the 4 rows holding
// x[c0..c3].  Each warp's lane 0 issues GB gather4s per batch into its smem
// slot and waits on its mbarrier.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tmagather tmagather.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__host__ __device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int GB, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) tma_gather(const __grid_constant__ CUtensorMap map, const int* __restrict__ idx,
                                                         uint32_t n, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* slot = sm + warp * GB * 128;  // gather4 destinations 128-B aligned
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint32_t per = GB * 4;
  const uint32_t gw = gridDim.x * WARPS, w = blockIdx.x * WARPS + warp;
  double acc = 0.0;
  uint32_t phase = 0;
  for (uint32_t base = w * per; base < n; base += gw * per) {
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(GB * 64) : "memory");
      for (int g = 0; g < GB; ++g) {
        const uint32_t k = base + g * 4;
        const int r0 = idx[k] >> 1, r1 = idx[k + 1] >> 1, r2 = idx[k + 2] >> 1, r3 = idx[k + 3] >> 1;
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(slot + g * 128);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
            : "memory");
      }
    }
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(b),
                 "r"(phase) : "memory");
    phase ^= 1u;
    for (int g = lane; g < GB * 8; g += 32) acc += reinterpret_cast<const double*>(slot)[(g >> 3) * 16 + (g & 7)];
    __syncwarp();
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  const uint32_t nx = 1u << 20, n = 1u << 24;
  double *x, *o;
  int* idx;
  cudaMalloc(&x, (size_t)nx * 8);
  cudaMalloc(&o, 64);
  cudaMalloc(&idx, (size_t)n * 4);
  int* h = (int*)malloc((size_t)n * 4);
  for (uint32_t i = 0; i < n; ++i) h[i] = (int)(hash(i * 3 + 7) % nx);
  cudaMemcpy(idx, h, (size_t)n * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  const cuuint64_t dims[2] = {2, nx / 2};
  const cuuint64_t strides[1] = {16};
  const cuuint32_t box[2] = {2, 1};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
#define RUN(GB, WARPS, CPS)                                                                                  \
  {                                                                                                          \
    const size_t smem = (size_t)WARPS * GB * 128;                                                            \
    cudaFuncSetAttribute(tma_gather<GB, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    tma_gather<GB, WARPS><<<sms * CPS, 32 * WARPS, smem>>>(map, idx, n, o);                                  \
    cudaEventRecord(e0);                                                                                     \
    for (int it = 0; it < 5; ++it) tma_gather<GB, WARPS><<<sms * CPS, 32 * WARPS, smem>>>(map, idx, n, o);   \
    cudaEventRecord(e1);                                                                                     \
    cudaError_t err = cudaEventSynchronize(e1);                                                              \
    float ms;                                                                                                \
    cudaEventElapsedTime(&ms, e0, e1);                                                                       \
    ms /= 5;                                                                                                 \
    printf("gather4 batch %3d warps %2d ctas/SM %d: %8.2f us  %6.2f gathers/clk/SM  %s\n", GB, WARPS, CPS,  \
           ms * 1e3, n / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(err));                             \
    if (err != cudaSuccess) return 1;                                                                        \
  }
  RUN(8, 4, 4) RUN(16, 4, 4) RUN(32, 4, 4) RUN(32, 8, 4) RUN(64, 8, 2) RUN(128, 4, 4)
  return 0;
}
