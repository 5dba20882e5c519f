// Do the LSU gather path (~0.9 L2 requests/clk/SM, l2gather.cu) and TMA
// gather4 (~0.34, tmagather.cu) ADD UP when they run at the same time on the
// same SMs?  One kernel: LW warps per CTA gather x[idx[k]] with LDG for
// k < nL, one warp per CTA issues gather4s for k >= nL.  If the two paths
// share the SM's L2 request port, the mixed runs are no faster than LSU-only.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_mix gather_mix.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

static uint32_t hash_h(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

constexpr int G4L = 2;  // gather4s per lane per batch

template <int LW, int TW>
__global__ void __launch_bounds__(32 * (LW + TW)) mix(const __grid_constant__ CUtensorMap map, const double* __restrict__ x,
                                                      const int* __restrict__ idx, uint32_t nL, uint32_t n, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[TW > 0 ? TW * 2 : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0.0;
  if (warp < LW) {
    const uint32_t stride = gridDim.x * LW * 32 * 4;
    for (uint32_t base = (blockIdx.x * LW + warp) * 128 + lane; base < nL; base += stride) {
      int j[4];
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) j[u] = base + u * 32 < nL ? __ldg(idx + base + u * 32) : 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(x + j[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u];
    }
  } else if (TW > 0) {
    // every lane of a TMA warp issues G4L gather4s per batch (lane 0 posts
    // the batch's expect_tx first), double-buffered per warp
    constexpr int BATCH = 32 * G4L;  // gather4s per warp batch
    const int tw = warp - LW;
    unsigned char* slot = sm + tw * 2 * BATCH * 128;
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bars[tw * 2]);
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t per = BATCH * 4;
    const uint32_t gw = gridDim.x * TW, w = blockIdx.x * TW + tw;
    uint32_t ph[2] = {0, 0};
    int s = 0;
    auto issue = [&](uint32_t base, int st) {
      const uint32_t b = b0 + 8 * st;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(BATCH * 64) : "memory");
      __syncwarp();
      int4 q[G4L];
#pragma unroll
      for (int g = 0; g < G4L; ++g) q[g] = __ldg(reinterpret_cast<const int4*>(idx + base) + g * 32 + lane);
#pragma unroll
      for (int g = 0; g < G4L; ++g) {
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(slot + (st * BATCH + g * 32 + lane) * 128);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(q[g].x >> 1), "r"(q[g].y >> 1), "r"(q[g].z >> 1),
            "r"(q[g].w >> 1), "r"(b)
            : "memory");
      }
    };
    uint32_t base = nL + w * per;
    if (base + per <= n) issue(base, 0);
    for (; base + per <= n; base += gw * per) {
      const uint32_t nxt = base + gw * per;
      if (nxt + per <= n) issue(nxt, s ^ 1);
      const uint32_t b = b0 + 8 * s;
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(b),
                   "r"(ph[s]) : "memory");
      ph[s] ^= 1u;
      const double* sd = reinterpret_cast<const double*>(slot + s * BATCH * 128);
#pragma unroll
      for (int g = 0; g < G4L; ++g) acc += sd[(g * 32 + lane) * 16] + sd[(g * 32 + lane) * 16 + 6];
      __syncwarp();
      s ^= 1;
    }
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
  cudaMemset(x, 0, (size_t)nx * 8);
  int* h = (int*)malloc((size_t)n * 4);
  for (uint32_t i = 0; i < n; ++i) h[i] = (int)(hash_h(i * 3 + 7) % nx);
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
  encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
#define RUN(LW, TW, CPS, FRAC)                                                                                   \
  {                                                                                                              \
    uint32_t nL = (uint32_t)((1.0 - (FRAC)) * n) & ~1023u;                                                          \
    const size_t smem = (size_t)(TW > 0 ? TW : 1) * 2 * 32 * G4L * 128;                                                \
    cudaFuncSetAttribute(mix<LW, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                   \
    cudaFuncSetAttribute(mix<LW, TW>, cudaFuncAttributePreferredSharedMemoryCarveout, 25);                       \
    mix<LW, TW><<<sms * CPS, 32 * (LW + TW), smem>>>(map, x, idx, nL, n, o);                                     \
    cudaEventRecord(e0);                                                                                         \
    for (int it = 0; it < 10; ++it) mix<LW, TW><<<sms * CPS, 32 * (LW + TW), smem>>>(map, x, idx, nL, n, o);      \
    cudaEventRecord(e1);                                                                                         \
    cudaError_t err = cudaEventSynchronize(e1);                                                                  \
    float ms;                                                                                                    \
    cudaEventElapsedTime(&ms, e0, e1);                                                                           \
    ms /= 10;                                                                                                    \
    printf("LSU warps %2d TMA warps %d ctas/SM %d tma share %.2f: %8.2f us  %5.2f gathers/clk/SM  %s\n", LW, TW, \
           CPS, (double)(FRAC), ms * 1e3, n / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(err));                       \
    if (err != cudaSuccess) return 1;                                                                            \
  }
  RUN(16, 0, 2, 0.0)
  RUN(16, 4, 2, 0.0)
  RUN(16, 4, 2, 0.15) RUN(16, 4, 2, 0.20) RUN(16, 4, 2, 0.25) RUN(16, 4, 2, 0.30)
  RUN(8, 4, 2, 0.25) RUN(8, 8, 2, 0.25) RUN(16, 8, 2, 0.25)
  RUN(1, 4, 2, 0.99) RUN(1, 8, 2, 0.99) RUN(1, 4, 4, 0.99)
  return 0;
}
