// Streaming rate of cp.async.bulk (TMA 1-D bulk copies) vs chunk size and
// copies in flight, against plain 16-byte LDG: can per-warp bulk copies of a
// few KB feed an HBM-bound kernel on B200?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bulkstream bulkstream.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk(void* smem, const void* g, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)), "l"(g), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

// each warp: lane 0 keeps S chunks of CH bytes in flight; all lanes touch one word per chunk
template <int CH, int S, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) bulk_stream(const char* __restrict__ src, size_t bytes, unsigned* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[WARPS][S];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* buf = sm + (size_t)warp * S * CH;
  uint64_t* bar = bars[warp];
  const size_t nch = bytes / CH;
  const size_t gw = (size_t)gridDim.x * WARPS, w = (size_t)blockIdx.x * WARPS + warp;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < S; ++s) {
      const size_t c = w + s * gw;
      if (c < nch) {
        mbar_expect_tx(&bar[s], CH);
        bulk(buf + s * CH, src + c * CH, CH, &bar[s]);
      }
    }
  }
  __syncwarp();
  unsigned acc = 0;
  int s = 0;
  uint32_t ph = 0;
  for (size_t c = w; c < nch; c += gw) {
    mbar_wait(&bar[s], ph);
    acc += ((const unsigned*)(buf + s * CH))[lane];
    __syncwarp();
    const size_t nc = c + S * gw;
    if (lane == 0 && nc < nch) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bar[s], CH);
      bulk(buf + s * CH, src + nc * CH, CH, &bar[s]);
    }
    if (++s == S) { s = 0; ph ^= 1; }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void ldg_stream(const uint4* __restrict__ src, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
    acc += v.x ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const size_t bytes = 1ull << 30;
  char* src;
  unsigned* out;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaMalloc(&out, 64);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  ldg_stream<<<sms * 4, 512>>>((const uint4*)src, bytes / 16, out);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) ldg_stream<<<sms * 4, 512>>>((const uint4*)src, bytes / 16, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("LDG.128 grid-stride: %.0f GB/s\n", 5.0 * bytes / (ms * 1e-3) / 1e9);
#define RUN(CH, S, W, CPS)                                                                             \
  {                                                                                                    \
    const size_t sm = (size_t)W * S * CH;                                                              \
    cudaFuncSetAttribute(bulk_stream<CH, S, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    bulk_stream<CH, S, W><<<sms * CPS, 32 * W, sm>>>(src, bytes, out);                                 \
    cudaEventRecord(e0);                                                                               \
    for (int r = 0; r < 5; ++r) bulk_stream<CH, S, W><<<sms * CPS, 32 * W, sm>>>(src, bytes, out);     \
    cudaEventRecord(e1);                                                                               \
    cudaEventSynchronize(e1);                                                                          \
    cudaEventElapsedTime(&ms, e0, e1);                                                                 \
    printf("bulk chunk %6d B  stages %d  warps/CTA %2d  CTAs/SM %d  (%3zu KB in flight/SM): %6.0f GB/s  %s\n", CH, S, W, CPS, \
           sm * CPS / 1024, 5.0 * bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));    \
  }
  RUN(1024, 3, 4, 4) RUN(2048, 3, 4, 4) RUN(3072, 3, 4, 4) RUN(4096, 3, 4, 4) RUN(8192, 3, 4, 2)
  RUN(1024, 4, 8, 2) RUN(2048, 4, 8, 2) RUN(4096, 4, 8, 1) RUN(8192, 4, 4, 1) RUN(16384, 4, 2, 1)
  RUN(32768, 4, 1, 1) RUN(16384, 6, 1, 2) RUN(2048, 8, 8, 1) RUN(1024, 8, 16, 1) RUN(512, 8, 16, 2)
  return 0;
}
