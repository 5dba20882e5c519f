// Minimal 2-D TMA tile load check (uint8 image, box W x H) with the encoder
// obtained through cudaGetDriverEntryPoint.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__global__ void k(const __grid_constant__ CUtensorMap map, uint8_t* out, int bw, int bh, int x, int y) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bw * bh) : "memory");
    uint32_t d = (uint32_t)__cvta_generic_to_shared(sm);
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(d), "l"(reinterpret_cast<uint64_t>(&map)), "r"(x), "r"(y), "r"(b) : "memory");
  }
  __syncthreads();
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b) : "memory");
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
  const int W = 1024, H = 1024;
  uint8_t *img, *out;
  cudaMalloc(&img, W * H);
  cudaMalloc(&out, 1 << 16);
  uint8_t* h = new uint8_t[W * H];
  for (int i = 0; i < W * H; ++i) h[i] = (uint8_t)(i * 7 + i / W);
  cudaMemcpy(img, h, W * H, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  printf("entry point: %s q=%d fn=%p\n", cudaGetErrorString(e), (int)q, fn);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  int shapes[][2] = {{80, 42}, {64, 32}, {128, 16}};
  const int X0 = argc > 1 ? atoi(argv[1]) : 48, Y0 = argc > 2 ? atoi(argv[2]) : 100;
  for (auto& sh : shapes) {
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
    const cuuint64_t strides[1] = {(cuuint64_t)W};
    const cuuint32_t box[2] = {(cuuint32_t)sh[0], (cuuint32_t)sh[1]};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, img, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 128, 16384>>>(map, out, sh[0], sh[1], X0, Y0);
    cudaError_t ke = cudaDeviceSynchronize();
    uint8_t got[16384];
    int bad = -1;
    if (ke == cudaSuccess) {
      cudaMemcpy(got, out, sh[0] * sh[1], cudaMemcpyDeviceToHost);
      bad = 0;
      for (int yy = 0; yy < sh[1]; ++yy)
        for (int xx = 0; xx < sh[0]; ++xx) bad += got[yy * sh[0] + xx] != h[(Y0 + yy) * W + X0 + xx];
    }
    printf("box %dx%d: encode %d, kernel %s, mismatches %d\n", sh[0], sh[1], (int)r, cudaGetErrorString(ke), bad);
    if (ke != cudaSuccess) return 1;
  }
  return 0;
}
