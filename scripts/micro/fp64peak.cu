// Peak fp64 instruction rate on B200 (DADD / DMUL / DFMA, many independent
// chains per thread): the denominator of the compute roofline of the
// bit-exact fp64 filters (bilateral: 2 DMUL + 2 DADD per tap, conv: 1 + 1).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64peak fp64peak.cu
#include <cuda_runtime.h>
#include <cstdio>

template <int OP, int C>
__global__ void __launch_bounds__(256) fp64_loop(double* out, int iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (OP == 0) x[c] = __dadd_rn(x[c], a);
      else if (OP == 1) x[c] = __dmul_rn(x[c], b);
      else x[c] = __fma_rn(x[c], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o;
  cudaMalloc(&o, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
#define RUN(OP, C, CPS)                                                                           \
  {                                                                                               \
    const int grid = sms * CPS;                                                                   \
    fp64_loop<OP, C><<<grid, 256>>>(o, iters, 1e-9, 0.999999);                                    \
    cudaEventRecord(e0);                                                                          \
    fp64_loop<OP, C><<<grid, 256>>>(o, iters, 1e-9, 0.999999);                                    \
    cudaEventRecord(e1);                                                                          \
    cudaEventSynchronize(e1);                                                                     \
    float ms;                                                                                     \
    cudaEventElapsedTime(&ms, e0, e1);                                                            \
    const double ops = (double)grid * 256 * iters * C;                                            \
    printf("%s chains %2d ctas/SM %d: %7.2f T instr/s  (%.1f lanes/clk/SM at 1.965 GHz)\n",      \
           OP == 0 ? "DADD" : OP == 1 ? "DMUL" : "DFMA", C, CPS, ops / (ms * 1e-3) / 1e12,         \
           ops / (ms * 1e-3) / sms / 1.965e9);                                                    \
  }
  RUN(0, 8, 4) RUN(0, 16, 4) RUN(0, 8, 8) RUN(1, 8, 4) RUN(1, 16, 4) RUN(2, 8, 4) RUN(2, 16, 4) RUN(2, 8, 8)
  RUN(0, 8, 2) RUN(0, 16, 2) RUN(0, 8, 1) RUN(0, 16, 1) RUN(0, 4, 2) RUN(0, 4, 3)
  return 0;
}
