// D2H of 1-32 MB into cudaHostAlloc'd memory: non-blocking stream vs the
// legacy default stream, cudaMalloc vs cudaMallocAsync (mem pool) sources,
// and right after a kernel wrote the source.
//   nvcc -O3 -o d2h_small d2h_small.cu
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
__global__ void touch(char* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 1;
}
int main() {
  char *d, *h;
  cudaMalloc(&d, 64 << 20);
  cudaMemset(d, 1, 64 << 20);
  cudaHostAlloc((void**)&h, 32 << 20, cudaHostAllocDefault);
  cudaStream_t nb;
  cudaStreamCreateWithFlags(&nb, cudaStreamNonBlocking);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  auto run = [&](const char* name, char* src, cudaStream_t s, bool kernel_first) {
    double best = 1e9, sum = 0;
    for (int r = 0; r < 10; ++r) {
      if (kernel_first) { touch<<<592, 256, 0, s>>>(src, 8 << 20); cudaStreamSynchronize(s); }
      double t0 = now();
      cudaMemcpyAsync(h, src, 8 << 20, cudaMemcpyDeviceToHost, s);
      cudaEventRecord(ev, s);
      cudaEventSynchronize(ev);
      double dt = now() - t0;
      best = std::min(best, dt);
      sum += dt;
    }
    printf("%-44s best %.3f ms  mean %.3f ms\n", name, best * 1e3, sum / 10 * 1e3);
  };
  run("cudaMalloc src, non-blocking stream", d, nb, false);
  run("cudaMalloc src, legacy stream 0", d, 0, false);
  run("cudaMalloc src, stream 0, after a kernel", d, 0, true);
  for (int k = 0; k < 3; ++k) {
    char* a;
    cudaMallocAsync((void**)&a, 8 << 20, 0);
    touch<<<592, 256>>>(a, 8 << 20);
    cudaStreamSynchronize(0);
    run("cudaMallocAsync src, stream 0, fresh", a, 0, false);
    cudaFreeAsync(a, 0);
  }
  return 0;
}
