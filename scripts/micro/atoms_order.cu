// Does a warp's shared-memory atomicAdd(&cnt[d], 1) return old values in
// LANE ORDER among lanes hitting the same counter (i.e. a stable rank)?
// Random 8-bit digits per lane, many rows; each lane's returned value is
// compared with the stable rank (previous count + lower lanes with the same
// digit).  Also prints the SASS-level instruction the compiler picked.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o atoms_order atoms_order.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int MOD>
__global__ void check(unsigned long long* bad, int rows) {
  __shared__ uint32_t cnt[8][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = lane; i < 256; i += 32) cnt[warp][i] = 0;
  __syncwarp();
  uint32_t ref = 0;  // lane-local copy of the counters is too big; recompute from ballots
  unsigned long long errs = 0;
  for (int r = 0; r < rows; ++r) {
    const uint32_t d = hash((blockIdx.x * 8 + warp) * 1000003u + r * 97u + lane) % MOD;
    // stable rank: counter value before this row + lower lanes with the same digit
    const uint32_t before = cnt[warp][d];
    __syncwarp();
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t below = __popc(peers & ((1u << lane) - 1));
    const uint32_t got = atomicAdd(&cnt[warp][d], 1u);
    __syncwarp();
    if (got != before + below) ++errs;
  }
  (void)ref;
  if (errs) atomicAdd(bad, errs);
}

int main() {
  unsigned long long* bad;
  cudaMalloc(&bad, 8);
  for (int mod : {2, 7, 32, 256}) {
    cudaMemset(bad, 0, 8);
    if (mod == 2) check<2><<<1024, 256>>>(bad, 2000);
    if (mod == 7) check<7><<<1024, 256>>>(bad, 2000);
    if (mod == 32) check<32><<<1024, 256>>>(bad, 2000);
    if (mod == 256) check<256><<<1024, 256>>>(bad, 2000);
    unsigned long long h = 0;
    cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
    printf("digits mod %3d: %llu of %llu lane results differ from the stable rank (%s)\n", mod, h,
           1024ull * 256 * 2000, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
