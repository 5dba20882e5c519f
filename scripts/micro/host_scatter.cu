// Host un-permute y[perm[i]] = t[i] (SpMV's original-order result, 10^6 rows)
// into different kinds of destination memory: cudaHostAlloc'd (pinned, 4 KB
// pages), malloc + THP, and with destinations pre-sorted — is the scatter
// bound by TLB misses on pinned memory?
//   nvcc -O3 -o host_scatter host_scatter.cu -lpthread
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

double scatter(double* y, const int64_t* perm, const double* t, int64_t n, int T) {
  double best = 1e9;
  for (int rep = 0; rep < 7; ++rep) {
    double t0 = now();
    std::vector<std::thread> th;
    for (int k = 0; k < T; ++k)
      th.emplace_back([=] {
        for (int64_t i = n * k / T, e = n * (k + 1) / T; i < e; ++i) y[perm[i]] = t[i];
      });
    for (auto& x : th) x.join();
    best = std::min(best, now() - t0);
  }
  return best * 1e3;
}

int main() {
  const int64_t n = 1000000;
  std::vector<int64_t> perm(n), sorted(n);
  std::iota(perm.begin(), perm.end(), 0);
  std::shuffle(perm.begin(), perm.end(), std::mt19937_64(1));
  std::vector<double> t(n, 1.0);
  double* pinned;
  cudaHostAlloc((void**)&pinned, n * 8, cudaHostAllocDefault);
  double* thp = (double*)aligned_alloc(2 << 20, ((n * 8 + (2 << 20) - 1) / (2 << 20)) * (2 << 20));
  madvise(thp, n * 8, MADV_HUGEPAGE);
  for (int64_t i = 0; i < n; ++i) pinned[i] = thp[i] = 0.0;
  std::iota(sorted.begin(), sorted.end(), 0);
  for (int T : {1, 4, 16}) {
    printf("T=%2d  pinned random %.3f ms  THP random %.3f ms  pinned sorted %.3f ms\n", T,
           scatter(pinned, perm.data(), t.data(), n, T), scatter(thp, perm.data(), t.data(), n, T),
           scatter(pinned, sorted.data(), t.data(), n, T));
  }
  return 0;
}
