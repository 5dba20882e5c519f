// Host memory rates for the list-ranking transfer idea (g++ -O3 -march=native -pthread host_narrow.cpp):
// int64 -> int32 narrowing of 2^28 values, int32 -> int64 widening, and memcpy of 1 GiB,
// with T threads over contiguous slices (arrays touched first).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

template <typename F>
double timed(int T, F&& f) {
  auto a = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int k = 0; k < T; ++k) th.emplace_back(f, k);
  for (auto& t : th) t.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
}

int main() {
  const int64_t n = 1ll << 28;
  int64_t* w = (int64_t*)aligned_alloc(4096, n * 8);
  int32_t* s = (int32_t*)aligned_alloc(4096, n * 4);
  char* c = (char*)aligned_alloc(4096, n * 4);
  for (int64_t i = 0; i < n; ++i) w[i] = (i * 2654435761ll) & 0x7fffffff;
  memset(s, 1, n * 4);
  memset(c, 1, n * 4);
  for (int T : {1, 4, 8, 15, 16}) {
    double best[3] = {1e9, 1e9, 1e9};
    for (int r = 0; r < 3; ++r) {
      best[0] = std::min(best[0], timed(T, [&](int k) {
        const int64_t a = n * k / T, b = n * (k + 1) / T;
        bool bad = false;
        for (int64_t i = a; i < b; ++i) {
          const int64_t v = w[i];
          bad |= v != (int32_t)v;
          s[i] = (int32_t)v;
        }
        if (bad) abort();
      }));
      best[1] = std::min(best[1], timed(T, [&](int k) {
        const int64_t a = n * k / T, b = n * (k + 1) / T;
        for (int64_t i = a; i < b; ++i) w[i] = s[i];
      }));
      best[2] = std::min(best[2], timed(T, [&](int k) {
        const int64_t a = (n * 4) * k / T, b = (n * 4) * (k + 1) / T;
        memcpy(c + a, reinterpret_cast<char*>(s) + a, b - a);
      }));
    }
    printf("T=%2d  narrow 2 GiB->1 GiB %6.1f ms   widen 1 GiB->2 GiB %6.1f ms   memcpy 1 GiB %6.1f ms\n", T,
           best[0] * 1e3, best[1] * 1e3, best[2] * 1e3);
  }
}
