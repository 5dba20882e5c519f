// Host byte-histogram variants (DeviceA share of the histogram): 4 / 8 tables,
// interleaved words, and a 65536-entry byte-pair table folded to 256 bins.
//   g++ -O3 -march=native -o host_hist host_hist.cpp -lpthread && ./host_hist <threads>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <thread>
#include <algorithm>
static inline double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
void h4(const uint8_t* d, size_t n, uint64_t* h) {
  static thread_local uint32_t sub[4][256]; memset(sub, 0, sizeof(sub));
  size_t i = 0;
  for (; i + 8 <= n; i += 8) { uint64_t w; memcpy(&w, d + i, 8);
    ++sub[0][w & 255]; ++sub[1][(w >> 8) & 255]; ++sub[2][(w >> 16) & 255]; ++sub[3][(w >> 24) & 255];
    ++sub[0][(w >> 32) & 255]; ++sub[1][(w >> 40) & 255]; ++sub[2][(w >> 48) & 255]; ++sub[3][w >> 56]; }
  for (; i < n; ++i) ++sub[0][d[i]];
  for (int v = 0; v < 256; ++v) h[v] += (uint64_t)sub[0][v] + sub[1][v] + sub[2][v] + sub[3][v];
}
void h8(const uint8_t* d, size_t n, uint64_t* h) {
  static thread_local uint32_t sub[8][256]; memset(sub, 0, sizeof(sub));
  size_t i = 0;
  for (; i + 16 <= n; i += 16) { uint64_t w, u; memcpy(&w, d + i, 8); memcpy(&u, d + i + 8, 8);
    ++sub[0][w & 255]; ++sub[1][(w >> 8) & 255]; ++sub[2][(w >> 16) & 255]; ++sub[3][(w >> 24) & 255];
    ++sub[4][(w >> 32) & 255]; ++sub[5][(w >> 40) & 255]; ++sub[6][(w >> 48) & 255]; ++sub[7][w >> 56];
    ++sub[0][u & 255]; ++sub[1][(u >> 8) & 255]; ++sub[2][(u >> 16) & 255]; ++sub[3][(u >> 24) & 255];
    ++sub[4][(u >> 32) & 255]; ++sub[5][(u >> 40) & 255]; ++sub[6][(u >> 48) & 255]; ++sub[7][u >> 56]; }
  for (; i < n; ++i) ++sub[0][d[i]];
  for (int v = 0; v < 256; ++v) { uint64_t t = 0; for (int k = 0; k < 8; ++k) t += sub[k][v]; h[v] += t; }
}
void hpair(const uint8_t* d, size_t n, uint64_t* h) {
  static thread_local std::vector<uint32_t> pt(65536); std::fill(pt.begin(), pt.end(), 0);
  size_t i = 0;
  for (; i + 8 <= n; i += 8) { uint64_t w; memcpy(&w, d + i, 8);
    ++pt[w & 0xffff]; ++pt[(w >> 16) & 0xffff]; ++pt[(w >> 32) & 0xffff]; ++pt[w >> 48]; }
  for (; i < n; ++i) ++h[d[i]];
  for (int a = 0; a < 256; ++a) for (int b = 0; b < 256; ++b) { uint32_t c = pt[a * 256 + b]; h[a] += c; h[b] += c; }
}
// 4 tables of uint16-pairs? plus unrolled two words interleaved to break chains
void h4x2(const uint8_t* d, size_t n, uint64_t* h) {
  static thread_local uint32_t sub[4][256]; memset(sub, 0, sizeof(sub));
  size_t i = 0;
  for (; i + 16 <= n; i += 16) { uint64_t w, u; memcpy(&w, d + i, 8); memcpy(&u, d + i + 8, 8);
    ++sub[0][w & 255]; ++sub[1][u & 255]; ++sub[2][(w >> 8) & 255]; ++sub[3][(u >> 8) & 255];
    ++sub[0][(w >> 16) & 255]; ++sub[1][(u >> 16) & 255]; ++sub[2][(w >> 24) & 255]; ++sub[3][(u >> 24) & 255];
    ++sub[0][(w >> 32) & 255]; ++sub[1][(u >> 32) & 255]; ++sub[2][(w >> 40) & 255]; ++sub[3][(u >> 40) & 255];
    ++sub[0][(w >> 48) & 255]; ++sub[1][(u >> 48) & 255]; ++sub[2][w >> 56]; ++sub[3][u >> 56]; }
  for (; i < n; ++i) ++sub[0][d[i]];
  for (int v = 0; v < 256; ++v) h[v] += (uint64_t)sub[0][v] + sub[1][v] + sub[2][v] + sub[3][v];
}
// 8 tables, four words per iteration (more independent increments in flight)
void h8x4(const uint8_t* d, size_t n, uint64_t* h) {
  static thread_local uint32_t sub[8][256]; memset(sub, 0, sizeof(sub));
  size_t i = 0;
#define B8(w) ++sub[0][w & 255]; ++sub[1][(w >> 8) & 255]; ++sub[2][(w >> 16) & 255]; ++sub[3][(w >> 24) & 255]; \
    ++sub[4][(w >> 32) & 255]; ++sub[5][(w >> 40) & 255]; ++sub[6][(w >> 48) & 255]; ++sub[7][w >> 56];
  for (; i + 32 <= n; i += 32) { uint64_t a, b, c, e; memcpy(&a, d + i, 8); memcpy(&b, d + i + 8, 8);
    memcpy(&c, d + i + 16, 8); memcpy(&e, d + i + 24, 8); B8(a) B8(b) B8(c) B8(e) }
#undef B8
  for (; i < n; ++i) ++sub[0][d[i]];
  for (int v = 0; v < 256; ++v) { uint64_t t = 0; for (int k = 0; k < 8; ++k) t += sub[k][v]; h[v] += t; }
}
// 16 tables of uint16 counters (flushed every 2^16 - 1 iterations per table): half the table bytes
void h16s(const uint8_t* d, size_t n, uint64_t* h) {
  static thread_local uint16_t sub[16][256];
  size_t i = 0;
  while (i + 16 <= n) {
    memset(sub, 0, sizeof(sub));
    const size_t e = std::min(n, i + (size_t)65535 * 16);
    for (; i + 16 <= e; i += 16) { uint64_t w, u; memcpy(&w, d + i, 8); memcpy(&u, d + i + 8, 8);
      ++sub[0][w & 255]; ++sub[1][(w >> 8) & 255]; ++sub[2][(w >> 16) & 255]; ++sub[3][(w >> 24) & 255];
      ++sub[4][(w >> 32) & 255]; ++sub[5][(w >> 40) & 255]; ++sub[6][(w >> 48) & 255]; ++sub[7][w >> 56];
      ++sub[8][u & 255]; ++sub[9][(u >> 8) & 255]; ++sub[10][(u >> 16) & 255]; ++sub[11][(u >> 24) & 255];
      ++sub[12][(u >> 32) & 255]; ++sub[13][(u >> 40) & 255]; ++sub[14][(u >> 48) & 255]; ++sub[15][u >> 56]; }
    for (int v = 0; v < 256; ++v) { uint64_t t = 0; for (int k = 0; k < 16; ++k) t += sub[k][v]; h[v] += t; }
  }
  for (; i < n; ++i) ++h[d[i]];
}
int main(int argc, char** argv) {
  const size_t n = argc > 2 ? (size_t)atoll(argv[2]) : (size_t)1 << 28;
  std::vector<uint8_t> d(n);
  uint64_t x = 1; for (size_t i = 0; i < n; ++i) { x = x * 6364136223846793005ull + 1442695040888963407ull; d[i] = (uint8_t)(x >> 56); }
  int T = argc > 1 ? atoi(argv[1]) : 1;
  auto run = [&](const char* name, void (*f)(const uint8_t*, size_t, uint64_t*)) {
    std::vector<std::vector<uint64_t>> hs(T, std::vector<uint64_t>(256));
    for (int rep = 0; rep < 2; ++rep) {
      for (auto& hh : hs) std::fill(hh.begin(), hh.end(), 0);
      double t0 = now();
      std::vector<std::thread> th;
      for (int k = 0; k < T; ++k) th.emplace_back([&, k] { f(d.data() + n * k / T, n * (k + 1) / T - n * k / T, hs[k].data()); });
      for (auto& t : th) t.join();
      double dt = now() - t0;
      uint64_t tot = 0; for (auto& hh : hs) for (auto v : hh) tot += v;
      if (rep) printf("%-6s T=%d %.2f GB/s (tot ok %d)\n", name, T, n / dt / 1e9, (int)(tot == n));
    }
  };
  run("h8", h8); run("h8x4", h8x4); run("h16s", h16s); run("h4x2", h4x2);
}
