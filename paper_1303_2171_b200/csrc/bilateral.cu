// bilateral.cu — LUT bilateral filter on row strips (replaces bilateral_rows /
// BilateralApplyWorkload.run_part, reference kernels_regular.py:461-511).
//
// Arithmetic is the reference's, bit for bit: for every tap (dy, dx) in
// row-major order, w = spatial[tap] * range[|nb - c|] (rounded fp64 multiply),
// num += w * nb, den += w (rounded, no FMA), out = num / den (IEEE division).
// Clamp-to-edge borders.  Output fp64 (the reference's dtype) or fp32.
//
// Layout: one CTA = a TILE_H x TILE_W output tile;
// the clamped (TILE_H+2R) x (TILE_W+2R) input halo tile is staged in shared
// memory as int32; the 256-entry range table is stored LANE-STRIPED
// (entry e of lane l at [e][l]) so the 16 lanes of a half-warp read 16
// distinct 8-byte bank pairs for any intensity differences — conflict-free
// lookups; each thread owns PX horizontally adjacent output pixels and keeps
// one input row segment (PX+2R values, converted to fp64 once) in registers
// while it sweeps the 2R+1 taps of that row, so shared-memory traffic per tap
// is one range-table load.  The bound is fp64 issue (2 DMUL + 2 DADD per tap).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "common.cuh"

namespace hb {
namespace {

constexpr int kTileH = 32;
constexpr int kTileW = 64;
constexpr int kPx = 8;                        // pixels per thread (one row segment)
constexpr int kThreads = kTileH * kTileW / kPx;  // 256
constexpr int kMaxR = 8;

template <int R, typename OUT, int STRIPE = 32, int MINB = 2>
__global__ void __launch_bounds__(kThreads, MINB)
    bilateral_tile_kernel(const uint8_t* __restrict__ img, int H, int W, int row0, int row1,
                          const double* __restrict__ spatial, const double* __restrict__ range,
                          OUT* __restrict__ out) {
  constexpr int S = 2 * R + 1;
  constexpr int TH = kTileH + 2 * R, TW = kTileW + 2 * R;
  extern __shared__ __align__(16) unsigned char smem[];
  // range table striped over STRIPE lanes: entry e of lane l at [e][l % STRIPE];
  // 8-byte loads are served per half-warp, so 16 stripes are already
  // conflict-free and halve the table (32 KB)
  constexpr int SH = STRIPE == 32 ? 5 : 4;
  double* rng = reinterpret_cast<double*>(smem);            // [256][STRIPE]
  double* sp = rng + 256 * STRIPE;                          // [S*S]
  int* tile = reinterpret_cast<int*>(sp + S * S);           // [TH][TW]

  const int tid = threadIdx.x;
  const int lane = tid & (STRIPE - 1);
  const int y0 = row0 + blockIdx.y * kTileH;  // first output row of the tile
  const int x0 = blockIdx.x * kTileW;

  for (int i = tid; i < 256 * STRIPE; i += kThreads) rng[i] = range[i >> SH];
  for (int i = tid; i < S * S; i += kThreads) sp[i] = spatial[i];
  for (int i = tid; i < TH * TW; i += kThreads) {
    const int ty = i / TW, tx = i - ty * TW;
    const int gy = min(max(y0 - R + ty, 0), H - 1);
    const int gx = min(max(x0 - R + tx, 0), W - 1);
    tile[i] = img[(int64_t)gy * W + gx];
  }
  __syncthreads();

  const int py = tid / (kTileW / kPx);          // output row within the tile
  const int px = (tid % (kTileW / kPx)) * kPx;  // first output column within the tile
  const int gy = y0 + py;
  if (gy >= row1) return;

  int c[kPx];
#pragma unroll
  for (int j = 0; j < kPx; ++j) c[j] = tile[(py + R) * TW + px + j + R];
  double num[kPx], den[kPx];
#pragma unroll
  for (int j = 0; j < kPx; ++j) num[j] = den[j] = 0.0;

  const double* lane_rng = rng + lane;
#pragma unroll 1
  for (int dy = 0; dy < S; ++dy) {
    int nb[kPx + 2 * R];
    double nbd[kPx + 2 * R];
    const int* trow = tile + (py + dy) * TW + px;
#pragma unroll
    for (int k = 0; k < kPx + 2 * R; ++k) {
      nb[k] = trow[k];
      nbd[k] = (double)nb[k];
    }
#pragma unroll
    for (int dx = 0; dx < S; ++dx) {
      const double s = sp[dy * S + dx];
#pragma unroll
      for (int j = 0; j < kPx; ++j) {
        const int d = abs(nb[j + dx] - c[j]);
        const double w = __dmul_rn(s, lane_rng[d << SH]);
        num[j] = __dadd_rn(num[j], __dmul_rn(w, nbd[j + dx]));
        den[j] = __dadd_rn(den[j], w);
      }
    }
  }
  OUT* o = out + (int64_t)(gy - row0) * W + x0 + px;
#pragma unroll
  for (int j = 0; j < kPx; ++j)
    if (x0 + px + j < W) o[j] = (OUT)__ddiv_rn(num[j], den[j]);
}

// Persistent variant (HB_BILAT_CFG=3; measured no faster than one CTA per
// tile, kept for the record): grid = 2 CTAs per SM, each CTA walks
// tiles round-robin.  The lane-striped range table is built once per CTA
// (not once per tile), and the halo of the NEXT tile is loaded into
// registers before the current tile is filtered and written to the other
// shared-memory buffer afterwards, so the global-load latency of the halo
// is hidden behind the fp64 work instead of stalling every tile.
template <int R, typename OUT>
__global__ void __launch_bounds__(kThreads, 2)
    bilateral_persist_kernel(const uint8_t* __restrict__ img, int H, int W, int row0, int row1,
                             const double* __restrict__ spatial, const double* __restrict__ range,
                             OUT* __restrict__ out, int tiles_x, int ntiles) {
  constexpr int S = 2 * R + 1;
  constexpr int TH = kTileH + 2 * R, TW = kTileW + 2 * R;
  constexpr int HALO = TH * TW;
  constexpr int PER = (HALO + kThreads - 1) / kThreads;  // halo pixels per thread
  extern __shared__ __align__(16) unsigned char smem[];
  double* rng = reinterpret_cast<double*>(smem);  // [256][32] lane-striped
  double* sp = rng + 256 * 32;                    // [S*S]
  int* tiles = reinterpret_cast<int*>(sp + S * S);  // [2][TH][TW]
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  for (int i = tid; i < 256 * 32; i += kThreads) rng[i] = range[i >> 5];
  for (int i = tid; i < S * S; i += kThreads) sp[i] = spatial[i];

  int pre[PER];
  auto fetch = [&](int t) {  // halo of tile t into registers (clamped)
    const int y0 = row0 + (t / tiles_x) * kTileH, x0 = (t % tiles_x) * kTileW;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = tid + u * kThreads;
      if (i < HALO) {
        const int ty = i / TW, tx = i - ty * TW;
        const int gy = min(max(y0 - R + ty, 0), H - 1);
        const int gx = min(max(x0 - R + tx, 0), W - 1);
        pre[u] = img[(int64_t)gy * W + gx];
      }
    }
  };
  auto stash = [&](int* buf) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = tid + u * kThreads;
      if (i < HALO) buf[i] = pre[u];
    }
  };
  int t = blockIdx.x;
  if (t >= ntiles) return;
  fetch(t);
  stash(tiles);
  __syncthreads();
  const int py = tid / (kTileW / kPx);
  const int px = (tid % (kTileW / kPx)) * kPx;
  const double* lane_rng = rng + lane;
  for (int b = 0; t < ntiles; t += gridDim.x, b ^= 1) {
    const int tn = t + gridDim.x;
    if (tn < ntiles) fetch(tn);  // in flight while this tile is filtered
    const int* tile = tiles + b * HALO;
    const int y0 = row0 + (t / tiles_x) * kTileH, x0 = (t % tiles_x) * kTileW;
    const int gy = y0 + py;
    if (gy < row1) {
      int c[kPx];
#pragma unroll
      for (int j = 0; j < kPx; ++j) c[j] = tile[(py + R) * TW + px + j + R];
      double num[kPx], den[kPx];
#pragma unroll
      for (int j = 0; j < kPx; ++j) num[j] = den[j] = 0.0;
#pragma unroll 1
      for (int dy = 0; dy < S; ++dy) {
        int nb[kPx + 2 * R];
        double nbd[kPx + 2 * R];
        const int* trow = tile + (py + dy) * TW + px;
#pragma unroll
        for (int k = 0; k < kPx + 2 * R; ++k) {
          nb[k] = trow[k];
          nbd[k] = (double)nb[k];
        }
#pragma unroll
        for (int dx = 0; dx < S; ++dx) {
          const double s = sp[dy * S + dx];
#pragma unroll
          for (int j = 0; j < kPx; ++j) {
            const int d = abs(nb[j + dx] - c[j]);
            const double w = __dmul_rn(s, lane_rng[d << 5]);
            num[j] = __dadd_rn(num[j], __dmul_rn(w, nbd[j + dx]));
            den[j] = __dadd_rn(den[j], w);
          }
        }
      }
      OUT* o = out + (int64_t)(gy - row0) * W + x0 + px;
#pragma unroll
      for (int j = 0; j < kPx; ++j)
        if (x0 + px + j < W) o[j] = (OUT)__ddiv_rn(num[j], den[j]);
    }
    if (tn < ntiles) stash(tiles + (b ^ 1) * HALO);
    __syncthreads();
  }
}

// TMA-staged variant (the default when the image allows a tensor map: row
// pitch a multiple of 16 bytes, 16-byte aligned base): the halo tile of an
// interior CTA — one whose clamped halo lies inside the image — arrives with
// ONE cp.async.bulk.tensor.2d issued by thread 0 (completion on an mbarrier)
// instead of (TH x TW) / 256 clamped byte loads per thread; border CTAs keep
// the clamped loads (TMA zero-fills out-of-range elements, the reference
// clamps).  Range table striped over 16 lanes, 3 CTAs/SM.
template <int R, int NR = 1>
struct TmaTile {
  // the innermost TMA coordinate must be 16-byte aligned (an unaligned start
  // faults: scripts/micro/tma2d.cu), so the box starts 16 columns left of the
  // tile and is 16 + 64 + 16 wide; logical halo column tx sits at tx + OFF
  static constexpr int TILE_H = kTileH * NR;
  static constexpr int TH = TILE_H + 2 * R, TW = kTileW + 2 * R;
  static constexpr int PADX = 16, TWB = kTileW + 2 * PADX, OFF = PADX - R;
  static_assert(R <= PADX, "halo wider than the aligned pad");
  static_assert(TH <= 256, "TMA box height");
};

// NR output rows per thread (tile 32·NR x 64): a loaded tap row segment (and
// its fp64 conversion) serves all NR rows; per pixel the taps stay in
// row-major order, so the result is bit-identical.
//
// VEC (HB_BILAT_CFG=8): a thread's row segment (kPx + 2R bytes at an
// unaligned offset) comes in as a few aligned 8-byte shared loads unpacked
// with shifts instead of one byte load per neighbour — fewer shared-memory
// wavefronts, but measured 2 % slower (26.5 vs 27.0 Gpix/s): the unpacking
// costs more issue slots than the byte loads cost wavefronts.
template <int R, typename OUT, int NR, int MINB, bool SYM = false, bool VEC = false>
__global__ void __launch_bounds__(kThreads, MINB)
    bilateral_tma_kernel(const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ img, int H, int W,
                         int row0, int row1, const double* __restrict__ spatial, const double* __restrict__ range,
                         OUT* __restrict__ out) {
  using T = TmaTile<R, NR>;
  constexpr int S = 2 * R + 1;
  constexpr int TH = T::TH, TW = T::TW, TWB = T::TWB, OFF = T::OFF;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  // SYM: the range table is stored for signed differences -255..255 (511
  // rows, entry 255+e = range[|e|]), so a tap indexes it with nb - c directly
  // — no IABS — at twice the shared memory
  constexpr int NE = SYM ? 511 : 256;
  uint8_t* tile = smem;                                                     // [TH][TWB], 128-B aligned
  double* rng = reinterpret_cast<double*>(smem + ((TH * TWB + 127) / 128) * 128);  // [NE][16]
  double* sp = rng + NE * 16;                                               // [S*S]
  const int tid = threadIdx.x;
  const int lane = tid & 15;
  const int y0 = row0 + blockIdx.y * T::TILE_H;
  const int x0 = blockIdx.x * kTileW;
  const bool interior = x0 - T::PADX >= 0 && x0 - T::PADX + TWB <= W && y0 - R >= 0 && y0 - R + TH <= H;
  if (interior && tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar, TH * TWB);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(tile);
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(d), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0 - T::PADX), "r"(y0 - R), "r"(b) : "memory");
  }
  for (int i = tid; i < NE * 16; i += kThreads) rng[i] = range[SYM ? abs((i >> 4) - 255) : (i >> 4)];
  for (int i = tid; i < S * S; i += kThreads) sp[i] = spatial[i];
  if (!interior) {
    for (int i = tid; i < TH * TW; i += kThreads) {
      const int ty = i / TW, tx = i - ty * TW;
      const int gy = min(max(y0 - R + ty, 0), H - 1);
      const int gx = min(max(x0 - R + tx, 0), W - 1);
      tile[ty * TWB + tx + OFF] = img[(int64_t)gy * W + gx];
    }
  }
  __syncthreads();
  if (interior) mbar_wait(&bar, 0);

  const int py = (tid / (kTileW / kPx)) * NR;
  const int px = (tid % (kTileW / kPx)) * kPx;
  const int gy = y0 + py;
  if (gy >= row1) return;
  int c[NR][kPx];
  double num[NR][kPx], den[NR][kPx];
#pragma unroll
  for (int k = 0; k < NR; ++k)
#pragma unroll
    for (int j = 0; j < kPx; ++j) {
      c[k][j] = tile[(py + k + R) * TWB + px + j + R + OFF];
      num[k][j] = den[k][j] = 0.0;
    }
  const double* lane_rng = rng + lane + (SYM ? 255 * 16 : 0);
  // SYM: per-pixel shared-memory byte address of range[nb - c] is
  // cbase[j] + nb*128 (the table row of difference 0, minus c rows), so a tap
  // costs one 32-bit add + one LDS instead of subtract + multiply-add
  uint32_t cbase[NR][kPx];
  if (SYM) {
    const uint32_t lr = (uint32_t)__cvta_generic_to_shared(lane_rng);
#pragma unroll
    for (int k = 0; k < NR; ++k)
#pragma unroll
      for (int j = 0; j < kPx; ++j) cbase[k][j] = lr - (uint32_t)c[k][j] * 128u;
  }
#pragma unroll 1
  for (int iy = 0; iy < S + NR - 1; ++iy) {
    int nb[kPx + 2 * R];
    double nbd[kPx + 2 * R];
    const uint8_t* trow = tile + (py + iy) * TWB + px + OFF;
    if (VEC) {
      constexpr int LO = OFF & ~7, SH = OFF - LO, NW = (SH + kPx + 2 * R + 7) / 8;
      static_assert((kTileW - kPx) + LO + 8 * NW <= TWB && TWB % 8 == 0 && kPx % 8 == 0, "aligned segment window");
      const uint64_t* wrow = reinterpret_cast<const uint64_t*>(tile + (py + iy) * TWB + px + LO);
      uint64_t wv[NW];
#pragma unroll
      for (int i = 0; i < NW; ++i) wv[i] = wrow[i];
#pragma unroll
      for (int q = 0; q < kPx + 2 * R; ++q) nb[q] = (int)((wv[(SH + q) >> 3] >> (((SH + q) & 7) * 8)) & 255u);
    } else {
#pragma unroll
      for (int q = 0; q < kPx + 2 * R; ++q) nb[q] = trow[q];
    }
#pragma unroll
    for (int q = 0; q < kPx + 2 * R; ++q) {
      nbd[q] = (double)nb[q];
      if (SYM) nb[q] *= 128;  // byte offset of the intensity's table row
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const int dy = iy - k;
      if (dy < 0 || dy >= S) continue;
#pragma unroll
      for (int dx = 0; dx < S; ++dx) {
        const double s = sp[dy * S + dx];
#pragma unroll
        for (int j = 0; j < kPx; ++j) {
          double r;
          if (SYM) {
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(cbase[k][j] + (uint32_t)nb[j + dx]));
          } else {
            r = lane_rng[abs(nb[j + dx] - c[k][j]) * 16];
          }
          const double w = __dmul_rn(s, r);
          num[k][j] = __dadd_rn(num[k][j], __dmul_rn(w, nbd[j + dx]));
          den[k][j] = __dadd_rn(den[k][j], w);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    if (gy + k >= row1) break;
    OUT* o = out + (int64_t)(gy + k - row0) * W + x0 + px;
#pragma unroll
    for (int j = 0; j < kPx; ++j)
      if (x0 + px + j < W) o[j] = (OUT)__ddiv_rn(num[k][j], den[k][j]);
  }
}

// Persistent variant (HB_BILAT_CFG=9): grid = SMs x MINB CTAs loop over the
// tiles, so the 64 KB signed range table and the spatial weights are built
// once per CTA instead of once per tile, and the halo tile of the NEXT tile
// is requested by TMA (second 4 KB buffer, own mbarrier) before the current
// one is filtered.  Same per-pixel arithmetic as bilateral_tma_kernel<SYM>.
template <int R, typename OUT, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    bilateral_tmap_kernel(const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ img, int H, int W,
                          int row0, int row1, const double* __restrict__ spatial,
                          const double* __restrict__ range, OUT* __restrict__ out, int tiles_x, int ntiles) {
  using T = TmaTile<R, 1>;
  constexpr int S = 2 * R + 1;
  constexpr int TH = T::TH, TW = T::TW, TWB = T::TWB, OFF = T::OFF;
  constexpr int TBYTES = ((TH * TWB + 127) / 128) * 128;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[2];
  uint8_t* tiles = smem;                                             // [2][TBYTES]
  double* rng = reinterpret_cast<double*>(smem + 2 * TBYTES);        // [511][16]
  double* sp = rng + 511 * 16;                                       // [S*S]
  const int tid = threadIdx.x;
  const int lane = tid & 15;
  auto origin = [&](int t, int& y0, int& x0) {
    y0 = row0 + (t / tiles_x) * kTileH;
    x0 = (t % tiles_x) * kTileW;
  };
  auto interior = [&](int y0, int x0) {
    return x0 - T::PADX >= 0 && x0 - T::PADX + TWB <= W && y0 - R >= 0 && y0 - R + TH <= H;
  };
  auto request = [&](int t, int b) {  // thread 0: TMA the halo of tile t into buffer b when interior
    int y0, x0;
    origin(t, y0, x0);
    if (!interior(y0, x0)) return;
    fence_proxy_async_smem();
    mbar_expect_tx(&bar[b], TH * TWB);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(tiles + b * TBYTES);
    const uint32_t bb = (uint32_t)__cvta_generic_to_shared(&bar[b]);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(d), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0 - T::PADX), "r"(y0 - R), "r"(bb) : "memory");
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if ((int)blockIdx.x < ntiles) request(blockIdx.x, 0);
  }
  for (int i = tid; i < 511 * 16; i += kThreads) rng[i] = range[abs((i >> 4) - 255)];
  for (int i = tid; i < S * S; i += kThreads) sp[i] = spatial[i];
  __syncthreads();
  const double* lane_rng = rng + lane + 255 * 16;
  const uint32_t lr = (uint32_t)__cvta_generic_to_shared(lane_rng);
  const int py = tid / (kTileW / kPx);
  const int px = (tid % (kTileW / kPx)) * kPx;
  uint32_t ph[2] = {0u, 0u};
  int b = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, b ^= 1) {
    int y0, x0;
    origin(t, y0, x0);
    uint8_t* tile = tiles + b * TBYTES;
    const bool in = interior(y0, x0);
    if (tid == 0 && t + (int)gridDim.x < ntiles) request(t + gridDim.x, b ^ 1);  // next tile's halo
    if (!in) {
      for (int i = tid; i < TH * TW; i += kThreads) {
        const int ty = i / TW, tx = i - ty * TW;
        const int gy = min(max(y0 - R + ty, 0), H - 1);
        const int gx = min(max(x0 - R + tx, 0), W - 1);
        tile[ty * TWB + tx + OFF] = img[(int64_t)gy * W + gx];
      }
      __syncthreads();
    } else {
      mbar_wait(&bar[b], ph[b]);
      ph[b] ^= 1u;
    }
    const int gy = y0 + py;
    if (gy < row1) {
      int c[kPx];
      double num[kPx], den[kPx];
      uint32_t cbase[kPx];
#pragma unroll
      for (int j = 0; j < kPx; ++j) {
        c[j] = tile[(py + R) * TWB + px + j + R + OFF];
        num[j] = den[j] = 0.0;
        cbase[j] = lr - (uint32_t)c[j] * 128u;
      }
#pragma unroll 1
      for (int dy = 0; dy < S; ++dy) {
        int nb[kPx + 2 * R];
        double nbd[kPx + 2 * R];
        const uint8_t* trow = tile + (py + dy) * TWB + px + OFF;
#pragma unroll
        for (int q = 0; q < kPx + 2 * R; ++q) {
          nb[q] = trow[q];
          nbd[q] = (double)nb[q];
          nb[q] *= 128;
        }
#pragma unroll
        for (int dx = 0; dx < S; ++dx) {
          const double sw = sp[dy * S + dx];
#pragma unroll
          for (int j = 0; j < kPx; ++j) {
            double r;
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(cbase[j] + (uint32_t)nb[j + dx]));
            const double w = __dmul_rn(sw, r);
            num[j] = __dadd_rn(num[j], __dmul_rn(w, nbd[j + dx]));
            den[j] = __dadd_rn(den[j], w);
          }
        }
      }
      OUT* o = out + (int64_t)(gy - row0) * W + x0 + px;
#pragma unroll
      for (int j = 0; j < kPx; ++j)
        if (x0 + px + j < W) o[j] = (OUT)__ddiv_rn(num[j], den[j]);
    }
    __syncthreads();  // buffer b is free for the tile after next
  }
}

// host: a 2-D uint8 tensor map over the image (driver entry point through
// the runtime, no libcuda link); false when the layout does not allow one
bool make_image_tmap(CUtensorMap* map, const uint8_t* img, int H, int W, int box_w, int box_h) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode || (W % 16) != 0 || ((uintptr_t)img % 16) != 0 || box_w > 256 || box_h > 256) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
  const cuuint64_t strides[1] = {(cuuint64_t)W};
  const cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(img), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// generic radius (> kMaxR): same arithmetic, neighbours read from global memory.
template <typename OUT>
__global__ void bilateral_generic_kernel(const uint8_t* __restrict__ img, int H, int W, int row0,
                                         int row1, int R, const double* __restrict__ spatial,
                                         const double* __restrict__ range, OUT* __restrict__ out) {
  const int64_t n = (int64_t)(row1 - row0) * W;
  const int S = 2 * R + 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int y = row0 + (int)(i / W), x = (int)(i % W);
    const int c = img[(int64_t)y * W + x];
    double num = 0.0, den = 0.0;
    for (int dy = 0; dy < S; ++dy) {
      const int yy = min(max(y + dy - R, 0), H - 1);
      for (int dx = 0; dx < S; ++dx) {
        const int xx = min(max(x + dx - R, 0), W - 1);
        const int v = img[(int64_t)yy * W + xx];
        const double w = __dmul_rn(spatial[dy * S + dx], range[abs(v - c)]);
        num = __dadd_rn(num, __dmul_rn(w, (double)v));
        den = __dadd_rn(den, w);
      }
    }
    out[i] = (OUT)__ddiv_rn(num, den);
  }
}

template <int R, typename OUT>
int launch_tile(const uint8_t* img, int H, int W, int row0, int row1, const double* sp,
                const double* rg, OUT* out, cudaStream_t s) {
  constexpr int S = 2 * R + 1;
  static const int variant = [] {
    const char* e = getenv("HB_BILAT_CFG");
    return e ? atoi(e) : 0;
  }();
  if (variant == 0 || (variant >= 4 && variant <= 9)) {
    // TMA-staged tiles.  default: one row per thread, symmetric 511-entry
    // range table, 3 CTAs/SM; HB_BILAT_CFG 4: |d| table, 5: 2 rows, 6: 3 rows,
    // 7: 2 rows with the symmetric table
    auto launch_tma = [&](auto kern, auto tag, bool sym) -> int {
      using T = decltype(tag);
      CUtensorMap map;
      if (!make_image_tmap(&map, img, H, W, T::TWB, T::TH)) return -1;
      const size_t smem = (size_t)(T::TH * T::TWB + 127) / 128 * 128 + (sym ? 511 : 256) * 16 * 8 + S * S * 8;
      HB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      dim3 grid((unsigned)ceil_div(W, kTileW), (unsigned)ceil_div(row1 - row0, T::TILE_H));
      kern<<<grid, kThreads, smem, s>>>(map, img, H, W, row0, row1, sp, rg, out);
      return check_launch();
    };
    int rc;
    if (variant == 4) rc = launch_tma(bilateral_tma_kernel<R, OUT, 1, 3>, TmaTile<R, 1>{}, false);
    else if (variant == 5) rc = launch_tma(bilateral_tma_kernel<R, OUT, 2, 2>, TmaTile<R, 2>{}, false);
    else if (variant == 6) rc = launch_tma(bilateral_tma_kernel<R, OUT, 3, 2>, TmaTile<R, 3>{}, false);
    else if (variant == 7) rc = launch_tma(bilateral_tma_kernel<R, OUT, 2, 2, true>, TmaTile<R, 2>{}, true);
    else if (variant == 8) rc = launch_tma(bilateral_tma_kernel<R, OUT, 1, 3, true, true>, TmaTile<R, 1>{}, true);
    else if (variant == 9) {
      using TT = TmaTile<R, 1>;
      CUtensorMap map;
      if (!make_image_tmap(&map, img, H, W, TT::TWB, TT::TH)) {
        rc = -1;
      } else {
        const size_t tb = (size_t)(TT::TH * TT::TWB + 127) / 128 * 128;
        const size_t smem = 2 * tb + 511 * 16 * 8 + S * S * 8;
        auto kern = bilateral_tmap_kernel<R, OUT, 3>;
        HB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        DeviceInfo di;
        HB_TRY(device_info(&di));
        const int tiles_x = (int)ceil_div(W, kTileW);
        const int64_t ntiles = (int64_t)tiles_x * ceil_div(row1 - row0, kTileH);
        HB_CHECK_ARG(ntiles < INT32_MAX, "image too large");
        int64_t grid = (int64_t)di.sms * 3;
        if (grid > ntiles) grid = ntiles;
        kern<<<(unsigned)grid, kThreads, smem, s>>>(map, img, H, W, row0, row1, sp, rg, out, tiles_x, (int)ntiles);
        rc = check_launch();
      }
    }
    else rc = launch_tma(bilateral_tma_kernel<R, OUT, 1, 3, true>, TmaTile<R, 1>{}, true);
    if (rc != -1) return rc;  // -1: no tensor map for this layout, plain tiles below
  }
  if (variant == 0 || variant == 2) {
    // one CTA per tile, 16-lane striped table (46 KB smem), 3 CTAs per SM
    const size_t smem = 256 * 16 * 8 + S * S * 8 + (size_t)(kTileH + 2 * R) * (kTileW + 2 * R) * 4;
    auto k = variant == 0 ? bilateral_tile_kernel<R, OUT, 16, 3> : bilateral_tile_kernel<R, OUT, 16, 2>;
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((unsigned)ceil_div(W, kTileW), (unsigned)ceil_div(row1 - row0, kTileH));
    k<<<grid, kThreads, smem, s>>>(img, H, W, row0, row1, sp, rg, out);
    return check_launch();
  }
  if (variant == 3) {
    const size_t smem = 256 * 32 * 8 + S * S * 8 + 2 * (size_t)(kTileH + 2 * R) * (kTileW + 2 * R) * 4;
    HB_CUDA_TRY(cudaFuncSetAttribute(bilateral_persist_kernel<R, OUT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DeviceInfo di;
    HB_TRY(device_info(&di));
    const int tiles_x = (int)ceil_div(W, kTileW);
    const int64_t ntiles = (int64_t)tiles_x * ceil_div(row1 - row0, kTileH);
    HB_CHECK_ARG(ntiles < INT32_MAX, "image too large");
    int64_t grid = (int64_t)di.sms * 2;
    if (grid > ntiles) grid = ntiles;
    bilateral_persist_kernel<R, OUT><<<(unsigned)grid, kThreads, smem, s>>>(img, H, W, row0, row1, sp, rg, out,
                                                                            tiles_x, (int)ntiles);
    return check_launch();
  }
  const size_t smem = 256 * 32 * 8 + S * S * 8 + (size_t)(kTileH + 2 * R) * (kTileW + 2 * R) * 4;
  HB_CUDA_TRY(cudaFuncSetAttribute(bilateral_tile_kernel<R, OUT>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)ceil_div(W, kTileW), (unsigned)ceil_div(row1 - row0, kTileH));
  bilateral_tile_kernel<R, OUT><<<grid, kThreads, smem, s>>>(img, H, W, row0, row1, sp, rg, out);
  return check_launch();
}

template <typename OUT>
int launch_bilateral(const uint8_t* img, int H, int W, int row0, int row1, int R, const double* sp,
                     const double* rg, OUT* out, cudaStream_t s) {
  switch (R) {
    case 0: return launch_tile<0, OUT>(img, H, W, row0, row1, sp, rg, out, s);
    case 1: return launch_tile<1, OUT>(img, H, W, row0, row1, sp, rg, out, s);
    case 2: return launch_tile<2, OUT>(img, H, W, row0, row1, sp, rg, out, s);
    case 3: return launch_tile<3, OUT>(img, H, W, row0, row1, sp, rg, out, s);
    case 4: return launch_tile<4, OUT>(img, H, W, row0, row1, sp, rg, out, s);
    case 5: return launch_tile<5, OUT>(img, H, W, row0, row1, sp, rg, out, s);
    case 6: return launch_tile<6, OUT>(img, H, W, row0, row1, sp, rg, out, s);
    case 7: return launch_tile<7, OUT>(img, H, W, row0, row1, sp, rg, out, s);
    case 8: return launch_tile<8, OUT>(img, H, W, row0, row1, sp, rg, out, s);
    default: {
      DeviceInfo di;
      HB_TRY(device_info(&di));
      int64_t n = (int64_t)(row1 - row0) * W;
      int64_t blocks = ceil_div(n, 256);
      if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
      bilateral_generic_kernel<OUT><<<(int)blocks, 256, 0, s>>>(img, H, W, row0, row1, R, sp, rg, out);
      return check_launch();
    }
  }
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hb_bilateral_u8(const uint8_t* img, int32_t height, int32_t width, int32_t radius,
                               const double* spatial, const double* range256, int32_t row0,
                               int32_t row1, void* out, int out_code, int flags, void* stream) {
  HB_CHECK_ARG(height > 0 && width > 0, "image must be non-empty");
  HB_CHECK_ARG(radius >= 0 && radius <= 255, "radius must be in [0, 255]");
  HB_CHECK_ARG(row0 >= 0 && row1 >= row0 && row1 <= height, "bad row range");
  HB_CHECK_ARG(out_code == 64 || out_code == 32, "out_code must be 64 (fp64) or 32 (fp32)");
  if (row1 == row0) return HB_OK;
  HB_CHECK_ARG(img && spatial && range256 && out, "NULL pointer");
  const bool dev = flags & HB_DEVICE_PTRS;
  HB_CHECK_ARG(dev || !(flags & HB_ASYNC), "HB_ASYNC requires device pointers");
  cudaStream_t s = as_stream(stream);
  const int S = 2 * radius + 1;
  // host calls: stage only the strip and its clamped halo rows
  int in0 = 0, in1 = height;
  if (!dev) {
    in0 = row0 - radius < 0 ? 0 : row0 - radius;
    in1 = row1 + radius > height ? height : row1 + radius;
  }
  DevBuf d_img, d_sp, d_rg, d_out;
  HB_TRY(stage_in(&d_sp, spatial, (size_t)S * S * 8, dev, s));
  HB_TRY(stage_in(&d_rg, range256, 256 * 8, dev, s));
  const size_t es = out_code == 64 ? 8 : 4;
  const size_t out_bytes = (size_t)(row1 - row0) * width * es;
  HB_TRY(stage_out(&d_out, out, out_bytes, dev, s));
  // the kernel sees a (in1-in0)-row image; clamping at its edges equals
  // clamping at the true image edges because the staged rows cover the halo
  const int h = in1 - in0;
  auto launch = [&](int a, int b) -> int {  // absolute rows [a, b)
    char* o = d_out.as<char>() + (size_t)(a - row0) * width * es;
    return out_code == 64
               ? launch_bilateral<double>(d_img.as<uint8_t>(), h, width, a - in0, b - in0, radius, d_sp.as<double>(), d_rg.as<double>(), reinterpret_cast<double*>(o), s)
               : launch_bilateral<float>(d_img.as<uint8_t>(), h, width, a - in0, b - in0, radius, d_sp.as<double>(), d_rg.as<double>(), reinterpret_cast<float*>(o), s);
  };
  if (dev) {
    d_img.ptr = const_cast<uint8_t*>(img);
    HB_TRY(launch(row0, row1));
  } else {
    // host buffers: row chunks with H2D / kernel / D2H overlapped
    HB_TRY(alloc(&d_img, (size_t)h * width, s));
    HB_TRY(row_pipeline(reinterpret_cast<const char*>(img) + (size_t)in0 * width, width, in0, in1, radius, row0,
                        row1, reinterpret_cast<char*>(out), width * es, d_img.as<char>(), d_out.as<char>(), s, launch));
  }
  return finish(flags, s);
}
