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

// ACC = float: the fp32-arithmetic mode (north_star: filter outputs within
// 1e-5 relative): fp32 tables striped over 32 lanes (the same 128-byte table
// rows), w = s·r, num = fma(w, nb, num), den += w — half the issue slots of
// the fp64 tap and one shared wavefront per warp-tap instead of two.
template <int R, typename OUT, int NR, int MINB, bool SYM = false, typename ACC = double>
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
  constexpr int ST = 128 / (int)sizeof(ACC);  // table stripes: one 128-byte row per intensity
  uint8_t* tile = smem;                                                     // [TH][TWB], 128-B aligned
  ACC* rng = reinterpret_cast<ACC*>(smem + ((TH * TWB + 127) / 128) * 128);  // [NE][ST]
  ACC* sp = rng + NE * ST;                                                  // [S*S]
  const int tid = threadIdx.x;
  const int lane = tid & (ST - 1);
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
  for (int i = tid; i < NE * ST; i += kThreads) rng[i] = (ACC)range[SYM ? abs(i / ST - 255) : i / ST];
  for (int i = tid; i < S * S; i += kThreads) sp[i] = (ACC)spatial[i];
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
  ACC num[NR][kPx], den[NR][kPx];
#pragma unroll
  for (int k = 0; k < NR; ++k)
#pragma unroll
    for (int j = 0; j < kPx; ++j) {
      c[k][j] = tile[(py + k + R) * TWB + px + j + R + OFF];
      num[k][j] = den[k][j] = (ACC)0;
    }
  const ACC* lane_rng = rng + lane + (SYM ? 255 * ST : 0);
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
    ACC nbd[kPx + 2 * R];
    const uint8_t* trow = tile + (py + iy) * TWB + px + OFF;
#pragma unroll
    for (int q = 0; q < kPx + 2 * R; ++q) nb[q] = trow[q];
#pragma unroll
    for (int q = 0; q < kPx + 2 * R; ++q) {
      nbd[q] = (ACC)nb[q];
      if (SYM) nb[q] *= 128;  // byte offset of the intensity's table row
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const int dy = iy - k;
      if (dy < 0 || dy >= S) continue;
#pragma unroll
      for (int dx = 0; dx < S; ++dx) {
        const ACC s = sp[dy * S + dx];
#pragma unroll
        for (int j = 0; j < kPx; ++j) {
          ACC r;
          if constexpr (sizeof(ACC) == 8) {
            if (SYM) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(cbase[k][j] + (uint32_t)nb[j + dx]));
            else r = lane_rng[abs(nb[j + dx] - c[k][j]) * ST];
            const double w = __dmul_rn(s, r);  // the reference's op order, no FMA (bit-exact)
            num[k][j] = __dadd_rn(num[k][j], __dmul_rn(w, nbd[j + dx]));
            den[k][j] = __dadd_rn(den[k][j], w);
          } else {
            if (SYM) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(cbase[k][j] + (uint32_t)nb[j + dx]));
            else r = lane_rng[abs(nb[j + dx] - c[k][j]) * ST];
            const float w = s * r;
            num[k][j] = fmaf(w, nbd[j + dx], num[k][j]);
            den[k][j] = den[k][j] + w;
          }
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
      if (x0 + px + j < W) {
        if constexpr (sizeof(ACC) == 8) o[j] = (OUT)__ddiv_rn(num[k][j], den[k][j]);
        else o[j] = (OUT)__fdiv_rn(num[k][j], den[k][j]);
      }
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
                const double* rg, OUT* out, bool fp32, cudaStream_t s) {
  constexpr int S = 2 * R + 1;
  // TMA-staged halo tiles, one row per thread, signed 511-entry range table
  // striped over 16 lanes (fp64) / 32 lanes (fp32), 3 CTAs/SM (measured best)
  {
    using T = TmaTile<R, 1>;
    auto kern = fp32 ? bilateral_tma_kernel<R, OUT, 1, 3, true, float> : bilateral_tma_kernel<R, OUT, 1, 3, true, double>;
    CUtensorMap map;
    if (make_image_tmap(&map, img, H, W, T::TWB, T::TH)) {
      const size_t smem = (size_t)(T::TH * T::TWB + 127) / 128 * 128 + 511 * 128 + S * S * (fp32 ? 4 : 8);
      HB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      dim3 grid((unsigned)ceil_div(W, kTileW), (unsigned)ceil_div(row1 - row0, T::TILE_H));
      kern<<<grid, kThreads, smem, s>>>(map, img, H, W, row0, row1, sp, rg, out);
      return check_launch();
    }
  }
  // no tensor map for this layout (row pitch not a multiple of 16 bytes):
  // plain halo tiles loaded by the CTA, same arithmetic
  const size_t smem = 256 * 16 * 8 + S * S * 8 + (size_t)(kTileH + 2 * R) * (kTileW + 2 * R) * 4;
  auto k = bilateral_tile_kernel<R, OUT, 16, 3>;
  HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)ceil_div(W, kTileW), (unsigned)ceil_div(row1 - row0, kTileH));
  k<<<grid, kThreads, smem, s>>>(img, H, W, row0, row1, sp, rg, out);
  return check_launch();
}

template <typename OUT>
int launch_bilateral(const uint8_t* img, int H, int W, int row0, int row1, int R, const double* sp,
                     const double* rg, OUT* out, bool fp32, cudaStream_t s) {
  switch (R) {
    case 0: return launch_tile<0, OUT>(img, H, W, row0, row1, sp, rg, out, fp32, s);
    case 1: return launch_tile<1, OUT>(img, H, W, row0, row1, sp, rg, out, fp32, s);
    case 2: return launch_tile<2, OUT>(img, H, W, row0, row1, sp, rg, out, fp32, s);
    case 3: return launch_tile<3, OUT>(img, H, W, row0, row1, sp, rg, out, fp32, s);
    case 4: return launch_tile<4, OUT>(img, H, W, row0, row1, sp, rg, out, fp32, s);
    case 5: return launch_tile<5, OUT>(img, H, W, row0, row1, sp, rg, out, fp32, s);
    case 6: return launch_tile<6, OUT>(img, H, W, row0, row1, sp, rg, out, fp32, s);
    case 7: return launch_tile<7, OUT>(img, H, W, row0, row1, sp, rg, out, fp32, s);
    case 8: return launch_tile<8, OUT>(img, H, W, row0, row1, sp, rg, out, fp32, s);
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
  const bool fp32 = flags & HB_FP32_ARITH;
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
               ? launch_bilateral<double>(d_img.as<uint8_t>(), h, width, a - in0, b - in0, radius, d_sp.as<double>(), d_rg.as<double>(), reinterpret_cast<double*>(o), fp32, s)
               : launch_bilateral<float>(d_img.as<uint8_t>(), h, width, a - in0, b - in0, radius, d_sp.as<double>(), d_rg.as<double>(), reinterpret_cast<float*>(o), fp32, s);
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
