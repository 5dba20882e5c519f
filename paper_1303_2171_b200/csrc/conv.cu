// conv.cu — clamp-to-edge 2-D correlation on row strips (replaces
// convolve_rows / ConvolutionWorkload.run_part, reference
// kernels_regular.py:359-414).
//
// Arithmetic is the reference's, bit for bit: the reference adds one weighted
// plane per tap, `out += weight * slab[dy:, dx:]`, in row-major (dy, dx)
// order, skipping taps whose weight is exactly 0.0 (:376-381).  Per pixel
// that is acc = acc + w*I with a rounded fp64 multiply and a rounded add (no
// FMA), acc starting at +0.0, the pixel converted to fp64 exactly
// (`pixels.astype(np.float64)`).  Zero taps are skipped here too, so -0.0,
// inf and NaN propagate exactly as in the reference.
//
// Layout: one CTA = a 32 x 64 output tile; the clamped (32+2R) x (64+2R)
// halo tile is staged in shared memory as fp64 (uint8 or fp64 input); each
// thread owns 8 horizontally adjacent outputs and holds the (8+2R)-wide row
// segment of the current tap row in registers, so each tap costs one DMUL +
// one DADD per pixel and no shared-memory traffic (the weight is a warp-wide
// broadcast).  Bound: fp64 issue (2 flops per tap per pixel), not HBM.
#include <stdlib.h>
#include <string.h>

#include <type_traits>
#include <vector>

#include "common.cuh"

namespace hb {
namespace {

constexpr int kTileH = 32;
constexpr int kTileW = 64;
constexpr int kPx = 8;
constexpr int kThreads = kTileH * kTileW / kPx;  // 256
constexpr int kMaxR = 8;

template <typename IN>
__device__ __forceinline__ double to_f64(IN v) { return (double)v; }

// NR output rows per thread (32·NR x 64 tile, 256 threads): each input row
// segment loaded from smem feeds all NR rows (tap row dy = iy - k for the
// thread's k-th row), cutting segment and weight loads per output by NR and
// multiplying the independent accumulation chains that hide the fp64 result
// latency.  Tap order per output pixel is still row-major (iy increases), so
// the result is bit-identical.
//
// The row segments come in as 16-byte shared loads, and lane l
// of a warp takes row group l % 4, pixel group l / 4, so the 8 lanes of each
// quarter-warp hit 8 distinct 16-byte bank slots (the row stride NR·TW is
// ≡ 2·odd mod 16 doubles) — conflict-free, where the row-major lane order
// put 4 lanes on each slot (ncu: 61 % of the shared wavefronts were
// conflicts).  Same pixels per thread, same tap order.
//
// ACC = float: the fp32-arithmetic mode (within 1e-5 relative of the fp64
// result, north_star's filter tolerance): fp32 tile and weights, one FMA per
// tap, 8-byte (float2) segment loads — the same lane mapping stays
// conflict-free (row stride 3·78 ≡ 10 mod 32 banks).
template <int R, typename IN, typename OUT, bool DENSE, int MINB, int NR, typename ACC = double>
__global__ void __launch_bounds__(kThreads, MINB)
    conv_rows_kernel(const IN* __restrict__ img, int H, int W, int row0, int row1,
                     const double* __restrict__ weights, OUT* __restrict__ out) {
  constexpr int S = 2 * R + 1;
  constexpr int SWP = (S * S + 3) & ~3;  // weights padded so the tile is 16-B aligned
  constexpr int TILE_H = kTileH * NR;
  constexpr int TH = TILE_H + 2 * R, TW = kTileW + 2 * R;
  extern __shared__ __align__(16) unsigned char smem[];
  ACC* sw = reinterpret_cast<ACC*>(smem);  // [S*S]
  ACC* tile = sw + SWP;                    // [TH][TW]
  const int tid = threadIdx.x;
  const int y0 = row0 + blockIdx.y * TILE_H;
  const int x0 = blockIdx.x * kTileW;
  for (int i = tid; i < S * S; i += kThreads) sw[i] = (ACC)weights[i];
  for (int i = tid; i < TH * TW; i += kThreads) {
    const int ty = i / TW, tx = i - ty * TW;
    const int gy = min(max(y0 - R + ty, 0), H - 1);
    const int gx = min(max(x0 - R + tx, 0), W - 1);
    tile[i] = (ACC)to_f64(img[(int64_t)gy * W + gx]);
  }
  __syncthreads();
  static_assert(kTileW / kPx == 8 && kThreads % 32 == 0, "lane mapping assumes 8 pixel groups per row");
  const int lane = tid & 31;
  const int rgrp = (tid >> 5) * 4 + (lane & 3);
  const int py = rgrp * NR;  // first of the thread's NR output rows
  const int px = (lane >> 2) * kPx;
  const int gy = y0 + py;
  if (gy >= row1) return;
  ACC acc[NR][kPx];
#pragma unroll
  for (int k = 0; k < NR; ++k)
#pragma unroll
    for (int j = 0; j < kPx; ++j) acc[k][j] = (ACC)0;
#pragma unroll 1
  for (int iy = 0; iy < S + NR - 1; ++iy) {  // input rows py .. py+S+NR-2 of the tile
    ACC seg[kPx + 2 * R];
    const ACC* trow = tile + (py + iy) * TW + px;
    static_assert(TW % 2 == 0 && (kPx + 2 * R) % 2 == 0, "two-element segment loads");
    using V2 = typename std::conditional<sizeof(ACC) == 8, double2, float2>::type;
#pragma unroll
    for (int q = 0; q < (kPx + 2 * R) / 2; ++q) {
      const V2 v = reinterpret_cast<const V2*>(trow)[q];
      seg[2 * q] = v.x;
      seg[2 * q + 1] = v.y;
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const int dy = iy - k;
      if (dy >= 0 && dy < S) {
#pragma unroll
        for (int dx = 0; dx < S; ++dx) {
          const ACC w = sw[dy * S + dx];
          if (DENSE || w != (ACC)0) {
#pragma unroll
            for (int j = 0; j < kPx; ++j) {
              if constexpr (sizeof(ACC) == 8) acc[k][j] = __dadd_rn(acc[k][j], __dmul_rn(w, seg[j + dx]));  // bit-exact
              else acc[k][j] = fmaf(w, seg[j + dx], acc[k][j]);
            }
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
      if (x0 + px + j < W) o[j] = (OUT)acc[k][j];
  }
}

// radius > kMaxR: same arithmetic, neighbours read from global memory
template <typename IN, typename OUT>
__global__ void conv_generic_kernel(const IN* __restrict__ img, int H, int W, int row0, int row1, int R,
                                    const double* __restrict__ weights, OUT* __restrict__ out) {
  const int64_t n = (int64_t)(row1 - row0) * W;
  const int S = 2 * R + 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = row0 + (int)(i / W), x = (int)(i % W);
    double acc = 0.0;
    for (int dy = 0; dy < S; ++dy) {
      const int yy = min(max(y + dy - R, 0), H - 1);
      for (int dx = 0; dx < S; ++dx) {
        const double w = weights[dy * S + dx];
        if (w == 0.0) continue;
        const int xx = min(max(x + dx - R, 0), W - 1);
        acc = __dadd_rn(acc, __dmul_rn(w, to_f64(img[(int64_t)yy * W + xx])));
      }
    }
    out[i] = (OUT)acc;
  }
}

// NR = 3 output rows per thread (96 x 64 tiles), 2 CTAs/SM (measured at
// r=7: 38 Gpix/s; 2 rows 0.68, 1 row 0.61 of the fp64 peak)
template <int R, typename IN, typename OUT>
int launch_tile(const IN* img, int H, int W, int row0, int row1, const double* w, bool dense, OUT* out,
                bool fp32, cudaStream_t s) {
  constexpr int S = 2 * R + 1, NR = 3;
  const size_t es = fp32 ? 4 : 8;
  const size_t smem = (size_t)((S * S + 3) & ~3) * es + (size_t)(kTileH * NR + 2 * R) * (kTileW + 2 * R) * es;
  dim3 grid((unsigned)ceil_div(W, kTileW), (unsigned)ceil_div(row1 - row0, kTileH * NR));
  auto launch = [&](auto kern) -> int {
    HB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, kThreads, smem, s>>>(img, H, W, row0, row1, w, out);
    return check_launch();
  };
  // all-non-zero weights: the branch-free variant; otherwise zero taps are skipped like the reference
  if (fp32)
    return dense ? launch(conv_rows_kernel<R, IN, OUT, true, 2, NR, float>)
                 : launch(conv_rows_kernel<R, IN, OUT, false, 2, NR, float>);
  return dense ? launch(conv_rows_kernel<R, IN, OUT, true, 2, NR>) : launch(conv_rows_kernel<R, IN, OUT, false, 2, NR>);
}

template <typename IN, typename OUT>
int launch_conv(const IN* img, int H, int W, int row0, int row1, int R, const double* w, bool dense, OUT* out,
                bool fp32, cudaStream_t s) {
  switch (R) {
    case 0: return launch_tile<0, IN, OUT>(img, H, W, row0, row1, w, dense, out, fp32, s);
    case 1: return launch_tile<1, IN, OUT>(img, H, W, row0, row1, w, dense, out, fp32, s);
    case 2: return launch_tile<2, IN, OUT>(img, H, W, row0, row1, w, dense, out, fp32, s);
    case 3: return launch_tile<3, IN, OUT>(img, H, W, row0, row1, w, dense, out, fp32, s);
    case 4: return launch_tile<4, IN, OUT>(img, H, W, row0, row1, w, dense, out, fp32, s);
    case 5: return launch_tile<5, IN, OUT>(img, H, W, row0, row1, w, dense, out, fp32, s);
    case 6: return launch_tile<6, IN, OUT>(img, H, W, row0, row1, w, dense, out, fp32, s);
    case 7: return launch_tile<7, IN, OUT>(img, H, W, row0, row1, w, dense, out, fp32, s);
    case 8: return launch_tile<8, IN, OUT>(img, H, W, row0, row1, w, dense, out, fp32, s);
    default: {
      DeviceInfo di;
      HB_TRY(device_info(&di));
      int64_t blocks = ceil_div((int64_t)(row1 - row0) * W, 256);
      if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
      conv_generic_kernel<IN, OUT><<<(int)blocks, 256, 0, s>>>(img, H, W, row0, row1, R, w, out);
      return check_launch();
    }
  }
}

template <typename IN>
int dispatch_out(const void* img, int H, int W, int row0, int row1, int R, const double* w, bool dense,
                 void* out, int out_code, bool fp32, cudaStream_t s) {
  auto in = reinterpret_cast<const IN*>(img);
  return out_code == 64 ? launch_conv<IN, double>(in, H, W, row0, row1, R, w, dense, reinterpret_cast<double*>(out), fp32, s)
                        : launch_conv<IN, float>(in, H, W, row0, row1, R, w, dense, reinterpret_cast<float*>(out), fp32, s);
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hb_convolve(const void* img, int in_code, int32_t height, int32_t width, int32_t radius,
                           const double* weights, int32_t row0, int32_t row1, void* out, int out_code,
                           int flags, void* stream) {
  HB_CHECK_ARG(height > 0 && width > 0, "image must be non-empty");
  HB_CHECK_ARG(radius >= 0 && radius <= 255, "radius must be in [0, 255]");
  HB_CHECK_ARG(row0 >= 0 && row1 >= row0 && row1 <= height, "bad row range");
  HB_CHECK_ARG(in_code == HB_U8 || in_code == HB_F64, "image must be uint8 or float64");
  HB_CHECK_ARG(out_code == 64 || out_code == 32, "out_code must be 64 (fp64) or 32 (fp32)");
  if (row1 == row0) return HB_OK;
  HB_CHECK_ARG(img && weights && out, "NULL pointer");
  const bool dev = flags & HB_DEVICE_PTRS;
  HB_CHECK_ARG(dev || !(flags & HB_ASYNC), "HB_ASYNC requires device pointers");
  cudaStream_t s = as_stream(stream);
  const bool fp32 = flags & HB_FP32_ARITH;
  const int S = 2 * radius + 1;
  const size_t es_in = in_code == HB_U8 ? 1 : 8;
  // host calls stage only the strip and its clamped halo rows
  int in0 = 0, in1 = height;
  if (!dev) {
    in0 = row0 - radius < 0 ? 0 : row0 - radius;
    in1 = row1 + radius > height ? height : row1 + radius;
  }
  DevBuf d_img, d_w, d_out;
  HB_TRY(stage_in(&d_w, weights, (size_t)S * S * 8, dev, s));
  const size_t es_out = out_code == 64 ? 8 : 4;
  const size_t out_bytes = (size_t)(row1 - row0) * width * es_out;
  HB_TRY(stage_out(&d_out, out, out_bytes, dev, s));
  // no zero tap → the branch-free kernel (the zero-skip test is the only
  // data-dependent branch of the tap loop); weights are read on the host
  bool dense = true;
  if (!(dev && (flags & HB_TAPS_DENSE))) {
    std::vector<double> hw((size_t)S * S);
    if (dev) {
      HB_CUDA_TRY(cudaMemcpyAsync(hw.data(), weights, hw.size() * 8, cudaMemcpyDeviceToHost, s));
      HB_CUDA_TRY(cudaStreamSynchronize(s));
    } else {
      memcpy(hw.data(), weights, hw.size() * 8);
    }
    for (double v : hw) dense &= v != 0.0;
  }
  const int h = in1 - in0;
  auto launch = [&](int a, int b) -> int {  // absolute rows [a, b)
    void* o = d_out.as<char>() + (size_t)(a - row0) * width * es_out;
    return in_code == HB_U8
               ? dispatch_out<uint8_t>(d_img.ptr, h, width, a - in0, b - in0, radius, d_w.as<double>(), dense, o, out_code, fp32, s)
               : dispatch_out<double>(d_img.ptr, h, width, a - in0, b - in0, radius, d_w.as<double>(), dense, o, out_code, fp32, s);
  };
  if (dev) {
    d_img.ptr = const_cast<void*>(img);
    HB_TRY(launch(row0, row1));
  } else {
    // host buffers: row chunks with H2D / kernel / D2H overlapped
    HB_TRY(alloc(&d_img, (size_t)h * width * es_in, s));
    HB_TRY(row_pipeline(reinterpret_cast<const char*>(img) + (size_t)in0 * width * es_in, width * es_in, in0, in1,
                        radius, row0, row1, reinterpret_cast<char*>(out), width * es_out, d_img.as<char>(),
                        d_out.as<char>(), s, launch));
  }
  return finish(flags, s);
}
