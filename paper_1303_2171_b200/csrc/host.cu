// host.cu — native DeviceA (host-core) kernels.  The host share of a
// work-shared run (fraction_a of the input) is computed here instead of in
// numpy: same arithmetic as the reference's numpy bodies, bit for bit, on
// `workers` std::threads (the reference's Device.worker_count sub-chunks).
//   hb_host_hist        HistogramWorkload.run_part DeviceA   kernels_regular.py:149-154
//   hb_host_spmv_rows   _csr_range_matvec                    kernels_irregular.py:206-211
//   hb_host_conv_rows   convolve_rows                        kernels_regular.py:359-381
//   hb_host_bilateral   bilateral_rows                       kernels_regular.py:461-486
// Floating point: one rounded multiply then one rounded add per term, in the
// reference's order (the Makefile builds host code with -ffp-contract=off,
// so no FMA is ever formed).  No GPU is touched.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "common.cuh"

namespace hb {
namespace {

template <typename F>
void parallel_chunks(int64_t n, int tasks, int workers, F&& fn) {
  // contiguous chunks [k*n/t, (k+1)*n/t), task k each, claimed dynamically by
  // at most `workers` threads of the persistent host-kernel pool (no thread
  // spawn per call)
  if (tasks <= 1 || workers <= 1 || n < 2) {
    for (int k = 0; k < std::max(1, tasks); ++k) fn(k, n * k / std::max(1, tasks), n * (k + 1) / std::max(1, tasks));
    return;
  }
  host_kernel_parallel(tasks, [&](int k) { fn(k, n * k / tasks, n * (k + 1) / tasks); }, workers);
}

// Tasks for `workers` threads over n units: up to kOversplit per worker (the
// pool claims them dynamically, so a thread that shares its core with another
// busy thread — e.g. the GPU side's synchronising caller — runs fewer chunks
// instead of holding up the whole host share with one static chunk), at
// least `min_units` units per task.  Chunking never changes a result: every
// host kernel's output is per element, per row or an integer sum.
constexpr int kOversplit = 16;
int task_count(int64_t n, int workers, int64_t min_units) {
  const int64_t by_size = std::max<int64_t>(1, n / std::max<int64_t>(1, min_units));
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)workers * kOversplit, by_size));
}

int clamp_workers(int w) {
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  return std::max(1, std::min(w, hw));
}

// uint8 fast path: two 8-byte words per iteration, byte k of each word counted
// in sub-histogram k (8 tables: no store-to-load dependency between nearby
// equal bytes; ~30 % faster than 4 tables on the B200 box's host,
// scripts/micro/host_hist.cpp), flushed to the 64-bit counts every 2^30 bytes.
bool hist_u8_fast(const uint8_t* d, int64_t a, int64_t b, int32_t bins, uint64_t* h) {
  if (bins < 256) return false;  // values >= bins possible: generic path checks them
  static thread_local uint32_t sub[8][256];
  int64_t i = a;
  while (i < b) {
    memset(sub, 0, sizeof(sub));
    const int64_t e = std::min(b, i + ((int64_t)1 << 30));
    for (; i < e && (i & 7); ++i) ++sub[0][d[i]];
    for (; i + 16 <= e; i += 16) {
      uint64_t w, u;
      memcpy(&w, d + i, 8);
      memcpy(&u, d + i + 8, 8);
      ++sub[0][w & 255];
      ++sub[1][(w >> 8) & 255];
      ++sub[2][(w >> 16) & 255];
      ++sub[3][(w >> 24) & 255];
      ++sub[4][(w >> 32) & 255];
      ++sub[5][(w >> 40) & 255];
      ++sub[6][(w >> 48) & 255];
      ++sub[7][w >> 56];
      ++sub[0][u & 255];
      ++sub[1][(u >> 8) & 255];
      ++sub[2][(u >> 16) & 255];
      ++sub[3][(u >> 24) & 255];
      ++sub[4][(u >> 32) & 255];
      ++sub[5][(u >> 40) & 255];
      ++sub[6][(u >> 48) & 255];
      ++sub[7][u >> 56];
    }
    for (; i < e; ++i) ++sub[0][d[i]];
    for (int v = 0; v < 256; ++v) {
      uint64_t t = 0;
      for (int k = 0; k < 8; ++k) t += sub[k][v];
      h[v] += t;
    }
  }
  return true;
}

template <typename T>
bool hist_body(const T* d, int64_t a, int64_t b, int32_t bins, uint64_t* h) {
  bool ok = true;
  for (int64_t i = a; i < b; ++i) {
    const int64_t v = (int64_t)d[i];
    if (v < 0 || v >= bins) {
      ok = false;
      continue;
    }
    ++h[v];
  }
  return ok;
}

int64_t idx_at(const void* p, int code, int64_t i) {
  return code == HB_I32 ? (int64_t) reinterpret_cast<const int32_t*>(p)[i] : reinterpret_cast<const int64_t*>(p)[i];
}

template <typename IN>
void conv_rows(const IN* img, int H, int W, int R, const double* w, int row0, int row1, double* out, int workers) {
  const int S = 2 * R + 1;
  parallel_chunks(row1 - row0, task_count(row1 - row0, workers, 1), workers, [&](int, int64_t a, int64_t b) {
    for (int64_t rr = a; rr < b; ++rr) {
      const int y = row0 + (int)rr;
      double* o = out + rr * W;
      for (int x = 0; x < W; ++x) o[x] = 0.0;
      // plane order of the reference: for each tap, all pixels of the row
      for (int dy = 0; dy < S; ++dy) {
        const IN* src = img + (int64_t)std::min(std::max(y + dy - R, 0), H - 1) * W;
        for (int dx = 0; dx < S; ++dx) {
          const double wt = w[dy * S + dx];
          if (wt == 0.0) continue;
          // interior columns need no clamp (contiguous, vectorised); borders clamp
          const int x0 = std::min(W, std::max(0, R - dx)), x1 = std::max(x0, std::min(W, W + R - dx));
          for (int x = 0; x < x0; ++x) {
            const double prod = wt * (double)src[std::min(std::max(x + dx - R, 0), W - 1)];
            o[x] = o[x] + prod;
          }
          const IN* s2 = src + dx - R;
          for (int x = x0; x < x1; ++x) {
            const double prod = wt * (double)s2[x];
            o[x] = o[x] + prod;
          }
          for (int x = x1; x < W; ++x) {
            const double prod = wt * (double)src[std::min(std::max(x + dx - R, 0), W - 1)];
            o[x] = o[x] + prod;
          }
        }
      }
    }
  });
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hb_host_hist(const void* data, int dtype, int64_t n, int32_t bin_count, uint64_t* bins_out,
                            int workers) {
  HB_CHECK_ARG(n >= 0, "n must be >= 0");
  HB_CHECK_ARG(bin_count >= 1, "bin_count must be >= 1");
  HB_CHECK_ARG(bins_out && (n == 0 || data), "NULL pointer");
  workers = clamp_workers(workers);
  // one private table per task: >= 2^18-element tasks, tables capped at 64 MB
  const int tasks = (int)std::max<int64_t>(
      1, std::min<int64_t>(task_count(n, workers, 1 << 18), (64ll << 20) / (8ll * bin_count)));
  std::vector<std::vector<uint64_t>> priv((size_t)tasks, std::vector<uint64_t>((size_t)bin_count, 0));
  std::vector<char> ok((size_t)tasks, 1);
  bool supported = true;
  parallel_chunks(n, tasks, workers, [&](int k, int64_t a, int64_t b) {
    uint64_t* h = priv[(size_t)k].data();
    bool r = true;
    switch (dtype) {
      case HB_U8:
        if (!hist_u8_fast(reinterpret_cast<const uint8_t*>(data), a, b, bin_count, h))
          r = hist_body(reinterpret_cast<const uint8_t*>(data), a, b, bin_count, h);
        break;
      case HB_I8: r = hist_body(reinterpret_cast<const int8_t*>(data), a, b, bin_count, h); break;
      case HB_U16: r = hist_body(reinterpret_cast<const uint16_t*>(data), a, b, bin_count, h); break;
      case HB_I16: r = hist_body(reinterpret_cast<const int16_t*>(data), a, b, bin_count, h); break;
      case HB_U32: r = hist_body(reinterpret_cast<const uint32_t*>(data), a, b, bin_count, h); break;
      case HB_I32: r = hist_body(reinterpret_cast<const int32_t*>(data), a, b, bin_count, h); break;
      case HB_U64: {
        const uint64_t* d = reinterpret_cast<const uint64_t*>(data);
        for (int64_t i = a; i < b; ++i) {
          if (d[i] >= (uint64_t)bin_count) r = false;
          else ++h[d[i]];
        }
        break;
      }
      case HB_I64: r = hist_body(reinterpret_cast<const int64_t*>(data), a, b, bin_count, h); break;
      default: supported = false;
    }
    ok[(size_t)k] = r;
  });
  HB_CHECK_ARG(supported, "unsupported histogram element type code %d", dtype);
  for (char c : ok) HB_CHECK_ARG(c, "element outside bin domain");
  for (int32_t j = 0; j < bin_count; ++j) {
    uint64_t t = 0;
    for (auto& h : priv) t += h[(size_t)j];
    bins_out[j] = t;
  }
  return HB_OK;
}

namespace hb {
namespace {

// CSR rows [row0, row1): typed loops (no per-element index-width dispatch),
// thread chunks balanced by nonzeros rather than rows (the nnz-sorted
// permuted matrix has very uneven row lengths), result written to y[i - row0]
// or scattered to y[perm[i]] when a permutation is given.
template <typename P, typename C, typename Q>
void spmv_rows_typed(const P* rp, const C* ci, const double* v, int64_t row0, int64_t row1, const double* x,
                     const Q* perm, double* y, int workers) {
  const int64_t rows = row1 - row0, nz0 = (int64_t)rp[row0], nnz = (int64_t)rp[row1] - nz0;
  const int tasks = (rows < 4096 || nnz < (1 << 16)) ? 1 : task_count(nnz, workers, 1 << 16);
  std::vector<int64_t> cut((size_t)tasks + 1);
  cut[0] = row0;
  cut[(size_t)tasks] = row1;
  for (int k = 1; k < tasks; ++k) {  // first row whose start reaches k/t of the nonzeros
    const int64_t target = nz0 + nnz * k / tasks;
    cut[(size_t)k] = std::max(cut[(size_t)k - 1], (int64_t)(std::lower_bound(rp + row0, rp + row1, (P)target) - rp));
  }
  parallel_chunks(tasks, tasks, workers, [&](int k, int64_t, int64_t) {
    for (int64_t r = cut[(size_t)k]; r < cut[(size_t)k + 1]; ++r) {
      const int64_t e = (int64_t)rp[r + 1];
      double acc = 0.0;
      for (int64_t j = (int64_t)rp[r]; j < e; ++j) {
        const double prod = v[j] * x[(int64_t)ci[j]];
        acc = acc + prod;
      }
      if (perm) y[(int64_t)perm[r]] = acc;
      else y[r - row0] = acc;
    }
  });
}

template <typename P, typename C>
void spmv_rows_perm(const P* rp, const C* ci, const double* v, int64_t row0, int64_t row1, const double* x,
                    const void* perm, int perm_code, double* y, int workers) {
  if (perm_code == HB_I32)
    spmv_rows_typed(rp, ci, v, row0, row1, x, reinterpret_cast<const int32_t*>(perm), y, workers);
  else
    spmv_rows_typed(rp, ci, v, row0, row1, x, reinterpret_cast<const int64_t*>(perm), y, workers);
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hb_host_spmv_rows(const void* row_ptr, int ptr_code, const void* col_idx, int col_code,
                                 const double* values, int64_t row0, int64_t row1, const double* x,
                                 const void* perm, int perm_code, double* y, int workers) {
  HB_CHECK_ARG((ptr_code == HB_I32 || ptr_code == HB_I64) && (col_code == HB_I32 || col_code == HB_I64),
               "row_ptr/col_idx must be int32 or int64");
  HB_CHECK_ARG(perm == nullptr || perm_code == HB_I32 || perm_code == HB_I64, "perm must be int32 or int64");
  HB_CHECK_ARG(row0 >= 0 && row1 >= row0, "bad row range");
  if (row1 == row0) return HB_OK;
  HB_CHECK_ARG(row_ptr && x && y, "NULL pointer");
  const int w = clamp_workers(workers);
  const bool p32 = ptr_code == HB_I32, c32 = col_code == HB_I32;
  const auto* p4 = reinterpret_cast<const int32_t*>(row_ptr);
  const auto* p8 = reinterpret_cast<const int64_t*>(row_ptr);
  const auto* c4 = reinterpret_cast<const int32_t*>(col_idx);
  const auto* c8 = reinterpret_cast<const int64_t*>(col_idx);
  if (p32 && c32) spmv_rows_perm(p4, c4, values, row0, row1, x, perm, perm_code, y, w);
  else if (p32) spmv_rows_perm(p4, c8, values, row0, row1, x, perm, perm_code, y, w);
  else if (c32) spmv_rows_perm(p8, c4, values, row0, row1, x, perm, perm_code, y, w);
  else spmv_rows_perm(p8, c8, values, row0, row1, x, perm, perm_code, y, w);
  return HB_OK;
}

extern "C" int hb_host_conv_rows(const void* img, int in_code, int32_t height, int32_t width, int32_t radius,
                                 const double* weights, int32_t row0, int32_t row1, double* out, int workers) {
  HB_CHECK_ARG(height > 0 && width > 0, "image must be non-empty");
  HB_CHECK_ARG(radius >= 0, "radius must be >= 0");
  HB_CHECK_ARG(row0 >= 0 && row1 >= row0 && row1 <= height, "bad row range");
  HB_CHECK_ARG(in_code == HB_U8 || in_code == HB_F64, "image must be uint8 or float64");
  if (row1 == row0) return HB_OK;
  HB_CHECK_ARG(img && weights && out, "NULL pointer");
  workers = clamp_workers(workers);
  if (in_code == HB_U8) conv_rows(reinterpret_cast<const uint8_t*>(img), height, width, radius, weights, row0, row1, out, workers);
  else conv_rows(reinterpret_cast<const double*>(img), height, width, radius, weights, row0, row1, out, workers);
  return HB_OK;
}

extern "C" int hb_host_bilateral(const uint8_t* img, int32_t height, int32_t width, int32_t radius,
                                 const double* spatial, const double* range256, int32_t row0, int32_t row1,
                                 double* out, int workers) {
  HB_CHECK_ARG(height > 0 && width > 0, "image must be non-empty");
  HB_CHECK_ARG(radius >= 0, "radius must be >= 0");
  HB_CHECK_ARG(row0 >= 0 && row1 >= row0 && row1 <= height, "bad row range");
  if (row1 == row0) return HB_OK;
  HB_CHECK_ARG(img && spatial && range256 && out, "NULL pointer");
  const int R = radius, S = 2 * R + 1, W = width, H = height;
  workers = clamp_workers(workers);
  parallel_chunks(row1 - row0, task_count(row1 - row0, workers, 1), workers, [&](int, int64_t a, int64_t b) {
    std::vector<double> num((size_t)W), den((size_t)W);
    for (int64_t rr = a; rr < b; ++rr) {
      const int y = row0 + (int)rr;
      const uint8_t* crow = img + (int64_t)y * W;
      std::fill(num.begin(), num.end(), 0.0);
      std::fill(den.begin(), den.end(), 0.0);
      for (int dy = 0; dy < S; ++dy) {
        const uint8_t* src = img + (int64_t)std::min(std::max(y + dy - R, 0), H - 1) * W;
        for (int dx = 0; dx < S; ++dx) {
          const double s = spatial[dy * S + dx];
          auto tap = [&](int x, int nb) {
            const double w = s * range256[abs(nb - (int)crow[x])];
            const double t = w * (double)nb;
            num[(size_t)x] = num[(size_t)x] + t;
            den[(size_t)x] = den[(size_t)x] + w;
          };
          const int x0 = std::min(W, std::max(0, R - dx)), x1 = std::max(x0, std::min(W, W + R - dx));
          for (int x = 0; x < x0; ++x) tap(x, src[std::min(std::max(x + dx - R, 0), W - 1)]);
          const uint8_t* s2 = src + dx - R;
          for (int x = x0; x < x1; ++x) tap(x, s2[x]);
          for (int x = x1; x < W; ++x) tap(x, src[std::min(std::max(x + dx - R, 0), W - 1)]);
        }
      }
      double* o = out + rr * W;
      for (int x = 0; x < W; ++x) o[x] = num[(size_t)x] / den[(size_t)x];
    }
  });
  return HB_OK;
}
