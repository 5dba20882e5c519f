// spmv.cu — row-blocked CSR SpMV over an nnz-sorted row range (replaces
// _csr_range_matvec / SpmvWorkload.run_part, reference
// kernels_irregular.py:206-211, :250-251) plus CSR structure validation
// (CsrMatrix.__post_init__, :44-60).
//
// HB_SPMV_SEQ (default) reproduces the reference arithmetic bit for bit:
// every product is one rounded fp64 multiply and every row is summed left to
// right from +0.0 with rounded adds, no FMA contraction (the reference's
// `np.bincount(row_of, weights=values*x[col])`).  Two kernels implement it:
// spmv_lpr_kernel (int32 row_ptr/col_idx, the layout spmv_preprocess emits;
// see its comment) and the generic spmv_seq_kernel (any index width):
//   * one CTA = ROWS consecutive rows; its nnz range is streamed in chunks of
//     CHUNK products: coalesced loads of values/col_idx (each warp load moves
//     256/128 contiguous bytes), x gathered through the read-only path (x is
//     L2-resident: 8 MB at the 1M config vs 126 MB of L2), products stored to
//     shared memory with an XOR swizzle;
//   * thread i owns row i of the block and adds its products sequentially
//     from shared memory; the swizzle makes the 16 lanes of a half-warp hit 16
//     distinct 8-byte bank pairs when consecutive rows have equal length (the
//     common case: rows are sorted by nnz), and the accumulator stays in a
//     register across chunks, so arbitrarily long rows are exact too;
//   * the store is fused with the inverse permutation when `perm` is given
//     (y[perm[i]] = row sum), otherwise y[i-row0] (the y_perm slice).
// HB_SPMV_WARP: warp-per-row tree reduction (one FMA-free product per lane,
// shuffle reduction): not bit-exact, within 1e-9 relative of the reference.
#include <stdlib.h>

#include <algorithm>
#include <type_traits>
#include <string.h>

#include <thread>
#include <vector>

#include "common.cuh"

namespace hb {
namespace {

constexpr int kRows = 256;      // rows per CTA == threads per CTA
constexpr int kChunk = 4096;    // products staged per chunk (32 KB smem)
constexpr int kUnroll = kChunk / kRows;
constexpr int kBatch = 8;          // loads in flight per thread per batch

__device__ __forceinline__ int swz(int k) { return k ^ ((k >> 4) & 15); }

template <typename P>
__device__ __forceinline__ int64_t ld_idx(const P* p, int64_t i) {
  return (int64_t)__ldg(p + i);
}

// L2 policies: the matrix streams through once (evict_first); x is reused by
// every row (evict_last keeps the 8 MB vector resident in the 126 MB L2).
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_keep(const double* a, uint64_t pol) {
  double d;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(d) : "l"(a), "l"(pol));
  return d;
}
__device__ __forceinline__ double ld_stream(const double* a, uint64_t pol) {
  double d;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(d) : "l"(a), "l"(pol));
  return d;
}
__device__ __forceinline__ int64_t ld_stream_idx(const int32_t* a, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int64_t ld_stream_idx(const int64_t* a, uint64_t pol) {
  int64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}

template <typename P, typename C, typename Q>
__global__ void __launch_bounds__(kRows, 4)
    spmv_seq_kernel(const P* __restrict__ row_ptr, const C* __restrict__ col,
                    const double* __restrict__ val, const double* __restrict__ x, int64_t row0,
                    int64_t row1, const Q* __restrict__ perm, double* __restrict__ y) {
  __shared__ double prod[kChunk];
  const int tid = threadIdx.x;
  const uint64_t keep = l2_evict_last(), stream = l2_evict_first();
  const int64_t blk0 = row0 + (int64_t)blockIdx.x * kRows;
  const int64_t r = blk0 + tid;
  const int64_t blk1 = min(blk0 + kRows, row1);
  const int64_t nz0 = ld_idx(row_ptr, blk0);
  const int64_t nz1 = ld_idx(row_ptr, blk1);
  int64_t rs = 0, re = 0;
  if (r < row1) {
    rs = ld_idx(row_ptr, r);
    re = ld_idx(row_ptr, r + 1);
  }
  double acc = 0.0;
  for (int64_t cs = nz0; cs < nz1; cs += kChunk) {
    const int n = (int)min((int64_t)kChunk, nz1 - cs);
    // products, kBatch independent (col, val) loads then kBatch x gathers in flight
#pragma unroll
    for (int u0 = 0; u0 < kUnroll; u0 += kBatch) {
      int64_t c[kBatch];
      double v[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int k = tid + (u0 + u) * kRows;
        if (k < n) {
          c[u] = ld_stream_idx(col + cs + k, stream);
          v[u] = ld_stream(val + cs + k, stream);
        }
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int k = tid + (u0 + u) * kRows;
        if (k < n) prod[swz(k)] = __dmul_rn(v[u], ld_keep(x + c[u], keep));
      }
    }
    __syncthreads();
    const int64_t a = max(rs, cs), b = min(re, cs + n);
    for (int64_t k = a; k < b; ++k) acc = __dadd_rn(acc, prod[swz((int)(k - cs))]);
    __syncthreads();
  }
  if (r < row1) {
    if (perm) y[(int64_t)perm[r]] = acc;
    else y[r - row0] = acc;
  }
}

// Lane-per-row, bulk-copy fed kernel (bit-exact; the default for int32
// indices).  What bounds it (measured, scripts/micro/*.cu):
//   * every nnz costs one random 8-byte x gather = one L2 sector request; an
//     SM issues <= ~0.9 such requests per clock (16M gathers alone: 62 us on
//     148 SMs), and together with the 200 MB matrix stream the floor is
//     ~72 us (micro: gathers + a coalesced 12 B/nnz stream);
//   * in-flight gather misses occupy L1: with less than ~100 KB of L1 left
//     over by the shared-memory carveout the gather rate halves, so shared
//     memory is kept to the bulk-copy stages and the carveout is set to
//     exactly what the resident CTAs need.
// Structure:
//   * a warp tile = 32 consecutive (nnz-sorted) rows, lane i owns row i;
//     tiles are dealt round-robin over all warps of the persistent grid;
//   * work item = chunk of <= CW nnz of a tile; lane 0 streams the val/col
//     ranges of the warp's next S items into the warp's private smem stages
//     with cp.async.bulk (per-warp mbarriers, expect_tx bytes) — the matrix
//     stream never occupies LSU request slots, which the gathers need;
//   * each lane walks its own row's slice of an item in order, B gathers in
//     flight per batch: acc = acc + val*x[col], rounded fp64 ops, no FMA —
//     the reference's bincount arithmetic — with no product buffer or
//     transposition through shared memory;
//   * tile bounds (producer) and row bounds + perm (consumers) are loaded
//     one tile ahead; the perm scatter y[perm[r]] is fused into the store.
// Bulk copies need 16-byte aligned addresses and sizes: an item copies the
// 16-byte blocks covering [cs, cs+n) and the consumers re-derive the offset of
// cs inside its block.  The copy never reaches past the 16-byte block holding
// the item's last element, so it never leaves the page of a valid byte.
template <int CW, int S, int WARPS>
struct LprLayout {
  static constexpr size_t kVal = (size_t)CW * 8 + 16;  // f64 stage (+ alignment slack)
  static constexpr size_t kCol = (size_t)CW * 4 + 16;  // i32 stage
  static constexpr size_t kStage = kVal + kCol;
  static constexpr size_t kWarp = S * kStage;
  static constexpr size_t kBytes = WARPS * kWarp;
};

template <typename Q, int CW, int S, int WARPS, int MINB, int B>
__global__ void __launch_bounds__(32 * WARPS, MINB)
    spmv_lpr_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                    const double* __restrict__ val, const double* __restrict__ x, int64_t row0,
                    int64_t row1, const Q* __restrict__ perm, double* __restrict__ y, int64_t ntiles) {
  using L = LprLayout<CW, S, WARPS>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_all[WARPS][S];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wsm = smem + warp * L::kWarp;
  uint64_t* full = full_all[warp];
  auto sval = [&](int s) { return reinterpret_cast<double*>(wsm + s * L::kStage); };
  auto scol = [&](int s) { return reinterpret_cast<int32_t*>(wsm + s * L::kStage + L::kVal); };
  const uint64_t keep = l2_evict_last();
  const int64_t nwarps = (int64_t)gridDim.x * WARPS;
  const int64_t first = (int64_t)blockIdx.x * WARPS + warp;
  if (first >= ntiles) return;
  auto tile_nz = [&](int64_t t, int64_t* a, int64_t* b) {
    const int64_t r0 = row0 + t * 32;
    *a = row_ptr[r0];
    *b = row_ptr[min(r0 + 32, row1)];
  };

  // ---- producer (lane 0): item cursor + prefetched bounds of the tile after
  int64_t p_tile = first, p_cs = 0, p_nz1 = 0, q_nz0 = 0, q_nz1 = 0;
  auto p_issue = [&](int s) {
    const int n = (int)min((int64_t)CW, p_nz1 - p_cs);
    const uintptr_t v0 = (uintptr_t)(val + p_cs) & ~(uintptr_t)15, v1 = ((uintptr_t)(val + p_cs + n) + 15) & ~(uintptr_t)15;
    const uintptr_t c0 = (uintptr_t)(col + p_cs) & ~(uintptr_t)15, c1 = ((uintptr_t)(col + p_cs + n) + 15) & ~(uintptr_t)15;
    const uint32_t vb = n ? (uint32_t)(v1 - v0) : 0u, cb = n ? (uint32_t)(c1 - c0) : 0u;
    mbar_expect_tx(&full[s], vb + cb);  // 0 bytes (empty tile) completes the phase at once
    if (n) {
      tma_bulk_g2s(sval(s), (const void*)v0, vb, &full[s]);
      tma_bulk_g2s(scol(s), (const void*)c0, cb, &full[s]);
    }
    p_cs += CW;
    if (p_cs >= p_nz1) {  // every tile has >= 1 item, so empty rows still write 0
      p_tile += nwarps;
      p_cs = q_nz0;
      p_nz1 = q_nz1;
      if (p_tile + nwarps < ntiles) tile_nz(p_tile + nwarps, &q_nz0, &q_nz1);
    }
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tile_nz(p_tile, &p_cs, &p_nz1);
    if (p_tile + nwarps < ntiles) tile_nz(p_tile + nwarps, &q_nz0, &q_nz1);
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (p_tile < ntiles) p_issue(s);
  }
  __syncwarp();

  // ---- consumers: this tile's row bounds + perm, next tile's prefetched
  auto row_info = [&](int64_t t, int64_t* rs, int64_t* re, int64_t* pm) {
    const int64_t r = row0 + t * 32 + lane;
    if (r < row1) {
      *rs = row_ptr[r];
      *re = row_ptr[r + 1];
      *pm = perm ? (int64_t)perm[r] : 0;
    } else {
      *rs = *re = *pm = 0;
    }
  };
  int64_t rs, re, pm, nrs = 0, nre = 0, npm = 0;
  row_info(first, &rs, &re, &pm);
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t tile = first; tile < ntiles; tile += nwarps) {
    if (tile + nwarps < ntiles) row_info(tile + nwarps, &nrs, &nre, &npm);
    const int64_t r0 = row0 + tile * 32;
    const int64_t nz0 = __shfl_sync(0xffffffffu, rs, 0);
    const int64_t nz1 = __shfl_sync(0xffffffffu, re, (int)min((int64_t)31, row1 - 1 - r0));
    double acc = 0.0;
    int64_t cs = nz0;
    do {
      const int n = (int)min((int64_t)CW, nz1 - cs);
      mbar_wait(&full[stage], phase);
      const double* sv = sval(stage) + (((uintptr_t)(val + cs) & 15) >> 3);
      const int32_t* sc = scol(stage) + (((uintptr_t)(col + cs) & 15) >> 2);
      const int a = (int)(max(rs, cs) - cs);
      const int cnt = max((int)(min(re, cs + n) - cs) - a, 0);
      const int m = __reduce_max_sync(0xffffffffu, cnt);
      for (int j0 = 0; j0 < m; j0 += B) {
        int c[B];
        double g[B];
#pragma unroll
        for (int j = 0; j < B; ++j) c[j] = j0 + j < cnt ? sc[a + j0 + j] : 0;
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (j0 + j < cnt) g[j] = ld_keep(x + c[j], keep);
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (j0 + j < cnt) acc = __dadd_rn(acc, __dmul_rn(sv[a + j0 + j], g[j]));
      }
      __syncwarp();
      if (lane == 0 && p_tile < ntiles) {  // stage consumed: refill it S items ahead
        fence_proxy_async_smem();
        p_issue(stage);
      }
      if (++stage == S) {
        stage = 0;
        phase ^= 1u;
      }
      cs += CW;
    } while (cs < nz1);
    if (r0 + lane < row1) {
      if (perm) y[pm] = acc;
      else y[r0 + lane - row0] = acc;
    }
    rs = nrs;
    re = nre;
    pm = npm;
  }
}

// warp-per-row tree reduction (not bit-exact)
template <typename P, typename C, typename Q>
__global__ void __launch_bounds__(256)
    spmv_warp_kernel(const P* __restrict__ row_ptr, const C* __restrict__ col,
                     const double* __restrict__ val, const double* __restrict__ x, int64_t row0,
                     int64_t row1, const Q* __restrict__ perm, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = row0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < row1;
       r += warps) {
    const int64_t a = ld_idx(row_ptr, r), b = ld_idx(row_ptr, r + 1);
    double acc = 0.0;
    for (int64_t k = a + lane; k < b; k += 32) acc += __dmul_rn(__ldg(val + k), __ldg(x + ld_idx(col, k)));
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      if (perm) y[(int64_t)perm[r]] = acc;
      else y[r - row0] = acc;
    }
  }
}

// ------------------------------------------------------------------ merge path
// HB_SPMV_MERGE: merge-path CSR SpMV (load-balanced for any row-length
// distribution, no preprocessing): the merge of the row-end offsets with the
// nnz indices (rows + nnz items) is cut into equal diagonal ranges — a tile
// of kMpThreads x kMpItems items per CTA, kMpItems per thread — so a row of
// 10^6 nnz costs the same as 10^6 rows of one.  Per tile: the CTA's merge
// coordinates are found by binary search, its products val*x[col] are
// computed cooperatively into shared memory (coalesced loads, parallel
// gathers), its row ends staged beside them; each thread then walks its
// kMpItems in merge order, writing every row that ends in its range and
// emitting a carry (row, partial) for the row it leaves open.  A second,
// tiny kernel adds each run of carries to its row in order.  Rows split
// across threads are summed in two or more pieces, so this mode is not
// bit-exact: within 1e-9 relative of the reference (north_star tolerance).
constexpr int kMpThreads = 128;
constexpr int kMpItems = 7;
constexpr int kMpTile = kMpThreads * kMpItems;

// first merge coordinate (rows consumed, nnz consumed) on diagonal d
template <typename P>
__device__ __forceinline__ void merge_search(const P* __restrict__ row_end, int64_t nrows, int64_t nnz0,
                                             int64_t nnz, int64_t d, int64_t* ri, int64_t* ki) {
  // row_end[i] = row_ptr[row0 + i + 1] (absolute); nz index k is "absolute - nnz0"
  int64_t lo = d - nnz > 0 ? d - nnz : 0, hi = d < nrows ? d : nrows;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)row_end[mid] - nnz0 <= d - mid - 1) lo = mid + 1;
    else hi = mid;
  }
  *ri = lo;
  *ki = d - lo;
}

template <typename P, typename C, typename Q>
__global__ void __launch_bounds__(kMpThreads)
    spmv_merge_kernel(const P* __restrict__ row_ptr, const C* __restrict__ col,
                      const double* __restrict__ val, const double* __restrict__ x, int64_t row0,
                      int64_t row1, const Q* __restrict__ perm, double* __restrict__ y,
                      int64_t* __restrict__ carry_row, double* __restrict__ carry_val) {
  __shared__ double s_prod[kMpTile + 1];
  __shared__ int64_t s_rend[kMpTile + 1];
  __shared__ int64_t s_coord[4];
  const int tid = threadIdx.x;
  const int64_t nrows = row1 - row0;
  const int64_t nnz0 = (int64_t)row_ptr[row0];
  const int64_t nnz = (int64_t)row_ptr[row1] - nnz0;
  const P* row_end = row_ptr + row0 + 1;
  const int64_t total = nrows + nnz;
  const int64_t d0 = (int64_t)blockIdx.x * kMpTile;
  const int64_t d1 = d0 + kMpTile < total ? d0 + kMpTile : total;
  if (tid < 2) {
    int64_t r, k;
    merge_search(row_end, nrows, nnz0, nnz, tid == 0 ? d0 : d1, &r, &k);
    s_coord[2 * tid] = r;
    s_coord[2 * tid + 1] = k;
  }
  __syncthreads();
  const int64_t tr0 = s_coord[0], tk0 = s_coord[1], tr1 = s_coord[2], tk1 = s_coord[3];
  // stage the tile's products and row ends
  for (int64_t k = tk0 + tid; k < tk1; k += kMpThreads) {
    const int64_t a = nnz0 + k;
    s_prod[k - tk0] = __dmul_rn(__ldg(val + a), __ldg(x + (int64_t)__ldg(col + a)));
  }
  for (int64_t r = tr0 + tid; r < tr1 + 1 && r < nrows; r += kMpThreads) s_rend[r - tr0] = (int64_t)row_end[r] - nnz0;
  __syncthreads();
  // this thread's diagonal range inside the tile
  const int64_t dt0 = d0 + (int64_t)tid * kMpItems;
  const int64_t gtid = (int64_t)blockIdx.x * kMpThreads + tid;
  if (dt0 >= d1) {
    carry_row[gtid] = -1;
    carry_val[gtid] = 0.0;
    return;
  }
  // local merge search against the staged row ends
  int64_t r, k;
  {
    const int64_t dl = dt0 - d0;  // diagonal within the tile
    const int64_t rn = tr1 - tr0 + (tr1 < nrows ? 1 : 0), kn = tk1 - tk0;
    int64_t lo = dl - kn > 0 ? dl - kn : 0, hi = dl < rn ? dl : rn;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (s_rend[mid] - tk0 <= dl - mid - 1) lo = mid + 1;
      else hi = mid;
    }
    r = tr0 + lo;
    k = tk0 + (dl - lo);
  }
  double acc = 0.0;
  const int64_t dend = dt0 + kMpItems < d1 ? dt0 + kMpItems : d1;
  for (int64_t dd = dt0; dd < dend; ++dd) {
    if (r < nrows && k >= s_rend[r - tr0]) {  // row r ends here
      if (perm) y[(int64_t)perm[row0 + r]] = acc;
      else y[r] = acc;
      acc = 0.0;
      ++r;
    } else {
      acc = __dadd_rn(acc, s_prod[k - tk0]);
      ++k;
    }
  }
  carry_row[gtid] = r < nrows ? r : -1;
  carry_val[gtid] = acc;
}

// add each run of carries (consecutive threads carrying the same row) to the
// row, in thread order
template <typename Q>
__global__ void spmv_merge_fixup(const int64_t* __restrict__ carry_row, const double* __restrict__ carry_val,
                                 int64_t ncarry, int64_t row0, const Q* __restrict__ perm, double* __restrict__ y) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ncarry; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = carry_row[t];
    if (r < 0 || (t > 0 && carry_row[t - 1] == r)) continue;  // not the head of a run
    double s = 0.0;
    for (int64_t u = t; u < ncarry && carry_row[u] == r; ++u) s = __dadd_rn(s, carry_val[u]);
    const int64_t dst = perm ? (int64_t)perm[row0 + r] : r;
    y[dst] = __dadd_rn(y[dst], s);
  }
}

// ------------------------------------------------------------------ validation
// Flags: 1 row_ptr[0] != 0 or row_ptr[rows] != nnz, 2 decreasing row_ptr,
//        4 column out of range, 8 columns not strictly increasing in a row.
template <typename P, typename C>
__global__ void csr_validate_kernel(const P* __restrict__ row_ptr, const C* __restrict__ col,
                                    int64_t rows, int64_t nnz, int64_t cols,
                                    unsigned int* __restrict__ flags) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned int f = 0;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t0 == 0 && ((int64_t)row_ptr[0] != 0 || (int64_t)row_ptr[rows] != nnz)) f |= 1;
  for (int64_t r = t0; r < rows; r += stride) {
    const int64_t a = row_ptr[r], b = row_ptr[r + 1];
    if (b < a) { f |= 2; continue; }
    if (a < 0 || b > nnz) { f |= 1; continue; }
    int64_t prev = -1;
    for (int64_t k = a; k < b; ++k) {
      const int64_t c = (int64_t)col[k];
      if (c < 0 || c >= cols) f |= 4;
      if (c <= prev) f |= 8;
      prev = c;
    }
  }
  if (f) atomicOr(flags, f);
}

int idx_size_ok(int code) { return code == HB_I32 || code == HB_I64; }

// Shared-memory carveout: just what the resident CTAs need.  The rest of the
// unified 256 KB stays L1, which holds the in-flight x gathers — with less
// than ~100 KB of L1 the SM's gather rate halves (scripts/micro/l2gather.cu:
// 0.88 gathers/clk/SM at carveout <= 64 %, 0.44 at >= 86 %).
inline int carveout_pct(size_t smem_per_sm) {
  const size_t max_smem = 228 * 1024;
  const int pct = (int)((smem_per_sm * 100 + max_smem - 1) / max_smem);
  return pct > 100 ? 100 : pct;
}

template <typename Q, int CW, int S, int WARPS, int MINB, int B>
int launch_lpr(const void* rp, const void* ci, const double* v, const double* x, int64_t row0,
               int64_t row1, const void* pm, double* y, const DeviceInfo& di, cudaStream_t s) {
  using L = LprLayout<CW, S, WARPS>;
  auto k = spmv_lpr_kernel<Q, CW, S, WARPS, MINB, B>;
  HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::kBytes));
  HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                   carveout_pct(MINB * (L::kBytes + 256 + 1024))));
  const int64_t ntiles = ceil_div(row1 - row0, 32);
  int64_t grid = (int64_t)di.sms * MINB;
  if (grid > ceil_div(ntiles, WARPS)) grid = ceil_div(ntiles, WARPS);
  k<<<(unsigned)grid, 32 * WARPS, L::kBytes, s>>>(reinterpret_cast<const int32_t*>(rp), reinterpret_cast<const int32_t*>(ci),
                                                  v, x, row0, row1, reinterpret_cast<const Q*>(pm), y, ntiles);
  return check_launch();
}

// Lane-per-row tiles: 256-nnz smem chunks, 2 stages, 4 warps per CTA, 6 CTAs/SM,
// 4 gathers in flight per lane (measured best of the shapes tried).
template <typename P, typename C, typename Q>
int launch_spmv(const void* rp, const void* ci, const double* v, const double* x, int64_t row0,
                int64_t row1, const void* pm, double* y, int mode, cudaStream_t s) {
  const int64_t rows = row1 - row0;
  if (rows <= 0) return HB_OK;
  DeviceInfo di;
  HB_TRY(device_info(&di));
  auto p = reinterpret_cast<const P*>(rp);
  auto c = reinterpret_cast<const C*>(ci);
  auto q = reinterpret_cast<const Q*>(pm);
  if (mode == 2) {
    // nnz of the range is needed for the grid: one small D2H read of row_ptr[row0], row_ptr[row1]
    P ends[2];
    HB_CUDA_TRY(cudaMemcpyAsync(&ends[0], p + row0, sizeof(P), cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaMemcpyAsync(&ends[1], p + row1, sizeof(P), cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    const int64_t total = rows + ((int64_t)ends[1] - (int64_t)ends[0]);
    const int64_t blocks = ceil_div(total, kMpTile);
    if (blocks > INT32_MAX) { set_error("too many rows"); return HB_EINVAL; }
    DevBuf crow, cval;
    HB_TRY(alloc(&crow, (size_t)blocks * kMpThreads * 8, s));
    HB_TRY(alloc(&cval, (size_t)blocks * kMpThreads * 8, s));
    spmv_merge_kernel<P, C, Q><<<(unsigned)blocks, kMpThreads, 0, s>>>(p, c, v, x, row0, row1, q, y,
                                                                       crow.as<int64_t>(), cval.as<double>());
    HB_TRY(check_launch());
    int64_t g = ceil_div(blocks * kMpThreads, 256);
    if (g > (int64_t)di.sms * 8) g = (int64_t)di.sms * 8;
    spmv_merge_fixup<Q><<<(int)g, 256, 0, s>>>(crow.as<int64_t>(), cval.as<double>(), blocks * kMpThreads, row0, q, y);
    return check_launch();
  }
  if (mode == 1) {
    int64_t blocks = ceil_div(rows, 8);
    if (blocks > (int64_t)di.sms * 8) blocks = (int64_t)di.sms * 8;
    spmv_warp_kernel<P, C, Q><<<(int)blocks, 256, 0, s>>>(p, c, v, x, row0, row1, q, y);
    return check_launch();
  }
  if (sizeof(P) == 4 && sizeof(C) == 4) return launch_lpr<Q, 256, 2, 4, 6, 4>(rp, ci, v, x, row0, row1, pm, y, di, s);
  const int64_t blocks = ceil_div(rows, kRows);
  if (blocks > INT32_MAX) { set_error("too many rows"); return HB_EINVAL; }
  spmv_seq_kernel<P, C, Q><<<(unsigned)blocks, kRows, 0, s>>>(p, c, v, x, row0, row1, q, y);
  return check_launch();
}

template <typename P, typename C>
int dispatch_perm(int perm_code, const void* rp, const void* ci, const double* v, const double* x,
                  int64_t row0, int64_t row1, const void* pm, double* y, int mode, cudaStream_t s) {
  if (perm_code == HB_I32) return launch_spmv<P, C, int32_t>(rp, ci, v, x, row0, row1, pm, y, mode, s);
  return launch_spmv<P, C, int64_t>(rp, ci, v, x, row0, row1, pm, y, mode, s);
}

template <typename I, typename O>
__global__ void rebase_kernel(const I* __restrict__ in, int64_t n, int64_t base, O* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (O)((int64_t)in[i] - base);
}

__global__ void narrow_i64_kernel(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

int read_index(const void* p, int code, int64_t i, bool dev, cudaStream_t s, int64_t* out) {
  const size_t es = code == HB_I32 ? 4 : 8;
  const char* src = reinterpret_cast<const char*>(p) + (size_t)i * es;
  int64_t v = 0;
  if (dev) {
    HB_CUDA_TRY(cudaMemcpyAsync(&v, src, es, cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
  } else {
    memcpy(&v, src, es);
  }
  *out = es == 4 ? (int64_t)(int32_t)(v & 0xffffffff) : v;
  return HB_OK;
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hb_spmv_csr(const void* row_ptr, int ptr_code, const void* col_idx, int col_code,
                           const double* values, int64_t row0, int64_t row1, int64_t cols,
                           const double* x, const void* perm, int perm_code, double* y, int mode,
                           int flags, void* stream) {
  HB_CHECK_ARG(idx_size_ok(ptr_code) && idx_size_ok(col_code), "row_ptr/col_idx must be int32 or int64");
  HB_CHECK_ARG(perm == nullptr || idx_size_ok(perm_code), "perm must be int32 or int64");
  HB_CHECK_ARG(row0 >= 0 && row1 >= row0, "bad row range [%lld, %lld)", (long long)row0, (long long)row1);
  HB_CHECK_ARG(cols >= 0, "cols must be >= 0");
  HB_CHECK_ARG(mode >= 0 && mode <= 2, "unknown SpMV mode %d", mode);
  if (row1 == row0) return HB_OK;
  HB_CHECK_ARG(row_ptr && y && x, "NULL row_ptr, x or y");
  const bool dev = flags & HB_DEVICE_PTRS;
  HB_CHECK_ARG(dev || !(flags & HB_ASYNC), "HB_ASYNC requires device pointers");
  cudaStream_t s = as_stream(stream);
  const size_t pe = ptr_code == HB_I32 ? 4 : 8, ce = col_code == HB_I32 ? 4 : 8;
  const size_t qe = perm_code == HB_I32 ? 4 : 8;
  const int64_t rows = row1 - row0;

  if (dev) {
    int rc;
    if (ptr_code == HB_I32 && col_code == HB_I32) rc = dispatch_perm<int32_t, int32_t>(perm_code, row_ptr, col_idx, values, x, row0, row1, perm, y, mode, s);
    else if (ptr_code == HB_I32) rc = dispatch_perm<int32_t, int64_t>(perm_code, row_ptr, col_idx, values, x, row0, row1, perm, y, mode, s);
    else if (col_code == HB_I32) rc = dispatch_perm<int64_t, int32_t>(perm_code, row_ptr, col_idx, values, x, row0, row1, perm, y, mode, s);
    else rc = dispatch_perm<int64_t, int64_t>(perm_code, row_ptr, col_idx, values, x, row0, row1, perm, y, mode, s);
    if (rc != HB_OK) return rc;
    return finish(flags, s);
  }

  // host arrays: stage only this row range (row_ptr slice, its nnz range, x)
  int64_t nz0 = 0, nz1 = 0;
  HB_TRY(read_index(row_ptr, ptr_code, row0, false, s, &nz0));
  HB_TRY(read_index(row_ptr, ptr_code, row1, false, s, &nz1));
  HB_CHECK_ARG(nz1 >= nz0 && nz0 >= 0, "row_ptr is not non-decreasing");
  DevBuf d_ptr, d_col, d_val, d_x, d_y;
  // rebase row_ptr so the staged col/val slices start at 0 — on the device,
  // from the raw slice (one DMA, no host pass); int32 when the range allows,
  // so int32 col_idx takes the lane-per-row kernel
  const bool p32 = nz1 - nz0 <= (int64_t)INT32_MAX;
  {
    DevBuf d_raw;
    HB_TRY(stage_in(&d_raw, reinterpret_cast<const char*>(row_ptr) + (size_t)row0 * pe, (size_t)(rows + 1) * pe, false, s));
    HB_TRY(alloc(&d_ptr, (size_t)(rows + 1) * (p32 ? 4 : 8), s));
    DeviceInfo di;
    HB_TRY(device_info(&di));
    int64_t g = ceil_div(rows + 1, 256);
    if (g > (int64_t)di.sms * 16) g = (int64_t)di.sms * 16;
    if (pe == 4 && p32) rebase_kernel<<<(int)g, 256, 0, s>>>(d_raw.as<int32_t>(), rows + 1, nz0, d_ptr.as<int32_t>());
    else if (pe == 4) rebase_kernel<<<(int)g, 256, 0, s>>>(d_raw.as<int32_t>(), rows + 1, nz0, d_ptr.as<int64_t>());
    else if (p32) rebase_kernel<<<(int)g, 256, 0, s>>>(d_raw.as<int64_t>(), rows + 1, nz0, d_ptr.as<int32_t>());
    else rebase_kernel<<<(int)g, 256, 0, s>>>(d_raw.as<int64_t>(), rows + 1, nz0, d_ptr.as<int64_t>());
    HB_TRY(check_launch());
  }
  HB_TRY(stage_in(&d_col, reinterpret_cast<const char*>(col_idx) + nz0 * ce, (size_t)(nz1 - nz0) * ce, false, s));
  HB_TRY(stage_in(&d_val, values + nz0, (size_t)(nz1 - nz0) * 8, false, s));
  HB_TRY(stage_in(&d_x, x, (size_t)cols * 8, false, s));
  // result rows go straight into page-locked host memory when there is some
  // (the caller's pinned y, or a pinned stage for the un-permute): the
  // kernel's coalesced y stores cross PCIe while it runs, which avoids a
  // separate D2H — whose first pass over freshly written device memory
  // measured ~1 ms for 8 MB here instead of 0.15 ms
  PinnedScratch scratch;
  void* ydev = nullptr;
  bool direct = false;
  if (perm == nullptr) direct = device_view(y, &ydev);
  else if ((size_t)rows * 8 <= ((size_t)32 << 20) && pinned_scratch(&scratch, (size_t)rows * 8) == HB_OK) {
    ydev = scratch.dev;
    direct = true;
  }
  if (!direct) HB_TRY(alloc(&d_y, (size_t)rows * 8, s));
  const double* dv = d_val.as<double>();
  const double* dx = d_x.as<double>();
  double* dy = direct ? reinterpret_cast<double*>(ydev) : d_y.as<double>();
  int rc;
  DevBuf d_col32;
  if (p32 && col_code == HB_I64 && cols <= (int64_t)INT32_MAX && nz1 > nz0) {
    // int64 host columns: narrow on the device so the lane-per-row kernel runs
    HB_TRY(alloc(&d_col32, (size_t)(nz1 - nz0) * 4, s));
    DeviceInfo di;
    HB_TRY(device_info(&di));
    int64_t g = ceil_div(nz1 - nz0, 256);
    if (g > (int64_t)di.sms * 16) g = (int64_t)di.sms * 16;
    narrow_i64_kernel<<<(int)g, 256, 0, s>>>(d_col.as<int64_t>(), nz1 - nz0, d_col32.as<int32_t>());
    HB_TRY(check_launch());
    rc = launch_spmv<int32_t, int32_t, int64_t>(d_ptr.ptr, d_col32.ptr, dv, dx, 0, rows, nullptr, dy, mode, s);
  } else if (p32) rc = col_code == HB_I32 ? launch_spmv<int32_t, int32_t, int64_t>(d_ptr.ptr, d_col.ptr, dv, dx, 0, rows, nullptr, dy, mode, s)
                                   : launch_spmv<int32_t, int64_t, int64_t>(d_ptr.ptr, d_col.ptr, dv, dx, 0, rows, nullptr, dy, mode, s);
  else rc = col_code == HB_I32 ? launch_spmv<int64_t, int32_t, int64_t>(d_ptr.ptr, d_col.ptr, dv, dx, 0, rows, nullptr, dy, mode, s)
                               : launch_spmv<int64_t, int64_t, int64_t>(d_ptr.ptr, d_col.ptr, dv, dx, 0, rows, nullptr, dy, mode, s);
  if (rc != HB_OK) return rc;
  if (perm == nullptr) {
    if (!direct) HB_TRY(copy_d2h(y, d_y.ptr, (size_t)rows * 8, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    return HB_OK;
  }
  if (direct) {  // un-permute from the pinned rows the kernel wrote
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    const double* t = reinterpret_cast<const double*>(scratch.host);
    auto scatter_direct = [&](auto* pm) {
      const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(host_threads(), rows >> 15));
      host_parallel(parts, [&](int k) {
        for (int64_t i = rows * k / parts, e = rows * (k + 1) / parts; i < e; ++i) y[(int64_t)pm[row0 + i]] = t[i];
      });
    };
    if (perm_code == HB_I32) scatter_direct(reinterpret_cast<const int32_t*>(perm));
    else scatter_direct(reinterpret_cast<const int64_t*>(perm));
    return HB_OK;
  }
  // un-permute on the host straight from the pinned stage: y[perm[row0 + i]] = row sum i
  auto scatter = [&](auto* pm) -> int {
    return d2h_visit(d_y.ptr, (size_t)rows * 8, s, [&](const char* h, size_t off, size_t len) {
      const double* t = reinterpret_cast<const double*>(h);
      const int64_t i0 = (int64_t)(off / 8), n = (int64_t)(len / 8);
      const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(host_threads(), n >> 15));
      host_parallel(parts, [&](int k) {
        for (int64_t i = n * k / parts, e = n * (k + 1) / parts; i < e; ++i) y[(int64_t)pm[row0 + i0 + i]] = t[i];
      });
    });
  };
  HB_TRY(perm_code == HB_I32 ? scatter(reinterpret_cast<const int32_t*>(perm))
                             : scatter(reinterpret_cast<const int64_t*>(perm)));
  (void)qe;
  return HB_OK;
}

extern "C" int hb_csr_validate(const void* row_ptr, int ptr_code, const void* col_idx, int col_code,
                               int64_t rows, int64_t nnz, int64_t cols, uint32_t* flags_out,
                               int flags, void* stream) {
  HB_CHECK_ARG(idx_size_ok(ptr_code) && idx_size_ok(col_code), "row_ptr/col_idx must be int32 or int64");
  HB_CHECK_ARG(rows >= 0 && nnz >= 0 && cols >= 0, "negative size");
  HB_CHECK_ARG(flags_out, "flags_out is NULL");
  const bool dev = flags & HB_DEVICE_PTRS;
  cudaStream_t s = as_stream(stream);
  const size_t pe = ptr_code == HB_I32 ? 4 : 8, ce = col_code == HB_I32 ? 4 : 8;
  DevBuf d_ptr, d_col, d_f;
  HB_TRY(stage_in(&d_ptr, row_ptr, (size_t)(rows + 1) * pe, dev, s));
  HB_TRY(stage_in(&d_col, col_idx, (size_t)nnz * ce, dev, s));
  HB_TRY(alloc(&d_f, 4, s));
  HB_CUDA_TRY(cudaMemsetAsync(d_f.ptr, 0, 4, s));
  DeviceInfo di;
  HB_TRY(device_info(&di));
  int64_t blocks = ceil_div(rows > 0 ? rows : 1, 256);
  if (blocks > (int64_t)di.sms * 8) blocks = (int64_t)di.sms * 8;
  auto f = d_f.as<unsigned int>();
  if (ptr_code == HB_I32 && col_code == HB_I32) csr_validate_kernel<int32_t, int32_t><<<(int)blocks, 256, 0, s>>>((const int32_t*)d_ptr.ptr, (const int32_t*)d_col.ptr, rows, nnz, cols, f);
  else if (ptr_code == HB_I32) csr_validate_kernel<int32_t, int64_t><<<(int)blocks, 256, 0, s>>>((const int32_t*)d_ptr.ptr, (const int64_t*)d_col.ptr, rows, nnz, cols, f);
  else if (col_code == HB_I32) csr_validate_kernel<int64_t, int32_t><<<(int)blocks, 256, 0, s>>>((const int64_t*)d_ptr.ptr, (const int32_t*)d_col.ptr, rows, nnz, cols, f);
  else csr_validate_kernel<int64_t, int64_t><<<(int)blocks, 256, 0, s>>>((const int64_t*)d_ptr.ptr, (const int64_t*)d_col.ptr, rows, nnz, cols, f);
  HB_TRY(check_launch());
  unsigned int host = 0;
  HB_CUDA_TRY(cudaMemcpyAsync(&host, d_f.ptr, 4, cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaStreamSynchronize(s));
  *flags_out = host;
  return HB_OK;
}

// ------------------------------------------------------------------ preprocess
// Device spmv_preprocess (kernels_irregular.py:171-203): rows stably sorted
// by nnz (hb_sort of the row lengths with a row-index payload), new row_ptr
// by an exclusive scan, rows gathered warp-per-row.
namespace hb {
namespace {

template <typename P>
__global__ void row_len_kernel(const P* __restrict__ rp, int64_t rows, uint32_t* __restrict__ len,
                               uint32_t* __restrict__ idx) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    len[r] = (uint32_t)((int64_t)rp[r + 1] - (int64_t)rp[r]);
    idx[r] = (uint32_t)r;
  }
}

// exclusive scan of u32 lengths into row_ptr (int64 or int32), 3 phases
constexpr int kScanT = 512, kScanI = 8, kScanTile = kScanT * kScanI;

__global__ void __launch_bounds__(kScanT) scan_tile_sums(const uint32_t* __restrict__ v, int64_t n,
                                                         int64_t* __restrict__ sums) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  int64_t t = 0;
  for (int i = 0; i < kScanI; ++i) {
    const int64_t k = base + i * kScanT + threadIdx.x;
    if (k < n) t += v[k];
  }
  __shared__ int64_t ws[kScanT / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t a = 0;
    for (int w = 0; w < kScanT / 32; ++w) a += ws[w];
    sums[blockIdx.x] = a;
  }
}

__global__ void scan_sums_serial(int64_t* __restrict__ sums, int64_t nb) {
  // nb = rows / 4096: a few thousand values, one thread is fine
  int64_t run = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t c = sums[b];
    sums[b] = run;
    run += c;
  }
  sums[nb] = run;
}

template <typename P>
__global__ void __launch_bounds__(kScanT) scan_tile_apply(const uint32_t* __restrict__ v, int64_t n,
                                                          const int64_t* __restrict__ sums,
                                                          P* __restrict__ out) {
  // blocked layout: thread t owns elements [t*kScanI, (t+1)*kScanI) of the tile
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanI;
  uint32_t x[kScanI];
  int64_t tsum = 0;
#pragma unroll
  for (int i = 0; i < kScanI; ++i) {
    x[i] = base + i < n ? v[base + i] : 0u;
    tsum += x[i];
  }
  // block exclusive scan of tsum
  __shared__ int64_t ws[kScanT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  int64_t wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += ws[w];
  int64_t run = sums[blockIdx.x] + wpre + incl - tsum;
#pragma unroll
  for (int i = 0; i < kScanI; ++i) {
    if (base + i < n) out[base + i] = (P)run;
    run += x[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanT - 1) out[n] = (P)sums[gridDim.x];
}

template <typename PI, typename CI, typename PO, typename CO, typename QO>
__global__ void gather_rows_kernel(const PI* __restrict__ rp, const CI* __restrict__ col,
                                   const double* __restrict__ val, int64_t rows,
                                   const uint32_t* __restrict__ perm, const PO* __restrict__ nrp,
                                   CO* __restrict__ ncol, double* __restrict__ nval,
                                   QO* __restrict__ perm_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const int64_t old = perm[r];
    const int64_t a = (int64_t)rp[old], b = (int64_t)rp[old + 1];
    const int64_t d = (int64_t)nrp[r];
    for (int64_t k = a + lane; k < b; k += 32) {
      ncol[d + (k - a)] = (CO)col[k];
      nval[d + (k - a)] = val[k];
    }
    if (lane == 0) perm_out[r] = (QO)old;
  }
}

template <typename PI, typename CI, typename PO, typename CO, typename QO>
int preprocess_impl(const void* rp, const void* col, const double* val, int64_t rows, void* perm_out,
                    void* nrp, void* ncol, double* nval, cudaStream_t s) {
  DeviceInfo di;
  HB_TRY(device_info(&di));
  DevBuf len, idx;
  HB_TRY(alloc(&len, (size_t)rows * 4, s));
  HB_TRY(alloc(&idx, (size_t)rows * 4, s));
  int64_t g = ceil_div(rows, 256);
  if (g > (int64_t)di.sms * 16) g = (int64_t)di.sms * 16;
  row_len_kernel<PI><<<(int)g, 256, 0, s>>>((const PI*)rp, rows, len.as<uint32_t>(), idx.as<uint32_t>());
  HB_TRY(check_launch());
  int32_t passes = 0;
  // stable argsort: the ballot ranking (its stability is by construction)
  HB_TRY(hb_sort(len.ptr, len.ptr, HB_U32, idx.as<uint32_t>(), idx.as<uint32_t>(), rows, &passes,
                 HB_DEVICE_PTRS | HB_ASYNC | HB_SORT_BALLOT, s));
  const int64_t nb = ceil_div(rows, kScanTile);
  DevBuf sums;
  HB_TRY(alloc(&sums, (size_t)(nb + 1) * 8, s));
  scan_tile_sums<<<(unsigned)nb, kScanT, 0, s>>>(len.as<uint32_t>(), rows, sums.as<int64_t>());
  scan_sums_serial<<<1, 1, 0, s>>>(sums.as<int64_t>(), nb);
  scan_tile_apply<PO><<<(unsigned)nb, kScanT, 0, s>>>(len.as<uint32_t>(), rows, sums.as<int64_t>(), (PO*)nrp);
  HB_TRY(check_launch());
  int64_t gw = ceil_div(rows, 8);
  if (gw > (int64_t)di.sms * 32) gw = (int64_t)di.sms * 32;
  gather_rows_kernel<PI, CI, PO, CO, QO><<<(int)gw, 256, 0, s>>>(
      (const PI*)rp, (const CI*)col, val, rows, idx.as<uint32_t>(), (const PO*)nrp, (CO*)ncol, nval, (QO*)perm_out);
  return check_launch();
}

}  // namespace
}  // namespace hb

extern "C" int hb_spmv_preprocess(const void* row_ptr, int ptr_code, const void* col_idx, int col_code,
                                  const double* values, int64_t rows, void* perm_out, int perm_code,
                                  void* new_row_ptr, void* new_col, double* new_values, int flags,
                                  void* stream) {
  using namespace hb;
  HB_CHECK_ARG(idx_size_ok(ptr_code) && idx_size_ok(col_code) && idx_size_ok(perm_code),
               "index arrays must be int32 or int64");
  HB_CHECK_ARG(rows >= 1 && rows < (1ll << 30), "rows out of range");
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_spmv_preprocess works on device arrays");
  cudaStream_t s = as_stream(stream);
  int rc;
  // output index types follow the inputs (perm: perm_code)
#define HB_PP(PI, CI, QO) preprocess_impl<PI, CI, PI, CI, QO>(row_ptr, col_idx, values, rows, perm_out, new_row_ptr, new_col, new_values, s)
  const bool p4 = ptr_code == HB_I32, c4 = col_code == HB_I32, q4 = perm_code == HB_I32;
  if (p4 && c4) rc = q4 ? HB_PP(int32_t, int32_t, int32_t) : HB_PP(int32_t, int32_t, int64_t);
  else if (p4) rc = q4 ? HB_PP(int32_t, int64_t, int32_t) : HB_PP(int32_t, int64_t, int64_t);
  else if (c4) rc = q4 ? HB_PP(int64_t, int32_t, int32_t) : HB_PP(int64_t, int32_t, int64_t);
  else rc = q4 ? HB_PP(int64_t, int64_t, int32_t) : HB_PP(int64_t, int64_t, int64_t);
#undef HB_PP
  if (rc != HB_OK) return rc;
  return finish(flags, s);
}

// ------------------------------------------------------------------ gen_csr
// Device gen_csr (reference datasets.py:37-55), bit-identical:
//   counts[r] = min(1 + draw_{r+1}(mix_seed(s,1)) % (2·avg-1), cols)
//   row r's column draws come from one sequential stream SplitMix64(mix_seed(s,2)):
//     its seed is draw (r + 1 + retries so far) of that stream, its 2k+8
//     candidates are draws 1..2k+8 of that seed, % cols; the row keeps the
//     k smallest distinct values (np.unique(...)[:k]); a row with fewer than
//     k distinct candidates takes further stream draws (the retry loop), which
//     shifts every later row's seed by one draw per retry;
//   values = 2·uniform_floats(mix_seed(s,3), nnz) - 1.
// Warp per row: candidates in shared memory, distinct ranks by counting
// (O(m²) compares on broadcast reads — m ≤ 70 at the 1M config), first
// occurrence owns the slot.  Rows needing a retry (vanishingly rare unless
// cols is tiny) are found in one pass; the first one is replayed on the
// host exactly like the reference and the pass resumes after it.
namespace hb {
namespace {

constexpr int kGenWarps = 4;
constexpr int kGenMaxM = 2048;  // 2k+8 candidates per row: k <= 1020

__global__ void gen_counts_kernel(uint64_t seed, int64_t rows, uint64_t bound, int64_t cols,
                                  uint32_t* __restrict__ counts) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = 1 + (int64_t)(splitmix64_at(seed, (uint64_t)r + 1) % bound);
    counts[r] = (uint32_t)(c < cols ? c : cols);
  }
}

template <typename P, typename C>
__global__ void __launch_bounds__(kGenWarps * 32)
    gen_csr_rows_kernel(const P* __restrict__ rp, int64_t r_begin, int64_t rows, uint64_t seed_rows, int64_t shift,
                        uint64_t cols, C* __restrict__ col, unsigned long long* __restrict__ first_bad) {
  __shared__ uint32_t cand[kGenWarps][kGenMaxM];
  __shared__ uint8_t first[kGenWarps][kGenMaxM];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t warps = (int64_t)gridDim.x * kGenWarps;
  uint32_t* cv = cand[w];
  uint8_t* fv = first[w];
  for (int64_t r = r_begin + (int64_t)blockIdx.x * kGenWarps + w; r < rows; r += warps) {
    const int64_t base = (int64_t)rp[r];
    const int k = (int)((int64_t)rp[r + 1] - base);
    const int m = 2 * k + 8;
    const uint64_t s = splitmix64_at(seed_rows, (uint64_t)(r + 1 + shift));
    for (int i = lane; i < m; i += 32) cv[i] = (uint32_t)(splitmix64_at(s, (uint64_t)i + 1) % cols);
    __syncwarp();
    int distinct = 0;
    for (int i = lane; i < m; i += 32) {
      const uint32_t v = cv[i];
      bool f = true;
      for (int j = 0; j < i; ++j) f &= cv[j] != v;
      fv[i] = f;
      distinct += f;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) distinct += __shfl_xor_sync(0xffffffffu, distinct, o);
    __syncwarp();
    if (distinct < k) {
      if (lane == 0) atomicMin(first_bad, (unsigned long long)r);
    } else {
      for (int i = lane; i < m; i += 32) {
        if (!fv[i]) continue;
        const uint32_t v = cv[i];
        int rank = 0;
        for (int j = 0; j < m; ++j) rank += (fv[j] && cv[j] < v);
        if (rank < k) col[base + rank] = (C)v;
      }
    }
    __syncwarp();
  }
}

__global__ void gen_values_kernel(uint64_t seed, int64_t n, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double u = (double)(splitmix64_at(seed, (uint64_t)i + 1) >> 11) * 0x1p-53;
    out[i] = __dadd_rn(__dmul_rn(2.0, u), -1.0);
  }
}

template <typename P, typename C>
int gen_csr_impl(int64_t rows, int64_t cols, uint64_t bound, uint64_t seed_counts, uint64_t seed_rows,
                 uint64_t seed_vals, P* rp, C* col, double* vals, int64_t nnz_cap, int64_t* nnz_out, cudaStream_t s) {
  DeviceInfo di;
  HB_TRY(device_info(&di));
  DevBuf counts, sums, bad;
  HB_TRY(alloc(&counts, (size_t)rows * 4, s));
  int64_t g = ceil_div(rows, 256);
  if (g > (int64_t)di.sms * 16) g = (int64_t)di.sms * 16;
  gen_counts_kernel<<<(int)g, 256, 0, s>>>(seed_counts, rows, bound, cols, counts.as<uint32_t>());
  const int64_t nb = ceil_div(rows, kScanTile);
  HB_TRY(alloc(&sums, (size_t)(nb + 1) * 8, s));
  scan_tile_sums<<<(unsigned)nb, kScanT, 0, s>>>(counts.as<uint32_t>(), rows, sums.as<int64_t>());
  scan_sums_serial<<<1, 1, 0, s>>>(sums.as<int64_t>(), nb);
  scan_tile_apply<P><<<(unsigned)nb, kScanT, 0, s>>>(counts.as<uint32_t>(), rows, sums.as<int64_t>(), rp);
  HB_TRY(check_launch());
  int64_t nnz = 0;
  HB_CUDA_TRY(cudaMemcpyAsync(&nnz, sums.as<int64_t>() + nb, 8, cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaStreamSynchronize(s));
  *nnz_out = nnz;
  if (col == nullptr) return HB_OK;  // sizing call
  HB_CHECK_ARG(nnz_cap >= nnz, "col/values hold %lld entries, need %lld", (long long)nnz_cap, (long long)nnz);
  if (std::is_same<P, int32_t>::value) HB_CHECK_ARG(nnz < (1ll << 31), "nnz needs an int64 row_ptr");
  // rows denser than the shared-memory candidate buffer are not supported
  const uint64_t max_k = cols < (int64_t)bound + 1 ? (uint64_t)cols : bound;
  HB_CHECK_ARG(2 * max_k + 8 <= (uint64_t)kGenMaxM, "rows of up to %d nonzeros are supported on the device",
               (kGenMaxM - 8) / 2);
  HB_TRY(alloc(&bad, 8, s));
  int64_t gw = ceil_div(rows, kGenWarps);
  if (gw > (int64_t)di.sms * 8) gw = (int64_t)di.sms * 8;
  int64_t r_begin = 0, shift = 0;
  while (r_begin < rows) {
    const unsigned long long none = ~0ull;
    HB_CUDA_TRY(cudaMemcpyAsync(bad.ptr, &none, 8, cudaMemcpyHostToDevice, s));
    gen_csr_rows_kernel<P, C><<<(int)gw, kGenWarps * 32, 0, s>>>(rp, r_begin, rows, seed_rows, shift,
                                                                  (uint64_t)cols, col, bad.as<unsigned long long>());
    HB_TRY(check_launch());
    unsigned long long first_bad = none;
    HB_CUDA_TRY(cudaMemcpyAsync(&first_bad, bad.ptr, 8, cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    if (first_bad == none) break;
    // replay row `r` exactly like the reference: union of the candidates of
    // successive stream draws until k distinct values exist; keep the k smallest
    const int64_t r = (int64_t)first_bad;
    P ends[2];
    HB_CUDA_TRY(cudaMemcpyAsync(ends, rp + r, 2 * sizeof(P), cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    const int64_t k = (int64_t)ends[1] - (int64_t)ends[0];
    std::vector<uint64_t> chosen;
    int64_t draw = r + 1 + shift;
    for (;;) {
      const uint64_t sd = splitmix64_at(seed_rows, (uint64_t)draw);
      for (int64_t i = 1; i <= 2 * k + 8; ++i) chosen.push_back(splitmix64_at(sd, (uint64_t)i) % (uint64_t)cols);
      std::sort(chosen.begin(), chosen.end());
      chosen.erase(std::unique(chosen.begin(), chosen.end()), chosen.end());
      if ((int64_t)chosen.size() >= k) break;
      ++draw;
      ++shift;
    }
    std::vector<C> row((size_t)k);
    for (int64_t i = 0; i < k; ++i) row[(size_t)i] = (C)chosen[(size_t)i];
    HB_CUDA_TRY(cudaMemcpyAsync(col + (int64_t)ends[0], row.data(), (size_t)k * sizeof(C), cudaMemcpyHostToDevice, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    r_begin = r + 1;
  }
  int64_t gv = ceil_div(nnz, 256);
  if (gv > (int64_t)di.sms * 16) gv = (int64_t)di.sms * 16;
  if (nnz) gen_values_kernel<<<(int)gv, 256, 0, s>>>(seed_vals, nnz, vals);
  return check_launch();
}

}  // namespace
}  // namespace hb

extern "C" int hb_gen_csr(int64_t rows, int64_t cols, int64_t avg, uint64_t seed_counts, uint64_t seed_rows,
                          uint64_t seed_vals, void* row_ptr, int ptr_code, void* col_idx, int col_code,
                          double* values, int64_t nnz_cap, int64_t* nnz_out, int flags, void* stream) {
  using namespace hb;
  HB_CHECK_ARG(rows >= 1 && rows < (1ll << 31) && cols >= 1 && cols <= (1ll << 31), "matrix shape out of range");
  HB_CHECK_ARG(avg >= 1, "avg must be >= 1");
  HB_CHECK_ARG(idx_size_ok(ptr_code) && idx_size_ok(col_code), "index arrays must be int32 or int64");
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_gen_csr writes device arrays");
  HB_CHECK_ARG(row_ptr && nnz_out && (!col_idx == !values), "NULL pointer");
  cudaStream_t s = as_stream(stream);
  const uint64_t bound = (uint64_t)(2 * avg - 1 > 1 ? 2 * avg - 1 : 1);
  int rc;
#define HB_GC(P, C) gen_csr_impl<P, C>(rows, cols, bound, seed_counts, seed_rows, seed_vals, (P*)row_ptr, (C*)col_idx, values, nnz_cap, nnz_out, s)
  if (ptr_code == HB_I32) rc = col_code == HB_I32 ? HB_GC(int32_t, int32_t) : HB_GC(int32_t, int64_t);
  else rc = col_code == HB_I32 ? HB_GC(int64_t, int32_t) : HB_GC(int64_t, int64_t);
#undef HB_GC
  if (rc != HB_OK) return rc;
  return finish(flags, s);
}

// ------------------------------------------------------------------ SELL-32 layout
// The lane-per-row kernel reads lane i's row slice at offset a_i + j of a
// CSR chunk in shared memory; nnz-sorted tiles have equal row lengths L, so
// the 32 lanes read at a stride of L elements — 8-byte reads conflict
// 16/gcd(L,16)-ways (ncu: 2.2 M of the 6.4 M shared wavefronts were bank
// conflicts, all on the L1 data path the x gathers need).  The SELL-32 copy
// of the matrix stores each 32-row tile column-major (element j of the
// tile's row i at tile_off[t] + 32 j + i, tile length = its longest row, the
// padding never read): the stage is still filled by one contiguous bulk copy
// per chunk, and a warp's reads of step j are 32 consecutive words —
// conflict-free, 3 wavefronts per 32 nonzeros instead of ~12.  Same per-row
// sequential fp64 arithmetic (bit-identical).  Built once per device matrix
// (the nnz-sorted matrix of spmv_preprocess: padding ~0).
namespace hb {
namespace {

__global__ void sell_size_kernel(const int32_t* __restrict__ rp, int64_t rows, int64_t* __restrict__ tlen) {
  const int64_t ntiles = ceil_div(rows, 32);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = 0;
    const int64_t r1 = min((t + 1) * 32, rows);
    for (int64_t r = t * 32; r < r1; ++r) m = max(m, (int64_t)rp[r + 1] - (int64_t)rp[r]);
    tlen[t] = m * 32;
  }
}

__global__ void sell_scan_kernel(int64_t* __restrict__ v, int64_t n) {
  // exclusive scan in place, v[n] = total; one CTA of 1024 threads, blocked
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t a = min((int64_t)tid * per, n), b = min(a + per, n);
  int64_t s = 0;
  for (int64_t i = a; i < b; ++i) s += v[i];
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int64_t run = 0;
    for (int k = 0; k < 1024; ++k) {
      const int64_t c = part[k];
      part[k] = run;
      run += c;
    }
    v[n] = run;
  }
  __syncthreads();
  int64_t run = part[tid];
  for (int64_t i = a; i < b; ++i) {
    const int64_t c = v[i];
    v[i] = run;
    run += c;
  }
}

__global__ void sell_fill_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 const double* __restrict__ val, int64_t rows, const int64_t* __restrict__ toff,
                                 int32_t* __restrict__ scol, double* __restrict__ sval) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t ntiles = ceil_div(rows, 32);
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntiles; t += warps) {
    const int64_t r = t * 32 + lane;
    const int64_t rs = r < rows ? rp[r] : 0, re = r < rows ? rp[r + 1] : 0;
    const int64_t base = toff[t], len = (toff[t + 1] - base) / 32;
    for (int64_t j = 0; j < len; ++j) {
      const bool in = rs + j < re;
      scol[base + j * 32 + lane] = in ? col[rs + j] : 0;
      sval[base + j * 32 + lane] = in ? val[rs + j] : 0.0;
    }
  }
}

constexpr int kSellCJ = 8;     // j-steps per stage item (32 x 8 elements: 2 KB vals + 1 KB cols)
constexpr int kSellS = 2;      // stages per warp
constexpr int kSellWarps = 4;  // warps per CTA
constexpr int kSellMinB = 6;   // CTAs per SM
constexpr int kSellB = 4;      // x gathers in flight per lane per batch
constexpr size_t kSellStage = (size_t)kSellCJ * 32 * 12;
constexpr size_t kSellBytes = (size_t)kSellWarps * kSellS * kSellStage;

template <typename Q>
__global__ void __launch_bounds__(32 * kSellWarps, kSellMinB)
    spmv_sell_kernel(const int32_t* __restrict__ row_ptr, const int64_t* __restrict__ toff,
                     const int32_t* __restrict__ scol, const double* __restrict__ sval, const double* __restrict__ x,
                     int64_t row0, int64_t row1, const Q* __restrict__ perm, double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_all[kSellWarps][kSellS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wsm = smem + (size_t)warp * kSellS * kSellStage;
  uint64_t* full = full_all[warp];
  auto stv = [&](int s) { return reinterpret_cast<const double*>(wsm + s * kSellStage); };
  auto stc = [&](int s) { return reinterpret_cast<const int32_t*>(wsm + s * kSellStage + kSellCJ * 32 * 8); };
  const uint64_t keep = l2_evict_last();
  const uint64_t once = l2_evict_first();  // the matrix streams through once: leave L2 to x
  const int64_t t0 = row0 / 32, t1 = (row1 + 31) / 32;
  const int64_t nwarps = (int64_t)gridDim.x * kSellWarps;
  const int64_t first = t0 + (int64_t)blockIdx.x * kSellWarps + warp;
  if (first >= t1) return;

  // ---- producer (lane 0): streams the items (tile, j-chunk) of this warp's tiles
  int64_t p_tile = first, p_j = 0, p_len = 0;
  auto p_issue = [&](int s) {
    const int64_t base = toff[p_tile];
    const int nj = (int)min((int64_t)kSellCJ, p_len - p_j);
    const uint32_t vb = (uint32_t)nj * 256u, cb = (uint32_t)nj * 128u;
    mbar_expect_tx(&full[s], vb + cb);  // 0 bytes (empty tile) completes the phase at once
    if (nj > 0) {
      tma_bulk_g2s_hint(const_cast<double*>(stv(s)), sval + base + p_j * 32, vb, &full[s], once);
      tma_bulk_g2s_hint(const_cast<int32_t*>(stc(s)), scol + base + p_j * 32, cb, &full[s], once);
    }
    p_j += kSellCJ;
    if (p_j >= p_len) {  // every tile has >= 1 item, so empty rows still write 0
      p_tile += nwarps;
      p_j = 0;
      if (p_tile < t1) p_len = (toff[p_tile + 1] - toff[p_tile]) / 32;
    }
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kSellS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    p_len = (toff[p_tile + 1] - toff[p_tile]) / 32;
#pragma unroll
    for (int s = 0; s < kSellS; ++s)
      if (p_tile < t1) p_issue(s);
  }
  __syncwarp();

  int stage = 0;
  uint32_t phase = 0;
  for (int64_t tile = first; tile < t1; tile += nwarps) {
    const int64_t r = tile * 32 + lane;
    const bool mine = r >= row0 && r < row1;
    const int len = mine ? (int)((int64_t)row_ptr[r + 1] - (int64_t)row_ptr[r]) : 0;
    const int64_t pm = (mine && perm) ? (int64_t)perm[r] : 0;
    const int64_t tlen = (toff[tile + 1] - toff[tile]) / 32;
    double acc = 0.0;
    int64_t j0 = 0;
    do {
      mbar_wait(&full[stage], phase);
      const double* sv = stv(stage);
      const int32_t* sc = stc(stage);
      const int cnt = (int)max((int64_t)0, min((int64_t)kSellCJ, (int64_t)len - j0));
      for (int jj = 0; jj < cnt; jj += kSellB) {
        int c[kSellB];
        double g[kSellB];
#pragma unroll
        for (int u = 0; u < kSellB; ++u) c[u] = jj + u < cnt ? sc[(jj + u) * 32 + lane] : 0;
#pragma unroll
        for (int u = 0; u < kSellB; ++u)
          if (jj + u < cnt) g[u] = ld_keep(x + c[u], keep);
#pragma unroll
        for (int u = 0; u < kSellB; ++u)
          if (jj + u < cnt) acc = __dadd_rn(acc, __dmul_rn(sv[(jj + u) * 32 + lane], g[u]));
      }
      __syncwarp();
      if (lane == 0 && p_tile < t1) {  // stage consumed: refill it S items ahead
        fence_proxy_async_smem();
        p_issue(stage);
      }
      if (++stage == kSellS) {
        stage = 0;
        phase ^= 1u;
      }
      j0 += kSellCJ;
    } while (j0 < tlen);
    if (mine) {
      if (perm) y[pm] = acc;
      else y[r - row0] = acc;
    }
  }
}

}  // namespace
}  // namespace hb

extern "C" int hb_spmv_sell_build(const int32_t* row_ptr, const int32_t* col_idx, const double* values, int64_t rows,
                                  int64_t* tile_off, int32_t* sell_col, double* sell_val, int64_t* total_out,
                                  int flags, void* stream) {
  using namespace hb;
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_spmv_sell_build works on device arrays");
  HB_CHECK_ARG(rows >= 1 && row_ptr && tile_off && total_out, "bad arguments");
  cudaStream_t s = as_stream(stream);
  DeviceInfo di;
  HB_TRY(device_info(&di));
  const int64_t ntiles = ceil_div(rows, 32);
  if (sell_col == nullptr) {  // sizing: tile_off (ntiles+1, device) and the total element count
    int64_t g = ceil_div(ntiles, 256);
    if (g > (int64_t)di.sms * 16) g = (int64_t)di.sms * 16;
    sell_size_kernel<<<(int)g, 256, 0, s>>>(row_ptr, rows, tile_off);
    sell_scan_kernel<<<1, 1024, 0, s>>>(tile_off, ntiles);
    HB_TRY(check_launch());
    HB_CUDA_TRY(cudaMemcpyAsync(total_out, tile_off + ntiles, 8, cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    return HB_OK;
  }
  HB_CHECK_ARG(col_idx && values && sell_val, "NULL pointer");
  int64_t g = ceil_div(ntiles, 8);
  if (g > (int64_t)di.sms * 16) g = (int64_t)di.sms * 16;
  sell_fill_kernel<<<(int)g, 256, 0, s>>>(row_ptr, col_idx, values, rows, tile_off, sell_col, sell_val);
  return finish(flags, s);
}

extern "C" int hb_spmv_sell(const int32_t* row_ptr, const int64_t* tile_off, const int32_t* sell_col,
                            const double* sell_val, int64_t row0, int64_t row1, const double* x, const void* perm,
                            int perm_code, double* y, int flags, void* stream) {
  using namespace hb;
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_spmv_sell works on device arrays");
  HB_CHECK_ARG(row0 >= 0 && row1 >= row0, "bad row range");
  HB_CHECK_ARG(perm == nullptr || idx_size_ok(perm_code), "perm must be int32 or int64");
  if (row1 == row0) return HB_OK;
  cudaStream_t s = as_stream(stream);
  DeviceInfo di;
  HB_TRY(device_info(&di));
  const int64_t ntiles = (row1 + 31) / 32 - row0 / 32;
  int64_t grid = (int64_t)di.sms * kSellMinB;
  if (grid > ceil_div(ntiles, kSellWarps)) grid = ceil_div(ntiles, kSellWarps);
  int rc;
  if (perm == nullptr || perm_code == HB_I32) {
    auto k = spmv_sell_kernel<int32_t>;
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSellBytes));
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     carveout_pct(kSellMinB * (kSellBytes + 256 + 1024))));
    k<<<(unsigned)grid, 32 * kSellWarps, kSellBytes, s>>>(row_ptr, tile_off, sell_col, sell_val, x, row0, row1,
                                                          reinterpret_cast<const int32_t*>(perm), y);
    rc = check_launch();
  } else {
    auto k = spmv_sell_kernel<int64_t>;
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSellBytes));
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     carveout_pct(kSellMinB * (kSellBytes + 256 + 1024))));
    k<<<(unsigned)grid, 32 * kSellWarps, kSellBytes, s>>>(row_ptr, tile_off, sell_col, sell_val, x, row0, row1,
                                                          reinterpret_cast<const int64_t*>(perm), y);
    rc = check_launch();
  }
  if (rc != HB_OK) return rc;
  return finish(flags, s);
}
