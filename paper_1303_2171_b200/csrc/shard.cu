// shard.cu — the multi-GPU side of the work-partitioned path: the device-side
// partitioner and the device halves of the merges that follow a collective.
//
//  hb_partition_nnz  SpMV shard boundaries: the reference's own
//                    searchsorted-on-nnz-prefix split rule
//                    (kernels_irregular.py:243-245, spmv_preprocess :196-197)
//                    evaluated at k/G for k = 1..G-1 by binary search over the
//                    device row_ptr — only G+1 integers leave the device.
//  hb_scatter_perm   y[perm[i]] = y_perm[i]: the un-permute of
//                    SpmvWorkload.merge (kernels_irregular.py:253-257), run
//                    on the all-gathered y_perm.
//  hb_merge_runs     stable merge of R sorted (key, payload) runs lying back to
//                    back — the local merge step of the multi-GPU sample-merge
//                    sort (the single-node analogue is the bin
//                    concatenation of sample_sort_hybrid, kernels_regular.py:310).
//                    log2(R) rounds of pairwise merge-path merges; ties keep run
//                    order, so runs received in rank order stay stable.
#include <vector>

#include "common.cuh"

namespace hb {
namespace {

// ------------------------------------------------------------- partitioner
template <typename P>
__global__ void partition_nnz_kernel(const P* __restrict__ rp, int64_t row0, int64_t row1, int parts,
                                     int64_t* __restrict__ bounds) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > parts) return;
  if (k == 0 || k == parts) {
    bounds[k] = k == 0 ? row0 : row1;
    return;
  }
  const int64_t base = (int64_t)rp[row0];
  const double total = (double)((int64_t)rp[row1] - base);
  // numpy: k * total / world, total a float64 → (k·total)/world in fp64
  const double thr = ((double)k * total) / (double)parts;
  // first i in [0, row1-row0] with cum[i] >= thr (searchsorted side='left')
  int64_t lo = 0, hi = row1 - row0 + 1;
  while (lo < hi) {
    const int64_t mid = lo + ((hi - lo) >> 1);
    const double c = (double)((int64_t)rp[row0 + mid] - base);
    if (c < thr) lo = mid + 1;
    else hi = mid;
  }
  bounds[k] = row0 + lo;
}

// ------------------------------------------------------------- permutation
template <typename T, typename I>
__global__ void scatter_perm_kernel(const T* __restrict__ src, int64_t n, const I* __restrict__ perm,
                                    T* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[(int64_t)perm[i]] = src[i];
}

// ------------------------------------------------------------- run merge
constexpr int kMergeThreads = 256;
constexpr int kMergeItems = 8;
constexpr int kMergeTile = kMergeThreads * kMergeItems;  // outputs per CTA

// Stable merge path (A wins ties): the number of A elements among the first
// `d` outputs of merge(A, B).
template <typename K, typename FA, typename FB>
__device__ __forceinline__ int64_t merge_path(FA a, int64_t na, FB b, int64_t nb, int64_t d) {
  int64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const K x = a(mid), y = b(d - 1 - mid);
    if (x <= y) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// One round: pair q merges runs [o[2q], o[2q+1]) and [o[2q+1], o[2q+2]) into
// the same output range.  tile_start[q] = first CTA of pair q.
template <typename K, bool PAY>
__global__ void __launch_bounds__(kMergeThreads)
    merge_round_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
                       uint32_t* __restrict__ vout, const int64_t* __restrict__ offs,
                       const int64_t* __restrict__ tile_start, int npairs) {
  __shared__ K sk[kMergeTile];
  __shared__ uint32_t sv[PAY ? kMergeTile : 1];
  __shared__ int64_t cut[2];
  // pair of this CTA (npairs is small: linear scan)
  int q = 0;
  while (q + 1 < npairs && tile_start[q + 1] <= (int64_t)blockIdx.x) ++q;
  const int64_t a0 = offs[2 * q], a1 = offs[2 * q + 1], b1 = offs[2 * q + 2];
  const int64_t na = a1 - a0, nb = b1 - a1;
  const int64_t t = (int64_t)blockIdx.x - tile_start[q];
  const int64_t d0 = t * kMergeTile;
  const int64_t d1 = min(d0 + (int64_t)kMergeTile, na + nb);
  const K* A = kin + a0;
  const K* B = kin + a1;
  if (threadIdx.x < 2) {
    const int64_t d = threadIdx.x == 0 ? d0 : d1;
    cut[threadIdx.x] = merge_path<K>([&](int64_t i) { return A[i]; }, na, [&](int64_t j) { return B[j]; }, nb, d);
  }
  __syncthreads();
  const int64_t i0 = cut[0], i1 = cut[1];
  const int64_t j0 = d0 - i0, j1 = d1 - i1;
  const int la = (int)(i1 - i0), lb = (int)(j1 - j0);
  // stage A[i0:i1] then B[j0:j1] (coalesced)
  for (int x = threadIdx.x; x < la; x += kMergeThreads) {
    sk[x] = A[i0 + x];
    if (PAY) sv[x] = vin[a0 + i0 + x];
  }
  for (int x = threadIdx.x; x < lb; x += kMergeThreads) {
    sk[la + x] = B[j0 + x];
    if (PAY) sv[la + x] = vin[a1 + j0 + x];
  }
  __syncthreads();
  // each thread merges kMergeItems outputs from its own diagonal
  const int dd = threadIdx.x * kMergeItems;
  const int tot = la + lb;
  K rk[kMergeItems];
  uint32_t rv[kMergeItems];
  int cnt = 0;
  if (dd < tot) {
    int i = (int)merge_path<K>([&](int64_t x) { return sk[x]; }, la, [&](int64_t y) { return sk[la + y]; }, lb, dd);
    int j = dd - i;
#pragma unroll
    for (int it = 0; it < kMergeItems; ++it) {
      if (dd + it >= tot) break;
      bool take_a;
      if (i >= la) take_a = false;
      else if (j >= lb) take_a = true;
      else take_a = sk[i] <= sk[la + j];
      const int src = take_a ? i : la + j;
      rk[it] = sk[src];
      if (PAY) rv[it] = sv[src];
      if (take_a) ++i;
      else ++j;
      ++cnt;
    }
  }
  __syncthreads();
  // restage in output order, then store coalesced
#pragma unroll
  for (int it = 0; it < kMergeItems; ++it) {
    if (it < cnt) {
      sk[dd + it] = rk[it];
      if (PAY) sv[dd + it] = rv[it];
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < tot; x += kMergeThreads) {
    kout[a0 + d0 + x] = sk[x];
    if (PAY) vout[a0 + d0 + x] = sv[x];
  }
}

template <typename K, bool PAY>
__global__ void copy_run_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
                                uint32_t* __restrict__ vout, int64_t lo, int64_t hi) {
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    kout[i] = kin[i];
    if (PAY) vout[i] = vin[i];
  }
}

template <typename K>
int merge_runs(const K* keys, const uint32_t* vals, int64_t n, const int64_t* offsets, int nruns, K* kout,
               uint32_t* vout, cudaStream_t s) {
  DeviceInfo di;
  HB_TRY(device_info(&di));
  const bool pay = vals != nullptr;
  std::vector<int64_t> runs(offsets, offsets + nruns + 1);
  // ping-pong: round r reads `src`, writes `dst`; the last round writes kout/vout
  int rounds = 0;
  for (int r = nruns; r > 1; r = (r + 1) / 2) ++rounds;
  if (rounds == 0) {
    if (keys != kout) HB_CUDA_TRY(cudaMemcpyAsync(kout, keys, (size_t)n * sizeof(K), cudaMemcpyDeviceToDevice, s));
    if (pay && vals != vout) HB_CUDA_TRY(cudaMemcpyAsync(vout, vals, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
    return HB_OK;
  }
  DevBuf tk, tv, d_offs, d_tiles;
  HB_TRY(alloc(&tk, (size_t)n * sizeof(K), s));
  if (pay) HB_TRY(alloc(&tv, (size_t)n * 4, s));
  HB_TRY(alloc(&d_offs, (size_t)(nruns + 2) * 8, s));
  HB_TRY(alloc(&d_tiles, (size_t)(nruns + 1) * 8, s));
  // buffers so that the final round lands in kout: with an even round count
  // the first round writes tk, with an odd count it writes kout
  const K* src_k = keys;
  const uint32_t* src_v = vals;
  std::vector<int64_t> h_offs, h_tiles;
  for (int r = 0; r < rounds; ++r) {
    const bool to_out = ((rounds - 1 - r) % 2) == 0;
    K* dst_k = to_out ? kout : tk.as<K>();
    uint32_t* dst_v = to_out ? vout : tv.as<uint32_t>();
    const int m = (int)runs.size() - 1;
    const int npairs = m / 2;
    h_offs.assign(runs.begin(), runs.end());
    h_tiles.assign((size_t)npairs + 1, 0);
    int64_t tiles = 0;
    for (int q = 0; q < npairs; ++q) {
      h_tiles[(size_t)q] = tiles;
      tiles += ceil_div(runs[(size_t)2 * q + 2] - runs[(size_t)2 * q], kMergeTile);
    }
    HB_CUDA_TRY(cudaMemcpyAsync(d_offs.ptr, h_offs.data(), h_offs.size() * 8, cudaMemcpyHostToDevice, s));
    HB_CUDA_TRY(cudaMemcpyAsync(d_tiles.ptr, h_tiles.data(), h_tiles.size() * 8, cudaMemcpyHostToDevice, s));
    if (tiles > 0) {
      if (pay)
        merge_round_kernel<K, true><<<(int)tiles, kMergeThreads, 0, s>>>(src_k, src_v, dst_k, dst_v, d_offs.as<int64_t>(),
                                                                        d_tiles.as<int64_t>(), npairs);
      else
        merge_round_kernel<K, false><<<(int)tiles, kMergeThreads, 0, s>>>(src_k, nullptr, dst_k, nullptr,
                                                                         d_offs.as<int64_t>(), d_tiles.as<int64_t>(), npairs);
      HB_TRY(check_launch());
    }
    if (m % 2) {  // odd run out: carried over unchanged
      const int64_t lo = runs[(size_t)m - 1], hi = runs[(size_t)m];
      if (hi > lo) {
        int64_t blocks = ceil_div(hi - lo, 256);
        if (blocks > (int64_t)di.sms * 8) blocks = (int64_t)di.sms * 8;
        if (pay) copy_run_kernel<K, true><<<(int)blocks, 256, 0, s>>>(src_k, src_v, dst_k, dst_v, lo, hi);
        else copy_run_kernel<K, false><<<(int)blocks, 256, 0, s>>>(src_k, nullptr, dst_k, nullptr, lo, hi);
        HB_TRY(check_launch());
      }
    }
    // the synchronisation point for h_offs/h_tiles reuse: the copies above are
    // stream-ordered but read host memory asynchronously only when pinned;
    // pageable sources are copied before cudaMemcpyAsync returns
    std::vector<int64_t> next;
    for (int q = 0; q < m; q += 2) next.push_back(runs[(size_t)q]);
    next.push_back(runs[(size_t)m]);
    runs.swap(next);
    src_k = dst_k;
    src_v = dst_v;
  }
  return HB_OK;
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hb_partition_nnz(const void* row_ptr, int ptr_code, int64_t row0, int64_t row1, int32_t parts,
                                int64_t* bounds_out, int flags, void* stream) {
  HB_CHECK_ARG(ptr_code == HB_I32 || ptr_code == HB_I64, "row_ptr must be int32 or int64");
  HB_CHECK_ARG(parts >= 1 && parts <= 65536, "parts out of range");
  HB_CHECK_ARG(0 <= row0 && row0 <= row1, "bad row range");
  HB_CHECK_ARG(row_ptr && bounds_out, "NULL pointer");
  const bool dev = flags & HB_DEVICE_PTRS;
  cudaStream_t s = as_stream(stream);
  const size_t pe = ptr_code == HB_I32 ? 4 : 8;
  DevBuf d_rp, d_b;
  // host row_ptr: only the [row0, row1] window is needed
  const char* base = (const char*)row_ptr + (dev ? 0 : (size_t)row0 * pe);
  HB_TRY(stage_in(&d_rp, base, (size_t)(row1 - row0 + 1) * pe, dev, s));
  const int64_t off = dev ? 0 : row0;  // window offset applied on the host side
  HB_TRY(alloc(&d_b, (size_t)(parts + 1) * 8, s));
  const int threads = 128;
  const int blocks = (int)ceil_div(parts + 1, threads);
  if (ptr_code == HB_I32)
    partition_nnz_kernel<int32_t><<<blocks, threads, 0, s>>>(d_rp.as<int32_t>(), row0 - off, row1 - off, parts, d_b.as<int64_t>());
  else
    partition_nnz_kernel<int64_t><<<blocks, threads, 0, s>>>(d_rp.as<int64_t>(), row0 - off, row1 - off, parts, d_b.as<int64_t>());
  HB_TRY(check_launch());
  HB_CUDA_TRY(cudaMemcpyAsync(bounds_out, d_b.ptr, (size_t)(parts + 1) * 8, cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaStreamSynchronize(s));
  for (int k = 0; k <= parts; ++k) bounds_out[k] += off;
  return HB_OK;
}

extern "C" int hb_scatter_perm(const void* src, int64_t n, int elem_bytes, const void* perm, int perm_code, void* dst,
                               int flags, void* stream) {
  HB_CHECK_ARG(elem_bytes == 4 || elem_bytes == 8, "elem_bytes must be 4 or 8");
  HB_CHECK_ARG(perm_code == HB_I32 || perm_code == HB_I64, "perm must be int32 or int64");
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_scatter_perm works on device arrays");
  HB_CHECK_ARG(n >= 0, "n must be >= 0");
  if (n == 0) return HB_OK;
  DeviceInfo di;
  HB_TRY(device_info(&di));
  cudaStream_t s = as_stream(stream);
  int64_t blocks = ceil_div(n, 256);
  if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
  if (elem_bytes == 8 && perm_code == HB_I32)
    scatter_perm_kernel<uint64_t, int32_t><<<(int)blocks, 256, 0, s>>>((const uint64_t*)src, n, (const int32_t*)perm, (uint64_t*)dst);
  else if (elem_bytes == 8)
    scatter_perm_kernel<uint64_t, int64_t><<<(int)blocks, 256, 0, s>>>((const uint64_t*)src, n, (const int64_t*)perm, (uint64_t*)dst);
  else if (perm_code == HB_I32)
    scatter_perm_kernel<uint32_t, int32_t><<<(int)blocks, 256, 0, s>>>((const uint32_t*)src, n, (const int32_t*)perm, (uint32_t*)dst);
  else
    scatter_perm_kernel<uint32_t, int64_t><<<(int)blocks, 256, 0, s>>>((const uint32_t*)src, n, (const int64_t*)perm, (uint32_t*)dst);
  return finish(flags, s);
}

extern "C" int hb_merge_runs(const void* keys, int key_code, const uint32_t* vals, int64_t n, const int64_t* offsets,
                             int32_t nruns, void* keys_out, uint32_t* vals_out, int flags, void* stream) {
  HB_CHECK_ARG(key_code == HB_U32 || key_code == HB_I32 || key_code == HB_U64 || key_code == HB_I64,
               "keys must be u32/i32/u64/i64");
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_merge_runs works on device arrays");
  HB_CHECK_ARG(nruns >= 1 && offsets, "need at least one run");
  HB_CHECK_ARG(offsets[0] == 0 && offsets[nruns] == n, "run offsets must span [0, n)");
  for (int r = 0; r < nruns; ++r) HB_CHECK_ARG(offsets[r] <= offsets[r + 1], "run offsets must be non-decreasing");
  HB_CHECK_ARG(keys_out != keys, "keys_out must not alias keys");
  HB_CHECK_ARG(!vals || (vals_out && vals_out != vals), "vals_out must be given and must not alias vals");
  if (n == 0) return HB_OK;
  cudaStream_t s = as_stream(stream);
  int rc;
  switch (key_code) {
    case HB_U32: rc = merge_runs<uint32_t>((const uint32_t*)keys, vals, n, offsets, nruns, (uint32_t*)keys_out, vals_out, s); break;
    case HB_I32: rc = merge_runs<int32_t>((const int32_t*)keys, vals, n, offsets, nruns, (int32_t*)keys_out, vals_out, s); break;
    case HB_U64: rc = merge_runs<uint64_t>((const uint64_t*)keys, vals, n, offsets, nruns, (uint64_t*)keys_out, vals_out, s); break;
    default: rc = merge_runs<int64_t>((const int64_t*)keys, vals, n, offsets, nruns, (int64_t*)keys_out, vals_out, s); break;
  }
  if (rc != HB_OK) return rc;
  return finish(flags, s);
}
