// hist.cu — privatised shared-memory histogram (replaces
// HistogramWorkload.run_part, reference kernels_regular.py:149-154).
//
// Design:
//  * HBM-bound streaming read: every thread issues UNROLL independent 16-byte
//    `ld.global.nc.L1::no_allocate` loads before touching shared memory (16
//    per round: 0.97-1.0 of the measured copy peak from 2^31 bytes up).  Grid = SMs x CTAs/SM
//    (persistent, grid-stride over 16-byte vectors).
//  * Privatisation: for bin_count <= 256 each CTA owns 32 sub-histograms laid
//    out LANE-STRIPED, word = bin*32 + lane, so the 32 shared-memory atomics
//    of one warp instruction always land in 32 distinct banks (conflict-free
//    for any data, including the all-equal adversary); warps of the CTA share
//    the copies through the atomic unit.  Each CTA then folds its 32 copies and
//    issues one 64-bit global atomic per bin (warp-aggregated merge).
//  * uint8 input with bin_count < 256 counts all 256 values and checks the
//    rows >= bin_count afterwards: no per-element domain test in the hot loop.
//  * Wider element types test the domain per element (the reference's
//    ValueError, kernels_regular.py:137-138) and raise a device flag.
//  * bin_count > 256: one CTA-shared copy (dynamic smem, <= 49152 bins).
#include <stdlib.h>

#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace hb {
namespace {

constexpr int kStripes = 32;         // sub-histograms per CTA (one per lane)
constexpr int kThreads = 512;        // 16 warps
constexpr int kUnroll = 16;          // 16-byte loads per thread per round (4: 176.4 us at 2^30, 8: 172.8, 16: 172.1)
constexpr int kMaxSharedBins = 49152;

template <typename T>
__device__ __forceinline__ bool in_domain(T v, uint32_t bins) {
  if constexpr (sizeof(T) == 1 && !((T)-1 < 0)) {
    return true;  // uint8 rows >= bins are checked after the fold
  } else if constexpr ((T)-1 < 0) {
    return v >= 0 && (uint64_t)v < bins;
  } else {
    return (uint64_t)v < bins;
  }
}

// Add one element to the lane-striped sub-histograms.
template <typename T, bool CHECK>
__device__ __forceinline__ void put_striped(uint32_t* s, T v, uint32_t bins, uint32_t lane,
                                            uint32_t& bad) {
  if (CHECK && !in_domain<T>(v, bins)) {
    bad++;
    return;
  }
  atomicAdd(&s[((uint32_t)v << 5) | lane], 1u);
}

template <bool CHECK>
__device__ __forceinline__ void put_vec_u8(uint32_t* s, uint4 q, uint32_t lane) {
  // __byte_perm(w, 0, 0x4440|k) = byte k of w zero-extended: one PRMT per element.
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t b = __byte_perm(w[j], 0, 0x4440 | k);
      atomicAdd(&s[(b << 5) | lane], 1u);
    }
  }
}

template <typename T, bool CHECK>
__device__ __forceinline__ void put_vec(uint32_t* s, uint4 q, uint32_t bins, uint32_t lane,
                                        uint32_t& bad) {
  if constexpr (sizeof(T) == 1 && !((T)-1 < 0)) {
    put_vec_u8<CHECK>(s, q, lane);
  } else {
    constexpr int E = 16 / sizeof(T);
    T e[E];
    memcpy(e, &q, 16);
#pragma unroll
    for (int k = 0; k < E; ++k) put_striped<T, CHECK>(s, e[k], bins, lane, bad);
  }
}

// bins <= 256: lane-striped privatised histogram.
// Per-stream scratch of the striped kernel: acc[0..255] bin sums, acc[256]
// out-of-domain count, ticket = CTAs done.  Invariant between calls: all
// zero.  The last CTA to finish publishes acc into the caller's bins (set or
// add), the domain-error count into *err_out, and zeroes acc and the ticket
// again — so a call needs no memset and no allocation (calls on one stream
// are ordered; each stream has its own scratch).
struct HistScratch {
  unsigned long long acc[257];
  unsigned int ticket;
  unsigned int err_out;
};

template <typename T, bool CHECK>
__global__ void __launch_bounds__(kThreads)
    hist_striped_kernel(const T* __restrict__ data, int64_t head, int64_t nvec, int64_t n,
                        uint32_t bins, unsigned long long* __restrict__ out,
                        HistScratch* __restrict__ sc, bool accumulate) {
  __shared__ uint32_t s[256 * kStripes];
  const uint32_t lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256 * kStripes; i += blockDim.x) s[i] = 0;
  __syncthreads();

  uint32_t bad = 0;
  const uint4* vec = reinterpret_cast<const uint4*>(data + head);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // main body: kUnroll loads in flight, then the shared-memory updates
  for (; i + (kUnroll - 1) * stride < nvec; i += kUnroll * stride) {
    uint4 q[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) q[u] = ldg_stream_v4(vec + i + u * stride);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) put_vec<T, CHECK>(s, q[u], bins, lane, bad);
  }
  for (; i < nvec; i += stride) put_vec<T, CHECK>(s, ldg_stream_v4(vec + i), bins, lane, bad);

  // unaligned head and ragged tail (< 16 bytes each), scalar
  if (blockIdx.x == 0) {
    constexpr int E = 16 / sizeof(T);
    const int64_t tail0 = head + nvec * E;
    for (int64_t j = threadIdx.x; j < head; j += blockDim.x)
      put_striped<T, CHECK || sizeof(T) != 1>(s, data[j], bins, lane, bad);
    for (int64_t j = tail0 + threadIdx.x; j < n; j += blockDim.x)
      put_striped<T, CHECK || sizeof(T) != 1>(s, data[j], bins, lane, bad);
  }
  if (bad) atomicAdd(&sc->acc[256], (unsigned long long)bad);
  __syncthreads();

  // fold the 32 stripes of each bin; rotate the start so the 32 threads of a
  // warp read 32 different banks
  for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x) {
    uint32_t sum = 0;
#pragma unroll 8
    for (uint32_t j = 0; j < kStripes; ++j) sum += s[(b << 5) | ((j + b) & 31)];
    if (sum) atomicAdd(&sc->acc[b < bins ? b : 256], (unsigned long long)sum);  // b >= bins: uint8 value >= bin_count
  }
  // the last CTA publishes and restores the all-zero scratch
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (uint32_t b = threadIdx.x; b < 257; b += blockDim.x) {
    const unsigned long long v = atomicExch(&sc->acc[b], 0ull);
    if (b < bins) out[b] = accumulate ? out[b] + v : v;
    else if (b == 256) sc->err_out = (unsigned int)v;
  }
  if (threadIdx.x == 0) sc->ticket = 0;
}

// bins > 256: one CTA-shared copy in dynamic shared memory.
template <typename T>
__global__ void __launch_bounds__(kThreads)
    hist_shared_kernel(const T* __restrict__ data, int64_t n, uint32_t bins,
                       unsigned long long* __restrict__ out, unsigned int* __restrict__ err) {
  extern __shared__ uint32_t sh[];
  for (uint32_t i = threadIdx.x; i < bins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    T v = data[i];
    if (in_domain<T>(v, bins)) atomicAdd(&sh[(uint32_t)v], 1u);
    else bad++;
  }
  if (bad) atomicAdd(err, bad);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < bins; b += blockDim.x)
    if (sh[b]) atomicAdd(out + b, (unsigned long long)sh[b]);
}

// the scratch of (current device, stream), created zeroed on first use
int hist_scratch(cudaStream_t s, HistScratch** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, HistScratch*> table;
  int dev = 0;
  HB_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = table.find({dev, s});
  if (it != table.end()) {
    *out = it->second;
    return HB_OK;
  }
  HistScratch* p = nullptr;
  HB_CUDA_TRY(cudaMalloc(&p, sizeof(HistScratch)));
  HB_CUDA_TRY(cudaMemset(p, 0, sizeof(HistScratch)));  // synchronous: zero before any use
  table[{dev, s}] = p;
  *out = p;
  return HB_OK;
}

template <typename T>
int launch_striped(const void* data, int64_t n, uint32_t bins, unsigned long long* out, bool accumulate,
                   HistScratch* sc, cudaStream_t s) {
  DeviceInfo di;
  HB_TRY(device_info(&di));
  const T* d = reinterpret_cast<const T*>(data);
  constexpr int E = 16 / sizeof(T);
  const uintptr_t addr = reinterpret_cast<uintptr_t>(d);
  int64_t head = (int64_t)(((16 - (addr & 15)) & 15) / sizeof(T));
  if (addr % sizeof(T) != 0) {
    set_error("histogram input is not aligned to its element size");
    return HB_EINVAL;
  }
  if (head > n) head = n;
  const int64_t nvec = (n - head) / E;
  int64_t blocks = ceil_div(nvec, (int64_t)kThreads * kUnroll);
  const int64_t cap = (int64_t)di.sms * 4;  // 4 CTAs x 32 KB smem per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const bool u8 = sizeof(T) == 1 && !((T)-1 < 0);
  if (u8 || bins == 0) {
    hist_striped_kernel<T, false><<<(int)blocks, kThreads, 0, s>>>(d, head, nvec, n, bins, out, sc, accumulate);
  } else {
    hist_striped_kernel<T, true><<<(int)blocks, kThreads, 0, s>>>(d, head, nvec, n, bins, out, sc, accumulate);
  }
  return check_launch();
}

template <typename T>
int launch_hist(const void* data, int64_t n, uint32_t bins, unsigned long long* out,
                unsigned int* err, cudaStream_t s) {
  DeviceInfo di;
  HB_TRY(device_info(&di));
  if (n == 0) return HB_OK;
  const T* d = reinterpret_cast<const T*>(data);
  {
    size_t smem = (size_t)bins * 4;
    HB_CUDA_TRY(cudaFuncSetAttribute(hist_shared_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    int per_sm = smem <= 48 * 1024 ? 4 : (smem <= 100 * 1024 ? 2 : 1);
    int64_t blocks = ceil_div(n, (int64_t)kThreads * 8);
    if (blocks > (int64_t)di.sms * per_sm) blocks = (int64_t)di.sms * per_sm;
    hist_shared_kernel<T><<<(int)blocks, kThreads, smem, s>>>(d, n, bins, out, err);
  }
  return check_launch();
}

size_t dtype_size(int dtype) {
  switch (dtype) {
    case HB_U8: case HB_I8: return 1;
    case HB_U16: case HB_I16: return 2;
    case HB_U32: case HB_I32: return 4;
    case HB_U64: case HB_I64: return 8;
    default: return 0;
  }
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hb_hist(const void* data, int dtype, int64_t n, int32_t bin_count,
                       uint64_t* bins_out, int flags, void* stream) {
  const size_t es = dtype_size(dtype);
  HB_CHECK_ARG(es != 0, "unsupported histogram element type code %d", dtype);
  HB_CHECK_ARG(n >= 0, "n must be >= 0");
  HB_CHECK_ARG(bin_count >= 1, "bin_count must be >= 1");
  HB_CHECK_ARG(bin_count <= kMaxSharedBins, "bin_count %d exceeds the supported %d", bin_count,
               kMaxSharedBins);
  HB_CHECK_ARG(bins_out != nullptr, "bins_out is NULL");
  HB_CHECK_ARG(n == 0 || data != nullptr, "data is NULL");
  const bool dev = flags & HB_DEVICE_PTRS;
  HB_CHECK_ARG(dev || !(flags & HB_ASYNC), "HB_ASYNC requires device pointers");
  cudaStream_t s = as_stream(stream);

  DevBuf in, out, err;
  HB_TRY(stage_in(&in, data, (size_t)n * es, dev, s));
  HB_TRY(stage_out(&out, bins_out, (size_t)bin_count * 8, dev, s));
  auto* o = out.as<unsigned long long>();
  const bool accumulate_dev = dev && (flags & HB_ACCUMULATE);
  int rc = HB_OK;
  HistScratch* sc = nullptr;
  if (bin_count <= 256 && n > 0) {
    // striped kernel: bins set (or added) and the domain count published by
    // its last CTA through the stream's scratch — no memset, no allocation
    HB_TRY(hist_scratch(s, &sc));
    switch (dtype) {
      case HB_U8: rc = launch_striped<uint8_t>(in.ptr, n, bin_count, o, accumulate_dev, sc, s); break;
      case HB_I8: rc = launch_striped<int8_t>(in.ptr, n, bin_count, o, accumulate_dev, sc, s); break;
      case HB_U16: rc = launch_striped<uint16_t>(in.ptr, n, bin_count, o, accumulate_dev, sc, s); break;
      case HB_I16: rc = launch_striped<int16_t>(in.ptr, n, bin_count, o, accumulate_dev, sc, s); break;
      case HB_U32: rc = launch_striped<uint32_t>(in.ptr, n, bin_count, o, accumulate_dev, sc, s); break;
      case HB_I32: rc = launch_striped<int32_t>(in.ptr, n, bin_count, o, accumulate_dev, sc, s); break;
      case HB_U64: rc = launch_striped<uint64_t>(in.ptr, n, bin_count, o, accumulate_dev, sc, s); break;
      default: rc = launch_striped<int64_t>(in.ptr, n, bin_count, o, accumulate_dev, sc, s); break;
    }
  } else {
    if (!accumulate_dev) HB_CUDA_TRY(cudaMemsetAsync(out.ptr, 0, (size_t)bin_count * 8, s));
    // domain-error counter: only read back when the call is synchronous
    HB_TRY(alloc(&err, 4, s));
    HB_CUDA_TRY(cudaMemsetAsync(err.ptr, 0, 4, s));
    auto* e = err.as<unsigned int>();
    switch (dtype) {
      case HB_U8: rc = launch_hist<uint8_t>(in.ptr, n, bin_count, o, e, s); break;
      case HB_I8: rc = launch_hist<int8_t>(in.ptr, n, bin_count, o, e, s); break;
      case HB_U16: rc = launch_hist<uint16_t>(in.ptr, n, bin_count, o, e, s); break;
      case HB_I16: rc = launch_hist<int16_t>(in.ptr, n, bin_count, o, e, s); break;
      case HB_U32: rc = launch_hist<uint32_t>(in.ptr, n, bin_count, o, e, s); break;
      case HB_I32: rc = launch_hist<int32_t>(in.ptr, n, bin_count, o, e, s); break;
      case HB_U64: rc = launch_hist<uint64_t>(in.ptr, n, bin_count, o, e, s); break;
      default: rc = launch_hist<int64_t>(in.ptr, n, bin_count, o, e, s); break;
    }
  }
  if (rc != HB_OK) return rc;
  if (flags & HB_ASYNC) return check_launch();

  unsigned int bad = 0;
  uint64_t* host_tmp = nullptr;
  if (!dev) {
    host_tmp = (flags & HB_ACCUMULATE) ? (uint64_t*)malloc((size_t)bin_count * 8) : bins_out;
    if (!host_tmp) { set_error("host allocation failed"); return HB_ENOMEM; }
    HB_CUDA_TRY(cudaMemcpyAsync(host_tmp, out.ptr, (size_t)bin_count * 8, cudaMemcpyDeviceToHost, s));
  }
  if (sc) HB_CUDA_TRY(cudaMemcpyAsync(&bad, &sc->err_out, 4, cudaMemcpyDeviceToHost, s));
  else if (err.ptr) HB_CUDA_TRY(cudaMemcpyAsync(&bad, err.ptr, 4, cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaStreamSynchronize(s));
  if (!dev && (flags & HB_ACCUMULATE)) {
    for (int32_t b = 0; b < bin_count; ++b) bins_out[b] += host_tmp[b];
    free(host_tmp);
  }
  if (bad) {
    set_error("element outside bin domain (%u elements)", bad);
    return HB_EINVAL;
  }
  return HB_OK;
}
