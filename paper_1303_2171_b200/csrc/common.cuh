// common.cuh — shared plumbing for libhb200.so: error reporting, stream-ordered
// staging buffers for host-pointer calls, launch geometry, PTX load helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <functional>
#include <string>

#include "../../include/hb200.h"

namespace hb {

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);

#define HB_CUDA_TRY(expr)                                                            \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      ::hb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return _e == cudaErrorMemoryAllocation ? HB_ENOMEM : HB_ECUDA;                 \
    }                                                                                \
  } while (0)

#define HB_TRY(expr)            \
  do {                          \
    int _rc = (expr);           \
    if (_rc != HB_OK) return _rc; \
  } while (0)

#define HB_CHECK_ARG(cond, ...)      \
  do {                               \
    if (!(cond)) {                   \
      ::hb::set_error(__VA_ARGS__);  \
      return HB_EINVAL;              \
    }                                \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------------ device info
struct DeviceInfo {
  int id = -1;
  int sms = 0;
  size_t smem_optin = 0;
};
int device_info(DeviceInfo* out);  // cached per device

// ------------------------------------------------------------------ buffers
// A device buffer that is either borrowed (caller passed a device pointer)
// or owned (stream-ordered allocation from the device's default mem pool,
// whose release threshold we raise so repeated calls reuse memory).
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  bool owned = false;
  cudaStream_t stream = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (owned && ptr) cudaFreeAsync(ptr, stream);
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(ptr); }
};

int alloc(DevBuf* b, size_t bytes, cudaStream_t s);
// Stage a caller buffer: borrow it when `device`, else allocate + H2D copy.
int stage_in(DevBuf* b, const void* src, size_t bytes, bool device, cudaStream_t s);
// Output buffer: borrow when `device`, else allocate (no copy).
int stage_out(DevBuf* b, void* dst, size_t bytes, bool device, cudaStream_t s);
int copy_out(void* dst, const DevBuf& b, size_t bytes, bool device, cudaStream_t s);
// host <-> device for caller buffers: pinned → cudaMemcpyAsync; pageable →
// pinned double buffer + multi-threaded memcpy (returns with D2H data landed)
int copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);
int copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s);
int finish(int flags, cudaStream_t s);  // sync unless HB_ASYNC, surface errors
// D2H of a device buffer through the pinned stage: fn(stage, offset, len)
// runs on each landed chunk (in order) while the next chunk's DMA is in flight.
int d2h_visit(const void* src, size_t bytes, cudaStream_t s,
              const std::function<void(const char*, size_t, size_t)>& fn);
// A pinned host buffer (one 32 MB stage) borrowed from the stager free list,
// with its device-mapped address, so a kernel can store results straight
// into host memory (UVA) — no separate D2H.  Returned to the list on scope exit.
struct PinnedScratch {
  void* lease = nullptr;
  char* host = nullptr;
  void* dev = nullptr;
  PinnedScratch() = default;
  PinnedScratch(const PinnedScratch&) = delete;
  PinnedScratch& operator=(const PinnedScratch&) = delete;
  ~PinnedScratch();
};
int pinned_scratch(PinnedScratch* out, size_t bytes);  // HB_EINVAL when bytes > one stage
// true (and the device-mapped address) when `host` is page-locked host memory
bool device_view(void* host, void** dev);
// fn(0..n-1) on the process-wide host thread pool (one region at a time).
void host_parallel(int n, const std::function<void(int)>& fn);
// the same on a second pool reserved for the host-share (DeviceA) kernels
void host_kernel_parallel(int n, const std::function<void(int)>& fn, int max_threads);
int host_threads();
// Host-buffer row filters: H2D of input rows (on a side stream), the kernel
// of each row chunk on `s` (launch(a, b) = absolute rows [a, b)), D2H of the
// chunk's output rows on another side stream; returns with the output landed.
int row_pipeline(const char* in_host, size_t in_row, int in0, int in1, int radius, int row0, int row1,
                 char* out_host, size_t out_row, char* d_in, char* d_out, cudaStream_t s,
                 const std::function<int(int, int)>& launch);
int check_launch();

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint4 ldg_stream_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// splitmix64 finaliser of draw k (1-based) of stream `seed` (rng.py:45-51).
__host__ __device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t k) {
  uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// mbarrier + bulk-copy (TMA 1-D) helpers: one elected thread arms a barrier
// with the expected byte count and issues cp.async.bulk; consumers wait on
// the barrier's phase parity.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(a), "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* smem, const void* g, uint32_t bytes, uint64_t* bar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(g), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s_hint(void* smem, const void* g, uint32_t bytes, uint64_t* bar,
                                                  uint64_t policy) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(d), "l"(g), "r"(bytes), "r"(b), "l"(policy) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// List ranking's level-1 log (csrc/listrank.cu): 8-byte slots in 32-slot,
// 256-byte-aligned chunks.  Node entry = node << 32 | offset in its sublist;
// marker = (kLogMark | sublist) << 32 (every chunk opens with one, every walk
// start inside a chunk writes one); padding = kLogEmpty << 32.
constexpr uint32_t kLogMark = 0x80000000u;
constexpr uint32_t kLogEmpty = 0xffffffffu;
constexpr int kLogChunkSlots = 32;
// One warp holds one chunk, lane = slot (all 32 lanes call this): the slot
// as a packed (rank << 32 | node) pair, rank = prefix[sublist] + offset;
// markers and padding become key 0xffffffff, rank 0.
__device__ __forceinline__ uint64_t log_slot_pair(uint64_t e, const int64_t* __restrict__ prefix) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t le = (2u << lane) - 1u;  // lanes <= me
  const uint32_t hi = (uint32_t)(e >> 32);
  const bool mark = (hi & kLogMark) && hi != kLogEmpty;
  const uint32_t mb = __ballot_sync(0xffffffffu, mark);
  const int src = 31 - __clz(mb & le);
  const uint32_t j = __shfl_sync(0xffffffffu, hi & ~kLogMark, src < 0 ? 0 : src);
  if (hi & kLogMark) return 0xffffffffull;
  return ((uint64_t)(uint32_t)(prefix[j] + (int64_t)(uint32_t)e) << 32) | hi;
}

}  // namespace hb
