// runtime.cu — error state, device info cache, staging buffers, generators.
#include <stdarg.h>

#include <mutex>

#include "common.cuh"

namespace hb {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

static std::mutex g_info_mu;
static DeviceInfo g_info[64];

int device_info(DeviceInfo* out) {
  int dev = 0;
  HB_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) {
    set_error("device id %d out of range", dev);
    return HB_ECUDA;
  }
  std::lock_guard<std::mutex> lk(g_info_mu);
  DeviceInfo& d = g_info[dev];
  if (d.id != dev) {
    HB_CUDA_TRY(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    int optin = 0;
    HB_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    d.smem_optin = (size_t)optin;
    // Keep freed stream-ordered allocations cached in the pool: staging buffers
    // of host-pointer calls are then reused instead of re-mapped every call.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    d.id = dev;
  }
  *out = d;
  return HB_OK;
}

int alloc(DevBuf* b, size_t bytes, cudaStream_t s) {
  b->bytes = bytes;
  b->stream = s;
  b->owned = true;
  if (bytes == 0) return HB_OK;
  DeviceInfo di;
  HB_TRY(device_info(&di));  // ensures the pool threshold is set
  HB_CUDA_TRY(cudaMallocAsync(&b->ptr, bytes, s));
  return HB_OK;
}

int stage_in(DevBuf* b, const void* src, size_t bytes, bool device, cudaStream_t s) {
  if (device) {
    b->ptr = const_cast<void*>(src);
    b->bytes = bytes;
    b->owned = false;
    return HB_OK;
  }
  HB_TRY(alloc(b, bytes, s));
  if (bytes) HB_CUDA_TRY(cudaMemcpyAsync(b->ptr, src, bytes, cudaMemcpyHostToDevice, s));
  return HB_OK;
}

int stage_out(DevBuf* b, void* dst, size_t bytes, bool device, cudaStream_t s) {
  if (device) {
    b->ptr = dst;
    b->bytes = bytes;
    b->owned = false;
    return HB_OK;
  }
  return alloc(b, bytes, s);
}

int copy_out(void* dst, const DevBuf& b, size_t bytes, bool device, cudaStream_t s) {
  if (device || bytes == 0) return HB_OK;
  HB_CUDA_TRY(cudaMemcpyAsync(dst, b.ptr, bytes, cudaMemcpyDeviceToHost, s));
  return HB_OK;
}

int check_launch() {
  HB_CUDA_TRY(cudaGetLastError());
  return HB_OK;
}

int finish(int flags, cudaStream_t s) {
  HB_TRY(check_launch());
  if (!(flags & HB_ASYNC)) HB_CUDA_TRY(cudaStreamSynchronize(s));
  return HB_OK;
}

// ------------------------------------------------------------------ generators
template <int KIND>
__global__ void gen_splitmix_kernel(uint64_t seed, uint64_t k0, int64_t n, uint64_t bound,
                                    void* __restrict__ out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t z = splitmix64_at(seed, k0 + (uint64_t)i + 1);
    if (KIND == HB_GEN_RAW) reinterpret_cast<uint64_t*>(out)[i] = z;
    if (KIND == HB_GEN_LOW8) reinterpret_cast<uint8_t*>(out)[i] = (uint8_t)(z & 255u);
    if (KIND == HB_GEN_HI32) reinterpret_cast<uint32_t*>(out)[i] = (uint32_t)(z >> 32);
    if (KIND == HB_GEN_MOD) reinterpret_cast<int64_t*>(out)[i] = (int64_t)(z % bound);
  }
}

}  // namespace hb

using namespace hb;

extern "C" {

int hb_version(void) { return 1; }

const char* hb_last_error(void) { return g_last_error.c_str(); }

int hb_device_count(int* count) {
  *count = 0;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    cudaGetLastError();
    *count = 0;
    return HB_OK;
  }
  HB_CUDA_TRY(e);
  return HB_OK;
}

int hb_sm_count(int* count) {
  DeviceInfo di;
  HB_TRY(device_info(&di));
  *count = di.sms;
  return HB_OK;
}

int hb_stream_sync(void* stream) {
  HB_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  HB_CUDA_TRY(cudaGetLastError());
  return HB_OK;
}

int hb_trim(void) {
  int dev = 0;
  HB_CUDA_TRY(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  HB_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  HB_CUDA_TRY(cudaDeviceSynchronize());
  HB_CUDA_TRY(cudaMemPoolTrimTo(pool, 0));
  return HB_OK;
}

int hb_gen_splitmix(uint64_t seed, uint64_t k0, int64_t n, int kind, uint64_t bound, void* out,
                    void* stream) {
  HB_CHECK_ARG(n >= 0, "n must be >= 0");
  HB_CHECK_ARG(kind >= HB_GEN_RAW && kind <= HB_GEN_MOD, "unknown generator kind %d", kind);
  HB_CHECK_ARG(kind != HB_GEN_MOD || bound > 0, "bound must be > 0");
  if (n == 0) return HB_OK;
  DeviceInfo di;
  HB_TRY(device_info(&di));
  cudaStream_t s = as_stream(stream);
  int threads = 256;
  int64_t blocks = ceil_div(n, threads);
  if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
  switch (kind) {
    case HB_GEN_RAW: gen_splitmix_kernel<HB_GEN_RAW><<<(int)blocks, threads, 0, s>>>(seed, k0, n, bound, out); break;
    case HB_GEN_LOW8: gen_splitmix_kernel<HB_GEN_LOW8><<<(int)blocks, threads, 0, s>>>(seed, k0, n, bound, out); break;
    case HB_GEN_HI32: gen_splitmix_kernel<HB_GEN_HI32><<<(int)blocks, threads, 0, s>>>(seed, k0, n, bound, out); break;
    default: gen_splitmix_kernel<HB_GEN_MOD><<<(int)blocks, threads, 0, s>>>(seed, k0, n, bound, out); break;
  }
  return check_launch();
}

}  // extern "C"
