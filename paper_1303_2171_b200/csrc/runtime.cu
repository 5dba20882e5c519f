// runtime.cu — error state, device info cache, staging buffers, generators.
#include <stdarg.h>
#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

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

// ------------------------------------------------------------------ host transfers
// Pageable host buffers (plain numpy arrays) cross PCIe through a pinned
// double buffer: the DMA of chunk i+1 overlaps the multi-threaded memcpy of
// chunk i between the pinned stage and the pageable array (which also
// spreads the first-touch page faults of a fresh output over threads).  The
// driver's own pageable path is single-threaded (~2-10 GB/s); pinned buffers
// go straight to cudaMemcpyAsync.
namespace {

// minimal fork-join pool: run(fn, n) calls fn(0..n-1) on up to `size` threads
class HostPool {
 public:
  // pool 0: transfer staging (memcpy / un-permute), pool 1: the host-share
  // (DeviceA) kernels — separate, so a GPU side's copies never queue behind
  // the concurrent host side of the same run_workshared
  static HostPool& get(int which = 0) {
    // never destroyed: its detached workers wait on cv_ until the process
    // ends, and destroying a condition variable with waiters blocks in glibc
    static HostPool* p[2] = {new HostPool(), new HostPool()};
    return *p[which & 1];
  }
  int size() const { return (int)workers_.size() + 1; }
  // n tasks, claimed dynamically by at most max_threads threads (the caller
  // included)
  void run(const std::function<void(int)>& fn, int n, int max_threads = 1 << 30) {
    std::unique_lock<std::mutex> lk(run_mu_);  // one parallel region at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      next_ = 0;
      n_ = n;
      done_ = 0;
      slots_ = std::max(0, std::min(max_threads, n) - 1);
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return done_ == n_; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    // the pageable side of a transfer is bound by first-touch page zeroing of
    // fresh output arrays (~10 GB/s per thread), so use every core
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int n = std::max(0, std::min(32, hw) - 1);
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    for (auto& t : workers_) t.detach();
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen && fn_ != nullptr; });
        seen = gen_;
        if (slots_ <= 0) continue;  // the region has its threads
        --slots_;
      }
      work();
    }
  }
  void work() {
    for (;;) {
      int i;
      const std::function<void(int)>* fn;
      {
        std::lock_guard<std::mutex> g(mu_);
        if (fn_ == nullptr || next_ >= n_) return;
        i = next_++;
        fn = fn_;
      }
      (*fn)(i);
      std::lock_guard<std::mutex> g(mu_);
      if (++done_ == n_) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int next_ = 0, n_ = 0, done_ = 0, slots_ = 0;
  uint64_t gen_ = 0;
};

constexpr size_t kStageChunk = (size_t)32 << 20;  // bytes per pinned stage
constexpr size_t kPinnedDirect = (size_t)4 << 20;  // smaller copies: plain cudaMemcpyAsync

struct Stager {
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
};

// Process-wide free list: a call borrows a stager (allocated once, pinned
// memory is expensive to allocate) and returns it when its copy is done.
// Calls come from short-lived Python pool threads, so per-thread buffers
// would be re-allocated (and leaked) on every call.
std::mutex g_stage_mu;
std::vector<Stager*> g_stage_free;

struct StagerLease {
  Stager* st = nullptr;
  ~StagerLease() {
    if (st) {
      std::lock_guard<std::mutex> g(g_stage_mu);
      g_stage_free.push_back(st);
    }
  }
};

int stager(StagerLease* lease) {
  {
    std::lock_guard<std::mutex> g(g_stage_mu);
    if (!g_stage_free.empty()) {
      lease->st = g_stage_free.back();
      g_stage_free.pop_back();
      return HB_OK;
    }
  }
  Stager* st = new Stager();
  for (int i = 0; i < 2; ++i) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&st->buf[i]), kStageChunk, cudaHostAllocDefault) != cudaSuccess ||
        cudaEventCreateWithFlags(&st->ev[i], cudaEventDisableTiming) != cudaSuccess) {
      set_error("pinned staging buffer: %s", cudaGetErrorString(cudaGetLastError()));
      return HB_ECUDA;  // (a partially built stager is leaked; this only happens when pinned memory runs out)
    }
  }
  lease->st = st;
  return HB_OK;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void par_memcpy(char* dst, const char* src, size_t bytes) {
  HostPool& pool = HostPool::get();
  const int parts = std::max(1, std::min(pool.size() * 2, (int)(bytes >> 20)));
  pool.run([&](int k) {
    const size_t a = bytes * (size_t)k / (size_t)parts, b = bytes * (size_t)(k + 1) / (size_t)parts;
    memcpy(dst + a, src + a, b - a);
  }, parts);
}

}  // namespace

int copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return HB_OK;
  if (bytes <= kPinnedDirect || is_pinned(src)) {
    HB_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return HB_OK;
  }
  StagerLease lease;
  HB_TRY(stager(&lease));
  Stager* st = lease.st;
  const char* in = reinterpret_cast<const char*>(src);
  char* out = reinterpret_cast<char*>(dst);
  for (size_t off = 0, i = 0; off < bytes; off += kStageChunk, ++i) {
    const size_t len = std::min(kStageChunk, bytes - off);
    const int b = (int)(i & 1);
    HB_CUDA_TRY(cudaEventSynchronize(st->ev[b]));  // the stage's previous DMA is done
    par_memcpy(st->buf[b], in + off, len);
    HB_CUDA_TRY(cudaMemcpyAsync(out + off, st->buf[b], len, cudaMemcpyHostToDevice, s));
    HB_CUDA_TRY(cudaEventRecord(st->ev[b], s));
  }
  // the stager goes back to the free list: its last DMAs must be done first
  HB_CUDA_TRY(cudaEventSynchronize(st->ev[0]));
  HB_CUDA_TRY(cudaEventSynchronize(st->ev[1]));
  return HB_OK;
}

int copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return HB_OK;
  if (bytes <= kPinnedDirect || is_pinned(dst)) {
    HB_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    return HB_OK;
  }
  StagerLease lease;
  HB_TRY(stager(&lease));
  Stager* st = lease.st;
  const char* in = reinterpret_cast<const char*>(src);
  char* out = reinterpret_cast<char*>(dst);
  const size_t n = (bytes + kStageChunk - 1) / kStageChunk;
  auto issue = [&](size_t i) -> int {
    const size_t off = i * kStageChunk, len = std::min(kStageChunk, bytes - off);
    HB_CUDA_TRY(cudaMemcpyAsync(st->buf[i & 1], in + off, len, cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaEventRecord(st->ev[i & 1], s));
    return HB_OK;
  };
  HB_TRY(issue(0));
  for (size_t i = 0; i < n; ++i) {
    if (i + 1 < n) HB_TRY(issue(i + 1));  // next chunk's DMA overlaps this chunk's memcpy
    HB_CUDA_TRY(cudaEventSynchronize(st->ev[i & 1]));
    const size_t off = i * kStageChunk, len = std::min(kStageChunk, bytes - off);
    par_memcpy(out + off, st->buf[i & 1], len);
  }
  return HB_OK;
}

void host_parallel(int n, const std::function<void(int)>& fn) { HostPool::get().run(fn, n); }

PinnedScratch::~PinnedScratch() {
  if (lease) {
    std::lock_guard<std::mutex> g(g_stage_mu);
    g_stage_free.push_back(static_cast<Stager*>(lease));
  }
}

int pinned_scratch(PinnedScratch* out, size_t bytes) {
  if (bytes > kStageChunk) return HB_EINVAL;
  StagerLease l;
  HB_TRY(stager(&l));
  out->lease = l.st;
  out->host = l.st->buf[0];
  l.st = nullptr;  // ownership moves to `out`
  return device_view(out->host, &out->dev) ? HB_OK : HB_ECUDA;
}

bool device_view(void* host, void** dev) {
  if (!is_pinned(host)) return false;
  if (cudaHostGetDevicePointer(dev, host, 0) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return true;
}

void host_kernel_parallel(int n, const std::function<void(int)>& fn, int max_threads) {
  HostPool::get(1).run(fn, n, max_threads);
}

int host_threads() { return HostPool::get().size(); }

int d2h_visit(const void* src, size_t bytes, cudaStream_t s,
              const std::function<void(const char*, size_t, size_t)>& fn) {
  if (bytes == 0) return HB_OK;
  StagerLease lease;
  HB_TRY(stager(&lease));
  Stager* st = lease.st;
  const char* in = reinterpret_cast<const char*>(src);
  const size_t n = (bytes + kStageChunk - 1) / kStageChunk;
  auto issue = [&](size_t i) -> int {
    const size_t off = i * kStageChunk, len = std::min(kStageChunk, bytes - off);
    HB_CUDA_TRY(cudaMemcpyAsync(st->buf[i & 1], in + off, len, cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaEventRecord(st->ev[i & 1], s));
    return HB_OK;
  };
  HB_TRY(issue(0));
  for (size_t i = 0; i < n; ++i) {
    if (i + 1 < n) HB_TRY(issue(i + 1));  // next chunk's DMA overlaps this chunk's visit
    HB_CUDA_TRY(cudaEventSynchronize(st->ev[i & 1]));
    const size_t off = i * kStageChunk;
    fn(st->buf[i & 1], off, std::min(kStageChunk, bytes - off));
  }
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
  return copy_h2d(b->ptr, src, bytes, s);
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
  return copy_d2h(dst, b.ptr, bytes, s);
}

// Row-strip pipeline for host-buffer filter calls.  Three streams: input
// rows cross PCIe on `is`, the kernel of chunk c runs on `s` once its rows
// (and halo) have landed, and chunk c's output rows go back on `cs` as soon
// as its kernel is done — so the D2H of chunk c overlaps the kernel of chunk
// c+1, and H2D runs beside D2H (PCIe is full duplex).  Always drains both
// side streams before returning, so the caller's stream-ordered buffers
// (freed on `s`) are not released under a copy in flight.
static const int kMaxChunks = [] {
  const char* e = getenv("HB_PIPE_CHUNKS");
  return e ? std::max(1, atoi(e)) : 32;  // measured 16 / 32 / 64: 40.3 / 39.9 / 40.1 ms per 2 GiB result
}();

int row_pipeline(const char* in_host, size_t in_row, int in0, int in1, int radius, int row0, int row1,
                 char* out_host, size_t out_row, char* d_in, char* d_out, cudaStream_t s,
                 const std::function<int(int, int)>& launch) {
  const int rows = row1 - row0;
  if (rows <= 0) return HB_OK;
  const size_t out_bytes = (size_t)rows * out_row;
  const int chunks = (int)std::min<size_t>({(size_t)kMaxChunks, (size_t)rows, std::max<size_t>(1, out_bytes >> 25)});
  const int per = (rows + chunks - 1) / chunks;
  if (chunks == 1) {  // small strips: in, kernel, out on `s`
    HB_TRY(copy_h2d(d_in, in_host, (size_t)(in1 - in0) * in_row, s));
    HB_TRY(launch(row0, row1));
    return copy_d2h(out_host, d_out, out_bytes, s);
  }
  struct Side {
    cudaStream_t is = nullptr, cs = nullptr;
    std::vector<cudaEvent_t> in_ev, k_ev;
    ~Side() {
      if (is) cudaStreamSynchronize(is);
      if (cs) cudaStreamSynchronize(cs);
      for (cudaEvent_t e : in_ev) if (e) cudaEventDestroy(e);
      for (cudaEvent_t e : k_ev) if (e) cudaEventDestroy(e);
      if (is) cudaStreamDestroy(is);
      if (cs) cudaStreamDestroy(cs);
    }
  } side;
  HB_CUDA_TRY(cudaStreamCreateWithFlags(&side.is, cudaStreamNonBlocking));
  HB_CUDA_TRY(cudaStreamCreateWithFlags(&side.cs, cudaStreamNonBlocking));
  side.in_ev.assign(chunks, nullptr);
  side.k_ev.assign(chunks, nullptr);
  for (int c = 0; c < chunks; ++c) {
    HB_CUDA_TRY(cudaEventCreateWithFlags(&side.in_ev[c], cudaEventDisableTiming));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&side.k_ev[c], cudaEventDisableTiming));
  }
  // the device buffers were allocated on `s`: the side streams start after that
  HB_CUDA_TRY(cudaEventRecord(side.k_ev[0], s));
  HB_CUDA_TRY(cudaStreamWaitEvent(side.is, side.k_ev[0], 0));
  HB_CUDA_TRY(cudaStreamWaitEvent(side.cs, side.k_ev[0], 0));
  // chunk c's kernel needs input rows [in0, need_c) resident
  int loaded = in0;
  for (int c = 0; c < chunks; ++c) {
    const int a = row0 + c * per, b = std::min(row1, a + per);
    const int need = c + 1 == chunks ? in1 : std::min(in1, b + radius);
    if (need > loaded) {
      HB_TRY(copy_h2d(d_in + (size_t)(loaded - in0) * in_row, in_host + (size_t)(loaded - in0) * in_row,
                      (size_t)(need - loaded) * in_row, side.is));
      loaded = need;
    }
    HB_CUDA_TRY(cudaEventRecord(side.in_ev[c], side.is));
    HB_CUDA_TRY(cudaStreamWaitEvent(s, side.in_ev[c], 0));
    if (a < b) HB_TRY(launch(a, b));
    HB_CUDA_TRY(cudaEventRecord(side.k_ev[c], s));
  }
  for (int c = 0; c < chunks; ++c) {
    const int a = row0 + c * per, b = std::min(row1, a + per);
    if (a >= b) continue;
    HB_CUDA_TRY(cudaStreamWaitEvent(side.cs, side.k_ev[c], 0));
    HB_TRY(copy_d2h(out_host + (size_t)(a - row0) * out_row, d_out + (size_t)(a - row0) * out_row,
                    (size_t)(b - a) * out_row, side.cs));
  }
  HB_CUDA_TRY(cudaStreamSynchronize(side.cs));
  return check_launch();
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

int hb_set_device(int device) {
  HB_CUDA_TRY(cudaSetDevice(device));
  return HB_OK;
}

int hb_buf_alloc(size_t bytes, void** out) {
  HB_CHECK_ARG(out != nullptr, "NULL out");
  *out = nullptr;
  if (bytes == 0) return HB_OK;
  HB_CUDA_TRY(cudaMalloc(out, bytes));
  return HB_OK;
}

int hb_buf_free(void* buf) {
  if (buf) HB_CUDA_TRY(cudaFree(buf));
  return HB_OK;
}

int hb_buf_upload(void* dst_device, const void* src_host, size_t bytes, int flags, void* stream) {
  HB_CHECK_ARG(bytes == 0 || (dst_device && src_host), "NULL pointer");
  if (bytes == 0) return HB_OK;
  cudaStream_t s = hb::as_stream(stream);
  HB_TRY(hb::copy_h2d(dst_device, src_host, bytes, s));
  return hb::finish(flags, s);
}

int hb_buf_download(void* dst_host, const void* src_device, size_t bytes, int flags, void* stream) {
  HB_CHECK_ARG(bytes == 0 || (dst_host && src_device), "NULL pointer");
  if (bytes == 0) return HB_OK;
  cudaStream_t s = hb::as_stream(stream);
  HB_TRY(hb::copy_d2h(dst_host, src_device, bytes, s));
  return hb::finish(flags, s);
}

int hb_stream_create(void** out) {
  HB_CHECK_ARG(out != nullptr, "NULL out");
  cudaStream_t s = nullptr;
  HB_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = s;
  return HB_OK;
}

int hb_stream_destroy(void* stream) {
  if (stream) HB_CUDA_TRY(cudaStreamDestroy(hb::as_stream(stream)));
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
