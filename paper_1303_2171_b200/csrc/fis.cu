// fis.cu — the reference's fractional-independent-set list reduction on the
// GPU (kernels_irregular.py:396-428) and its sublist-head selection
// (:431-448), so list_rank_with_stats returns the reference's ListRankStats
// exactly (fis_rounds, round_sizes, reduced_size, removed_total,
// sublist_count).  The ranks themselves come from hb_list_rank (they do not
// depend on the reduction).
//
// Round r: bit(i) = splitmix64 draw i+1 of mix_seed(seed, r), & 1.
//   1. flags:  removable[p] = p != head && bit(p) && (succ[p] < 0 || !bit(succ[p]))
//              for every live p (read-only: the reference evaluates the whole
//              round on the round-start list);
//   2. splice: for every live p whose successor s is removable,
//              succ[p] = succ[s] (race-free: s never splices in the same round,
//              because its successor has bit 0);
//   3. compact the live list, order-preserving (block counts → one-CTA scan
//              of the counts → block scan + scatter), so the survivors come out
//              in node-index order — the order the reference draws its sublist
//              heads in.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace hb {
namespace {

constexpr int kCT = 256;         // compaction CTA
constexpr int kCItems = 16;      // items per thread
constexpr int kCTile = kCT * kCItems;

__device__ __forceinline__ uint32_t rbit(uint64_t rs, int64_t i) {
  return (uint32_t)(splitmix64_at(rs, (uint64_t)i + 1) & 1ull);
}

__global__ void fis_init_kernel(const int64_t* __restrict__ s64, const int32_t* __restrict__ s32,
                                int64_t n, int32_t* __restrict__ succ, int32_t* __restrict__ live) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    succ[i] = s64 ? (int32_t)s64[i] : s32[i];
    live[i] = (int32_t)i;
  }
}

__global__ void fis_flags_kernel(const int32_t* __restrict__ live, int64_t m,
                                 const int32_t* __restrict__ succ, int64_t head, uint64_t rs,
                                 uint8_t* __restrict__ removable) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = live[k];
    const int32_t s = succ[p];
    const bool rm = p != head && rbit(rs, p) && (s < 0 || !rbit(rs, s));
    removable[p] = rm;
  }
}

__global__ void fis_splice_kernel(const int32_t* __restrict__ live, int64_t m,
                                  int32_t* __restrict__ succ, const uint8_t* __restrict__ removable) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = live[k];
    const int32_t s = succ[p];
    if (s >= 0 && removable[s]) succ[p] = succ[s];
  }
}

// order-preserving compaction of `live` keeping !removable
__global__ void __launch_bounds__(kCT) compact_count_kernel(const int32_t* __restrict__ live, int64_t m,
                                                            const uint8_t* __restrict__ removable,
                                                            int32_t* __restrict__ counts) {
  const int64_t base = (int64_t)blockIdx.x * kCTile;
  int c = 0;
#pragma unroll
  for (int i = 0; i < kCItems; ++i) {
    const int64_t k = base + i * kCT + threadIdx.x;
    if (k < m) c += !removable[live[k]];
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ int ws[kCT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kCT / 32; ++w) t += ws[w];
    counts[blockIdx.x] = t;
  }
}

// exclusive scan of block counts in one CTA (nb <= 1024 * 64); total → *total
__global__ void __launch_bounds__(1024) compact_scan_kernel(int32_t* __restrict__ counts, int64_t nb,
                                                            int64_t* __restrict__ total) {
  const int per = (int)((nb + 1023) / 1024);
  const int64_t a = (int64_t)threadIdx.x * per;
  int64_t sum = 0;
  for (int i = 0; i < per; ++i)
    if (a + i < nb) sum += counts[a + i];
  // block-wide exclusive scan of the per-thread sums
  __shared__ int64_t ws[32];
  int64_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    int64_t v = ws[threadIdx.x];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (threadIdx.x >= o) v += y;
    }
    ws[threadIdx.x] = v;
  }
  __syncthreads();
  int64_t run = x - sum + ((threadIdx.x >> 5) ? ws[(threadIdx.x >> 5) - 1] : 0);
  for (int i = 0; i < per; ++i)
    if (a + i < nb) {
      const int32_t c = counts[a + i];
      counts[a + i] = (int32_t)run;
      run += c;
    }
  if (threadIdx.x == 1023) *total = run;
}

__global__ void __launch_bounds__(kCT) compact_write_kernel(const int32_t* __restrict__ live, int64_t m,
                                                            const uint8_t* __restrict__ removable,
                                                            const int32_t* __restrict__ offsets,
                                                            int32_t* __restrict__ out) {
  const int64_t base = (int64_t)blockIdx.x * kCTile;
  __shared__ int ws[kCT / 32];
  int run = offsets[blockIdx.x];
  // rows of kCT items keep the input order: row i covers [base + i*kCT, +kCT)
  for (int i = 0; i < kCItems; ++i) {
    const int64_t k = base + i * kCT + threadIdx.x;
    int32_t v = 0;
    bool keep = false;
    if (k < m) {
      v = live[k];
      keep = !removable[v];
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) ws[warp] = __popc(bal);
    __syncthreads();
    int before = 0, row = 0;
    for (int w = 0; w < kCT / 32; ++w) {
      const int c = ws[w];
      if (w < warp) before += c;
      row += c;
    }
    if (keep) out[run + before + __popc(bal & ((1u << lane) - 1u))] = v;
    run += row;
    __syncthreads();
  }
}

// sublist heads: survivors (dense index k) whose draw of mix_seed(seed,0x5EED)
// is below `thr` are candidates for the s-1 smallest draws
__global__ void topk_candidates_kernel(int64_t m, uint64_t rs, uint64_t thr,
                                       unsigned long long* __restrict__ cand,
                                       unsigned int* __restrict__ count, unsigned int cap) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t d = splitmix64_at(rs, (uint64_t)k + 1);
    if (d < thr) {
      const unsigned int slot = atomicAdd(count, 1u);
      if (slot < cap) {
        cand[2 * slot] = d;
        cand[2 * slot + 1] = (unsigned long long)k;
      }
    }
  }
}

uint64_t host_mix_seed(uint64_t seed, uint64_t salt) {
  // rng.py:54-57: splitmix64((seed ^ (salt * MIX2)) mod 2^64)[1]
  const uint64_t st = (seed ^ (salt * 0x94D049BB133111EBull)) + 0x9E3779B97F4A7C15ull;
  uint64_t z = st;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hb_list_fis_stats(const void* succ, int succ_code, int64_t n, int64_t head,
                                 uint64_t seed, int32_t sublists, int64_t* round_sizes,
                                 int32_t round_cap, int64_t* stats, int flags, void* stream) {
  HB_CHECK_ARG(succ_code == HB_I32 || succ_code == HB_I64, "succ must be int32 or int64");
  HB_CHECK_ARG(n >= 1 && n < (1ll << 31), "n out of range");
  HB_CHECK_ARG(head >= 0 && head < n, "head out of range");
  HB_CHECK_ARG(stats && round_sizes && round_cap >= 0, "NULL output");
  const bool dev = flags & HB_DEVICE_PTRS;
  cudaStream_t s = as_stream(stream);
  DeviceInfo di;
  HB_TRY(device_info(&di));
  if (n == 1) {  // :486-487
    stats[0] = 0; stats[1] = 1; stats[2] = 0; stats[3] = 1;
    return HB_OK;
  }
  // target = max(int(n / log2 n), 2) if n > 2 else 2 (:488), in the reference's fp64 arithmetic
  int64_t target = 2;
  if (n > 2) {
    const double t = (double)n / std::log2((double)n);
    target = std::max<int64_t>((int64_t)t, 2);
  }
  const size_t se = succ_code == HB_I32 ? 4 : 8;
  DevBuf d_in, d_succ, live[2], rem, counts, total, cand, ccount;
  HB_TRY(stage_in(&d_in, succ, (size_t)n * se, dev, s));
  HB_TRY(alloc(&d_succ, (size_t)n * 4, s));
  HB_TRY(alloc(&live[0], (size_t)n * 4, s));
  HB_TRY(alloc(&live[1], (size_t)n * 4, s));
  HB_TRY(alloc(&rem, (size_t)n, s));
  const int64_t max_blocks = ceil_div(n, kCTile);
  HB_TRY(alloc(&counts, (size_t)max_blocks * 4, s));
  HB_TRY(alloc(&total, 8, s));
  int64_t g = ceil_div(n, 256);
  if (g > (int64_t)di.sms * 16) g = (int64_t)di.sms * 16;
  fis_init_kernel<<<(int)g, 256, 0, s>>>(succ_code == HB_I64 ? d_in.as<int64_t>() : nullptr,
                                         succ_code == HB_I32 ? d_in.as<int32_t>() : nullptr, n,
                                         d_succ.as<int32_t>(), live[0].as<int32_t>());
  HB_TRY(check_launch());

  int64_t alive = n;
  int rounds = 0;
  int cur = 0;
  while (alive > target && rounds < 1000) {
    if (rounds < round_cap) round_sizes[rounds] = alive;
    const uint64_t rs = host_mix_seed(seed, (uint64_t)rounds);
    int64_t gb = ceil_div(alive, 256);
    if (gb > (int64_t)di.sms * 16) gb = (int64_t)di.sms * 16;
    fis_flags_kernel<<<(int)gb, 256, 0, s>>>(live[cur].as<int32_t>(), alive, d_succ.as<int32_t>(), head, rs,
                                              rem.as<uint8_t>());
    fis_splice_kernel<<<(int)gb, 256, 0, s>>>(live[cur].as<int32_t>(), alive, d_succ.as<int32_t>(),
                                               rem.as<uint8_t>());
    const int64_t nb = ceil_div(alive, kCTile);
    if (nb > 1024 * 64) {
      set_error("list too long for the single-CTA block scan");
      return HB_EINVAL;
    }
    compact_count_kernel<<<(int)nb, kCT, 0, s>>>(live[cur].as<int32_t>(), alive, rem.as<uint8_t>(),
                                                 counts.as<int32_t>());
    compact_scan_kernel<<<1, 1024, 0, s>>>(counts.as<int32_t>(), nb, total.as<int64_t>());
    compact_write_kernel<<<(int)nb, kCT, 0, s>>>(live[cur].as<int32_t>(), alive, rem.as<uint8_t>(),
                                                 counts.as<int32_t>(), live[cur ^ 1].as<int32_t>());
    HB_TRY(check_launch());
    int64_t next = 0;
    HB_CUDA_TRY(cudaMemcpyAsync(&next, total.ptr, 8, cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    ++rounds;
    cur ^= 1;
    alive = next;
  }
  if (alive > target) {
    set_error("independent-set reduction failed to converge");
    return HB_ESTRUCT;
  }

  // sublist heads (:444-448): the s-1 survivors with the smallest draws of
  // mix_seed(seed, 0x5EED), in survivor (= node index) order, plus the head
  const int64_t sh = std::max<int64_t>(1, std::min<int64_t>(sublists, alive));
  int64_t used = 1;
  if (sh - 1 > 0) {
    const uint64_t rs = host_mix_seed(seed, 0x5EED);
    const unsigned int cap = 1u << 16;
    HB_TRY(alloc(&cand, (size_t)cap * 16, s));
    HB_TRY(alloc(&ccount, 4, s));
    double frac = std::min(1.0, 8.0 * (double)sh / (double)alive);
    std::vector<unsigned long long> hc;
    unsigned int got = 0;
    while (true) {
      const uint64_t thr = frac >= 1.0 ? UINT64_MAX : (uint64_t)(frac * 18446744073709551615.0);
      HB_CUDA_TRY(cudaMemsetAsync(ccount.ptr, 0, 4, s));
      int64_t gb = ceil_div(alive, 256);
      if (gb > (int64_t)di.sms * 16) gb = (int64_t)di.sms * 16;
      topk_candidates_kernel<<<(int)gb, 256, 0, s>>>(alive, rs, thr, cand.as<unsigned long long>(),
                                                       ccount.as<unsigned int>(), cap);
      HB_TRY(check_launch());
      HB_CUDA_TRY(cudaMemcpyAsync(&got, ccount.ptr, 4, cudaMemcpyDeviceToHost, s));
      HB_CUDA_TRY(cudaStreamSynchronize(s));
      if (got > cap) { frac /= 4.0; continue; }
      if ((int64_t)got >= sh - 1 || frac >= 1.0) break;
      frac = std::min(1.0, frac * 4.0);
    }
    hc.resize((size_t)got * 2);
    HB_CUDA_TRY(cudaMemcpyAsync(hc.data(), cand.ptr, (size_t)got * 16, cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<std::pair<unsigned long long, unsigned long long>> v;
    for (unsigned int i = 0; i < got; ++i) v.push_back({hc[2 * i], hc[2 * i + 1]});
    std::sort(v.begin(), v.end());  // (draw, index): the stable argsort order
    // dense indices of the chosen survivors → node ids: survivors are live[cur] in index order
    std::vector<int32_t> nodes((size_t)(sh - 1));
    bool head_chosen = false;
    for (int64_t i = 0; i < sh - 1; ++i) {
      int32_t node = 0;
      HB_CUDA_TRY(cudaMemcpyAsync(&node, live[cur].as<int32_t>() + v[(size_t)i].second, 4,
                                  cudaMemcpyDeviceToHost, s));
      HB_CUDA_TRY(cudaStreamSynchronize(s));
      if (node == head) head_chosen = true;
    }
    used = (sh - 1) + (head_chosen ? 0 : 1);
  }
  stats[0] = rounds;
  stats[1] = alive;
  stats[2] = n - alive;
  stats[3] = used;
  return HB_OK;
}
