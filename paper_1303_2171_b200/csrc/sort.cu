// sort.cu — LSD radix sort, onesweep style (replaces the DeviceB side of
// sample_sort_hybrid, reference kernels_regular.py:239-310; the sorted
// multiset is unique, so the output equals the reference's bit for bit; the
// optional uint32 payload makes it the STABLE argsort).
//
//   1. digit_hist_kernel: one read of the keys builds the 256-bucket
//      histogram of every 8-bit digit position at once (privatised smem
//      counters, 8 copies per bucket).
//   2. per non-trivial digit position, onesweep_kernel (one launch):
//      * tiles of THREADS*ITEMS keys, tile ids taken from an atomic counter
//        (a tile's predecessors are always resident or done: forward progress);
//      * warp-striped coalesced loads; stable warp-level ranking with eight
//        __ballot_sync per key row (warp multi-split) into per-warp smem
//        counters; cross-warp exclusive scan per digit;
//      * decoupled look-back per digit (one thread per digit): the tile
//        publishes its digit counts (AGGREGATE), walks back over predecessor
//        tiles until it finds an INCLUSIVE prefix, then publishes its own
//        inclusive prefix — 32-bit words, 2 flag bits + 30 count bits, so
//        one relaxed store publishes flag and count together;
//      * keys (and payload) are re-ordered by digit in shared memory and
//        written out in digit runs (coalesced segments).
//   A digit position whose histogram has a single bucket is skipped (a stable
//   pass over one bucket is the identity) — int64 keys below 2^32 sort in 4
//   passes, a constant array in 0.
#include <stdlib.h>

#include <mutex>
#include <utility>

#include "common.cuh"

namespace hb {
namespace {

constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1;

template <typename K>
struct SortCfg;
template <>
struct SortCfg<uint32_t> {
  static constexpr int kThreads = 512, kItems = 12, kPasses = 4;
};
template <>
struct SortCfg<uint64_t> {
  static constexpr int kThreads = 512, kItems = 8, kPasses = 8;
};

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lanes of the warp holding the same 8-bit digit: peers &= ~(ballot_b ^ m_b),
// m_b = all-ones when bit b of my digit is set — four instructions per bit
// (LOP3 → predicate, VOTE, SELP, LOP3 0x90).
__device__ __forceinline__ uint32_t match_digit8(uint32_t d) {
  uint32_t peers = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t, bal, m;\n\t"
        "and.b32 t, %1, %2;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "vote.sync.ballot.b32 bal, p, 0xffffffff;\n\t"
        "selp.b32 m, 0xffffffff, 0, p;\n\t"
        "lop3.b32 %0, %0, bal, m, 0x90;\n\t}"
        : "+r"(peers)
        : "r"(d), "r"(1u << b));
  }
  return peers;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, K flip, int shift) {
  return (uint32_t)((key ^ flip) >> shift) & 255u;
}

// ------------------------------------------------------------------ 1. histogram
template <typename K>
__global__ void __launch_bounds__(512)
    digit_hist_kernel(const K* __restrict__ keys, int64_t n, K flip, uint32_t* __restrict__ hist) {
  constexpr int P = SortCfg<K>::kPasses;
  constexpr int C = 32 / P;  // copies per bucket (32 KB of counters)
  __shared__ uint32_t s[P * 256 * C];
  for (int i = threadIdx.x; i < P * 256 * C; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const uint32_t copy = threadIdx.x & (C - 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const K k = keys[i] ^ flip;
#pragma unroll
    for (int p = 0; p < P; ++p) atomicAdd(&s[((p * 256) + (uint32_t)((k >> (8 * p)) & 255)) * C + copy], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < P * 256; b += blockDim.x) {
    uint32_t sum = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) sum += s[b * C + ((c + b) & (C - 1))];
    if (sum) atomicAdd(hist + b, sum);
  }
}

// uint32 keys: 16-byte loads (4 keys), 4 in flight per thread, and
// LANE-STRIPED counters s[digit position][bucket][lane] (128 KB, one
// 1024-thread CTA per SM): the four atomics of a key hit 32 distinct banks
// across the warp for any data, like the 256-bin histogram kernel.
constexpr int kDh32Threads = 1024;
constexpr size_t kDh32Smem = (size_t)4 * 256 * 32 * 4;

__global__ void __launch_bounds__(kDh32Threads, 1)
    digit_hist32_kernel(const uint32_t* __restrict__ keys, int64_t n, uint32_t flip, uint32_t* __restrict__ hist) {
  extern __shared__ __align__(16) uint32_t s32[];  // [4][256][32]
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4 * 256 * 32; i += kDh32Threads) s32[i] = 0;
  __syncthreads();
  auto put = [&](uint32_t k) {
    k ^= flip;
#pragma unroll
    for (int p = 0; p < 4; ++p) atomicAdd(&s32[((p << 8) | ((k >> (8 * p)) & 255u)) * 32 + lane], 1u);
  };
  const int64_t nv = n >> 2;  // whole uint4 vectors (keys come from an aligned allocation)
  const uint4* v = reinterpret_cast<const uint4*>(keys);
  const int64_t stride = (int64_t)gridDim.x * kDh32Threads;
  int64_t i = (int64_t)blockIdx.x * kDh32Threads + threadIdx.x;
  constexpr int U = 4;
  for (; i + (U - 1) * stride < nv; i += U * stride) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = ldg_stream_v4(v + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      put(q[u].x);
      put(q[u].y);
      put(q[u].z);
      put(q[u].w);
    }
  }
  for (; i < nv; i += stride) {
    const uint4 q = ldg_stream_v4(v + i);
    put(q.x);
    put(q.y);
    put(q.z);
    put(q.w);
  }
  for (int64_t t = (nv << 2) + (int64_t)blockIdx.x * kDh32Threads + threadIdx.x; t < n; t += stride) put(keys[t]);
  __syncthreads();
  for (int b = threadIdx.x; b < 4 * 256; b += kDh32Threads) {
    uint32_t sum = 0;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) sum += s32[b * 32 + ((l + b) & 31)];
    if (sum) atomicAdd(hist + b, sum);
  }
}

// ------------------------------------------------------------------ 2. onesweep pass
// T threads x I items per tile; RANK_MATCH selects __match_any_sync (one
// MATCH per key row) instead of the eight-ballot multi-split.
template <typename K, bool HAS_V, int T, int I, bool RANK_MATCH>
__global__ void __launch_bounds__(T, 1024 / T)
    onesweep_kernel(const K* __restrict__ kin, K* __restrict__ kout, const uint32_t* __restrict__ vin,
                    uint32_t* __restrict__ vout, int64_t n, int shift, K flip,
                    const uint32_t* __restrict__ pass_hist, uint32_t* __restrict__ lookback,
                    uint32_t* __restrict__ tile_counter) {
  constexpr int W = T / 32, TILE = T * I;
  constexpr int DPT = 256 / T > 0 ? 256 / T : 1;  // digits per thread in digit-parallel phases
  __shared__ uint32_t s_whist[W][256];   // per-warp digit counters → exclusive warp offsets
  __shared__ uint32_t s_dstart[256];     // exclusive scan over digits of the tile counts
  __shared__ uint32_t s_goff[256];       // global offset of digit run minus its tile start
  __shared__ uint32_t s_gstart[256];     // global exclusive digit starts (this pass)
  __shared__ uint32_t s_scr[8];
  __shared__ uint32_t s_tile;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  K* s_keys = reinterpret_cast<K*>(s_dyn);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + TILE);
  static_assert(T >= 256 || DPT * T == 256, "digit phases need T | 256 or T >= 256");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < W * 256; i += T) (&s_whist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * TILE;
  const int valid = (int)min((int64_t)TILE, n - base);
  const K* kt = kin + base;
  const uint32_t* vt = HAS_V ? vin + base : nullptr;
  const int wbase = warp * 32 * I;

  // issue the tile's loads first; the global-start scan overlaps them
  K key[I];
  uint32_t val[I];
#pragma unroll
  for (int i = 0; i < I; ++i) {
    const int idx = wbase + i * 32 + lane;
    const bool ok = idx < valid;
    key[i] = ok ? kt[idx] : (K)(~(K)0 ^ flip);  // padding sorts last (digit 255)
    if (HAS_V) val[i] = ok ? vt[idx] : 0u;
  }
  // global digit starts: exclusive scan of this pass's histogram
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const int d = tid + q * T;
    if (d < 256) {
      const uint32_t h = pass_hist[d];
      uint32_t x = h;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      s_gstart[d] = x - h;
      if (lane == 31) s_scr[d >> 5] = x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const int d = tid + q * T;
    if (d < 256) {
      uint32_t add = 0;
      for (int g = 0; g < (d >> 5); ++g) add += s_scr[g];
      s_gstart[d] += add;
    }
  }

  // stable warp-level ranking of the I key rows
  uint32_t dig[I], rank[I];
  uint32_t* wh = s_whist[warp];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < I; ++i) {
    const uint32_t d = digit_of<K>(key[i], flip, shift);
    dig[i] = d;
    const uint32_t peers = RANK_MATCH ? __match_any_sync(0xffffffffu, d) : match_digit8(d);
    const uint32_t below = __popc(peers & lt);
    const uint32_t pre = wh[d];
    __syncwarp();
    if ((peers & ~(lt | (1u << lane))) == 0) wh[d] = pre + below + 1u;  // highest peer lane
    __syncwarp();
    rank[i] = pre + below;
  }
  __syncthreads();

  // per digit: exclusive offsets across warps, tile count, publish, look back
  uint32_t cnt[DPT], incl[DPT];
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const int d = tid + q * T;
    cnt[q] = 0;
    if (d < 256) {
      uint32_t c = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const uint32_t t = s_whist[w][d];
        s_whist[w][d] = c;
        c += t;
      }
      cnt[q] = c;
      if (tile == 0) st_relaxed(lookback + d, kFlagInc | c);
      else st_relaxed(lookback + (size_t)tile * 256 + d, kFlagAgg | c);
      uint32_t x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      incl[q] = x;
      if (lane == 31) s_scr[d >> 5] = x;
    }
  }
  __syncthreads();
  uint32_t dstart[DPT], excl[DPT];
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const int d = tid + q * T;
    dstart[q] = 0;
    excl[q] = 0;
    if (d < 256) {
      uint32_t add = 0;
      for (int g = 0; g < (d >> 5); ++g) add += s_scr[g];
      dstart[q] = incl[q] - cnt[q] + add;
      if (tile > 0) {
        int64_t t = (int64_t)tile - 1;
        uint32_t e = 0;
        while (true) {
          const uint32_t w = ld_relaxed(lookback + (size_t)t * 256 + d);
          const uint32_t flag = w & ~kCountMask;
          if (flag == 0) continue;  // predecessor still ranking: spin
          e += w & kCountMask;
          if (flag == kFlagInc) break;
          --t;
        }
        st_relaxed(lookback + (size_t)tile * 256 + d, kFlagInc | (e + cnt[q]));
        excl[q] = e;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const int d = tid + q * T;
    if (d < 256) {
      s_dstart[d] = dstart[q];
      s_goff[d] = s_gstart[d] + excl[q] - dstart[q];
    }
  }
  __syncthreads();

  // local re-order by digit (stable), then digit-run scatter
  uint32_t pos[I];
#pragma unroll
  for (int i = 0; i < I; ++i) {
    pos[i] = s_dstart[dig[i]] + s_whist[warp][dig[i]] + rank[i];
    s_keys[pos[i]] = key[i];
  }
  if (HAS_V) {
#pragma unroll
    for (int i = 0; i < I; ++i) s_vals[pos[i]] = val[i];
  }
  __syncthreads();
  for (int j = tid; j < valid; j += T) {
    const K k = s_keys[j];
    const uint32_t dst = s_goff[digit_of<K>(k, flip, shift)] + (uint32_t)j;
    kout[dst] = k;
    if (HAS_V) vout[dst] = s_vals[j];
  }
}

// ------------------------------------------------------------------ 2b. persistent onesweep
// Same pass as onesweep_kernel, but each CTA stays resident and loops over
// tiles: while tile a_i is ranked / looked back / scattered, the tile a_{i+1}
// (id taken one iteration earlier) is already streaming into the other
// shared-memory stage with cp.async, and the id of a_{i+2} is being fetched.
// Dependencies only point to smaller tile ids and every CTA handles its tiles
// in increasing order, so the smallest unfinished tile always progresses.
__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* g) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(a), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// stage a tile's keys/vals (valid elements only) into smem; 16-byte copies when aligned
template <typename K, bool HAS_V, int T, int I>
__device__ __forceinline__ void stage_tile(K* sk, uint32_t* sv, const K* kin, const uint32_t* vin,
                                           int64_t base, int valid, bool vec_ok) {
  constexpr int TILE = T * I;
  const int tid = threadIdx.x;
  if (vec_ok) {
    constexpr int KV = 16 / sizeof(K);
    const int kvec = valid / KV;
    for (int v = tid; v < kvec; v += T) cp_async16(sk + v * KV, kin + base + v * KV);
    for (int e = kvec * KV + tid; e < valid; e += T) {
      if constexpr (sizeof(K) == 4) cp_async4(sk + e, kin + base + e);
      else { cp_async4(reinterpret_cast<uint32_t*>(sk + e), reinterpret_cast<const uint32_t*>(kin + base + e));
             cp_async4(reinterpret_cast<uint32_t*>(sk + e) + 1, reinterpret_cast<const uint32_t*>(kin + base + e) + 1); }
    }
    if (HAS_V) {
      const int vvec = valid / 4;
      for (int v = tid; v < vvec; v += T) cp_async16(sv + v * 4, vin + base + v * 4);
      for (int e = vvec * 4 + tid; e < valid; e += T) cp_async4(sv + e, vin + base + e);
    }
  } else {
    for (int e = tid; e < valid; e += T) {
      if constexpr (sizeof(K) == 4) cp_async4(sk + e, kin + base + e);
      else { cp_async4(reinterpret_cast<uint32_t*>(sk + e), reinterpret_cast<const uint32_t*>(kin + base + e));
             cp_async4(reinterpret_cast<uint32_t*>(sk + e) + 1, reinterpret_cast<const uint32_t*>(kin + base + e) + 1); }
      if (HAS_V) cp_async4(sv + e, vin + base + e);
    }
  }
  (void)TILE;
  cp_async_commit();
}

template <typename K, bool HAS_V, int T, int I>
__global__ void __launch_bounds__(T, 3)
    onesweep_persist_kernel(const K* __restrict__ kin, K* __restrict__ kout,
                            const uint32_t* __restrict__ vin, uint32_t* __restrict__ vout, int64_t n,
                            int shift, K flip, const uint32_t* __restrict__ pass_hist,
                            uint32_t* __restrict__ lookback, uint32_t* __restrict__ tile_counter,
                            int64_t ntiles, int vec_ok) {
  constexpr int W = T / 32, TILE = T * I;
  static_assert(T == 256, "digit-parallel phases assume one digit per thread");
  __shared__ uint32_t s_whist[W][256];
  __shared__ uint32_t s_dstart[256];
  __shared__ uint32_t s_goff[256];
  __shared__ uint32_t s_gstart[256];
  __shared__ uint32_t s_scr[8];
  __shared__ uint32_t s_next[2];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  constexpr size_t STAGE = (size_t)TILE * sizeof(K) + (HAS_V ? (size_t)TILE * 4 : 0);
  auto stage_k = [&](int st) { return reinterpret_cast<K*>(s_dyn + st * STAGE); };
  auto stage_v = [&](int st) { return reinterpret_cast<uint32_t*>(s_dyn + st * STAGE + (size_t)TILE * sizeof(K)); };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // global digit starts (once per CTA)
  {
    const uint32_t h = pass_hist[tid];
    uint32_t x = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_gstart[tid] = x - h;
    if (lane == 31) s_scr[warp] = x;
    __syncthreads();
    uint32_t add = 0;
    for (int g = 0; g < warp; ++g) add += s_scr[g];
    s_gstart[tid] += add;
  }
  if (tid == 0) {
    s_next[0] = atomicAdd(tile_counter, 1u);
    s_next[1] = atomicAdd(tile_counter, 1u);
  }
  __syncthreads();
  uint32_t tile = s_next[0];
  uint32_t nxt = s_next[1];
  if (tile < ntiles) {
    const int64_t b0 = (int64_t)tile * TILE;
    stage_tile<K, HAS_V, T, I>(stage_k(0), stage_v(0), kin, vin, b0, (int)min((int64_t)TILE, n - b0), vec_ok);
  }
  int st = 0;
  const uint32_t lt = lanemask_lt();
  while (tile < ntiles) {
    const int64_t base = (int64_t)tile * TILE;
    const int valid = (int)min((int64_t)TILE, n - base);
    for (int i = tid; i < W * 256; i += T) (&s_whist[0][0])[i] = 0;
    cp_async_wait_all();
    __syncthreads();  // stage st landed; s_whist zeroed; s_next consumed
    // prefetch the next tile into the other stage and fetch the id after it
    if (nxt < ntiles) {
      const int64_t b1 = (int64_t)nxt * TILE;
      stage_tile<K, HAS_V, T, I>(stage_k(st ^ 1), stage_v(st ^ 1), kin, vin, b1,
                                 (int)min((int64_t)TILE, n - b1), vec_ok);
    }
    if (tid == 0) s_next[0] = atomicAdd(tile_counter, 1u);

    K* sk = stage_k(st);
    uint32_t* sv = stage_v(st);
    const int wbase = warp * 32 * I;
    K key[I];
    uint32_t val[I], dig[I], rank[I];
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const int idx = wbase + i * 32 + lane;
      const bool ok = idx < valid;
      key[i] = ok ? sk[idx] : (K)(~(K)0 ^ flip);
      if (HAS_V) val[i] = ok ? sv[idx] : 0u;
    }
    uint32_t* wh = s_whist[warp];
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const uint32_t d = digit_of<K>(key[i], flip, shift);
      dig[i] = d;
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? bal : ~bal;
      }
      const uint32_t below = __popc(peers & lt);
      const uint32_t pre = wh[d];
      __syncwarp();
      if ((peers & ~(lt | (1u << lane))) == 0) wh[d] = pre + below + 1u;
      __syncwarp();
      rank[i] = pre + below;
    }
    __syncthreads();  // all keys read from stage st (it becomes the re-order buffer)

    // digit tid: warp offsets, tile count, publish, scan, look back
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t t = s_whist[w][tid];
      s_whist[w][tid] = c;
      c += t;
    }
    if (tile == 0) st_relaxed(lookback + tid, kFlagInc | c);
    else st_relaxed(lookback + (size_t)tile * 256 + tid, kFlagAgg | c);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_scr[warp] = x;
    uint32_t excl = 0;
    if (tile > 0) {
      int64_t t = (int64_t)tile - 1;
      while (true) {
        const uint32_t w = ld_relaxed(lookback + (size_t)t * 256 + tid);
        const uint32_t flag = w & ~kCountMask;
        if (flag == 0) continue;
        excl += w & kCountMask;
        if (flag == kFlagInc) break;
        --t;
      }
      st_relaxed(lookback + (size_t)tile * 256 + tid, kFlagInc | (excl + c));
    }
    __syncthreads();
    uint32_t add = 0;
    for (int g = 0; g < warp; ++g) add += s_scr[g];
    const uint32_t dstart = x - c + add;
    s_dstart[tid] = dstart;
    s_goff[tid] = s_gstart[tid] + excl - dstart;
    const uint32_t after = s_next[0];  // id of the tile after the prefetched one
    __syncthreads();

#pragma unroll
    for (int i = 0; i < I; ++i) {
      const uint32_t p = s_dstart[dig[i]] + s_whist[warp][dig[i]] + rank[i];
      sk[p] = key[i];
      if (HAS_V) sv[p] = val[i];
    }
    __syncthreads();
    for (int j = tid; j < valid; j += T) {
      const K k = sk[j];
      const uint32_t dst = s_goff[digit_of<K>(k, flip, shift)] + (uint32_t)j;
      kout[dst] = k;
      if (HAS_V) vout[dst] = sv[j];
    }
    // rotate: the prefetched tile becomes current (the loop-top barrier
    // orders this stage's scatter before it is refilled)
    tile = nxt;
    nxt = after;
    st ^= 1;
  }
  cp_async_wait_all();
}

// ------------------------------------------------------------------ 2c. persistent onesweep, TMA bulk prefetch
// One elected thread per CTA takes the next tile id and streams that tile's
// keys/payload into the other shared-memory stage with cp.async.bulk
// (completion on an mbarrier, expect_tx bytes) while all warps work on the
// current tile.  Tile ids are taken when a tile starts (never two ahead), so
// a tile's predecessors are always current tiles of other CTAs.
template <typename K, bool HAS_V, int T, int I>
__device__ __forceinline__ void tma_stage(K* sk, uint32_t* sv, const K* kin, const uint32_t* vin,
                                          int64_t base, int valid, uint64_t* bar) {
  const uint32_t kb = (uint32_t)(valid * sizeof(K)) & ~15u;
  const uint32_t vb = HAS_V ? ((uint32_t)(valid * 4) & ~15u) : 0u;
  mbar_expect_tx(bar, kb + vb);
  if (kb) tma_bulk_g2s(sk, kin + base, kb, bar);
  if (vb) tma_bulk_g2s(sv, vin + base, vb, bar);
}

template <typename K, bool HAS_V, int T, int I>
__global__ void __launch_bounds__(T, 3)
    onesweep_tma_kernel(const K* __restrict__ kin, K* __restrict__ kout,
                        const uint32_t* __restrict__ vin, uint32_t* __restrict__ vout, int64_t n,
                        int shift, K flip, const uint32_t* __restrict__ pass_hist,
                        uint32_t* __restrict__ lookback, uint32_t* __restrict__ tile_counter,
                        int64_t ntiles) {
  constexpr int W = T / 32, TILE = T * I;
  static_assert(T == 256, "digit-parallel phases assume one digit per thread");
  __shared__ uint32_t s_whist[W][256];
  __shared__ uint32_t s_dstart[256];
  __shared__ uint32_t s_goff[256];
  __shared__ uint32_t s_gstart[256];
  __shared__ uint32_t s_scr[8];
  __shared__ uint32_t s_next;
  __shared__ __align__(8) uint64_t s_bar[2];
  extern __shared__ __align__(128) unsigned char s_dyn[];
  constexpr size_t STAGE = (size_t)TILE * sizeof(K) + (HAS_V ? (size_t)TILE * 4 : 0);
  auto stage_k = [&](int st) { return reinterpret_cast<K*>(s_dyn + st * STAGE); };
  auto stage_v = [&](int st) { return reinterpret_cast<uint32_t*>(s_dyn + st * STAGE + (size_t)TILE * sizeof(K)); };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t t0 = atomicAdd(tile_counter, 1u);
    s_next = t0;
    if (t0 < ntiles) {
      const int64_t b0 = (int64_t)t0 * TILE;
      tma_stage<K, HAS_V, T, I>(stage_k(0), stage_v(0), kin, vin, b0, (int)min((int64_t)TILE, n - b0), &s_bar[0]);
    }
  }
  {  // global digit starts (once per CTA)
    const uint32_t h = pass_hist[tid];
    uint32_t x = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_gstart[tid] = x - h;
    if (lane == 31) s_scr[warp] = x;
    __syncthreads();
    uint32_t add = 0;
    for (int g = 0; g < warp; ++g) add += s_scr[g];
    s_gstart[tid] += add;
  }
  uint32_t tile = s_next;
  uint32_t phase[2] = {0u, 0u};
  int st = 0;
  const uint32_t lt = lanemask_lt();
  while (tile < ntiles) {
    const int64_t base = (int64_t)tile * TILE;
    const int valid = (int)min((int64_t)TILE, n - base);
    for (int i = tid; i < W * 256; i += T) (&s_whist[0][0])[i] = 0;
    mbar_wait(&s_bar[st], phase[st]);
    phase[st] ^= 1u;
    __syncthreads();  // stage st landed; s_whist zeroed; previous stage fully consumed
    if (tid == 0) {  // next tile: id + bulk prefetch into the other stage
      const uint32_t nt = atomicAdd(tile_counter, 1u);
      s_next = nt;
      if (nt < ntiles) {
        const int64_t b1 = (int64_t)nt * TILE;
        tma_stage<K, HAS_V, T, I>(stage_k(st ^ 1), stage_v(st ^ 1), kin, vin, b1,
                                  (int)min((int64_t)TILE, n - b1), &s_bar[st ^ 1]);
      }
    }
    K* sk = stage_k(st);
    uint32_t* sv = stage_v(st);
    const int kvec = (int)(((uint32_t)(valid * sizeof(K)) & ~15u) / sizeof(K));
    const int vvec = (int)(((uint32_t)(valid * 4) & ~15u) / 4);
    const int wbase = warp * 32 * I;
    K key[I];
    uint32_t val[I], dig[I], rank[I];
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const int idx = wbase + i * 32 + lane;
      key[i] = idx < kvec ? sk[idx] : (idx < valid ? kin[base + idx] : (K)(~(K)0 ^ flip));
      if (HAS_V) val[i] = idx < vvec ? sv[idx] : (idx < valid ? vin[base + idx] : 0u);
    }
    uint32_t* wh = s_whist[warp];
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const uint32_t d = digit_of<K>(key[i], flip, shift);
      dig[i] = d;
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? bal : ~bal;
      }
      const uint32_t below = __popc(peers & lt);
      const uint32_t pre = wh[d];
      __syncwarp();
      if ((peers & ~(lt | (1u << lane))) == 0) wh[d] = pre + below + 1u;
      __syncwarp();
      rank[i] = pre + below;
    }
    __syncthreads();

    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t t = s_whist[w][tid];
      s_whist[w][tid] = c;
      c += t;
    }
    if (tile == 0) st_relaxed(lookback + tid, kFlagInc | c);
    else st_relaxed(lookback + (size_t)tile * 256 + tid, kFlagAgg | c);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_scr[warp] = x;
    uint32_t excl = 0;
    if (tile > 0) {
      int64_t t = (int64_t)tile - 1;
      while (true) {
        const uint32_t w = ld_relaxed(lookback + (size_t)t * 256 + tid);
        const uint32_t flag = w & ~kCountMask;
        if (flag == 0) continue;
        excl += w & kCountMask;
        if (flag == kFlagInc) break;
        --t;
      }
      st_relaxed(lookback + (size_t)tile * 256 + tid, kFlagInc | (excl + c));
    }
    __syncthreads();
    uint32_t add = 0;
    for (int g = 0; g < warp; ++g) add += s_scr[g];
    const uint32_t dstart = x - c + add;
    s_dstart[tid] = dstart;
    s_goff[tid] = s_gstart[tid] + excl - dstart;
    __syncthreads();

#pragma unroll
    for (int i = 0; i < I; ++i) {
      const uint32_t p = s_dstart[dig[i]] + s_whist[warp][dig[i]] + rank[i];
      sk[p] = key[i];
      if (HAS_V) sv[p] = val[i];
    }
    __syncthreads();
    for (int j = tid; j < valid; j += T) {
      const K k = sk[j];
      const uint32_t dst = s_goff[digit_of<K>(k, flip, shift)] + (uint32_t)j;
      kout[dst] = k;
      if (HAS_V) vout[dst] = sv[j];
    }
    // order this stage's generic-proxy accesses before the bulk copy that
    // will refill it (issued after the next loop-top barrier)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tile = s_next;
    st ^= 1;
  }
}

// ------------------------------------------------------------------ 2d. onesweep with early counts
// Critical-path restructuring of onesweep_kernel (CUB calls the idea "early
// counts"): the tile's digit counts come from per-warp shared-memory atomics
// right after the load, so the AGGREGATE is published before the ranking;
// warps 0-7 (one digit per thread) then run the look-back while warps 8-15
// already rank their keys; warps 0-7 rank after.  Ranks are warp-local
// (stable ballot multi-split); final positions = per-(warp, digit) base +
// rank.  Global digit starts come pre-scanned (scan_hist_kernel).
__global__ void scan_hist_kernel(const uint32_t* __restrict__ hist, uint32_t* __restrict__ gstart, int passes) {
  const int p = blockIdx.x;
  if (p >= passes) return;
  __shared__ uint32_t scr[8];
  const int d = threadIdx.x, lane = d & 31, warp = d >> 5;
  const uint32_t h = hist[p * 256 + d];
  uint32_t x = h;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scr[warp] = x;
  __syncthreads();
  uint32_t add = 0;
  for (int g = 0; g < warp; ++g) add += scr[g];
  gstart[p * 256 + d] = x - h + add;
}

__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <typename K, bool HAS_V, int I, int T, bool TWO_PHASE, int LBW = 1, bool MATCH = false,
          bool ATOMS_RANK = false>
__global__ void __launch_bounds__(T, 1024 / T)
    onesweep_ec_kernel(const K* __restrict__ kin, K* __restrict__ kout, const uint32_t* __restrict__ vin,
                       uint32_t* __restrict__ vout, int64_t n, int shift, K flip,
                       const uint32_t* __restrict__ gstart, uint32_t* __restrict__ lookback,
                       uint32_t* __restrict__ tile_counter) {
  constexpr int W = T / 32, TILE = T * I;
  static_assert(T > 256, "warps 8.. rank while warps 0-7 look back");
  __shared__ uint32_t s_base[W][256];   // per-warp counts → per-(warp, digit) tile positions
  __shared__ uint32_t s_run[W][256];    // warp-local running counts for the stable ranking
  __shared__ uint32_t s_goff[256];
  __shared__ uint32_t s_scr[8];
  __shared__ uint32_t s_tile;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  K* s_keys = reinterpret_cast<K*>(s_dyn);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + TILE);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < W * 256; i += T) {
    (&s_base[0][0])[i] = 0;
    (&s_run[0][0])[i] = 0;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * TILE;
  const int valid = (int)min((int64_t)TILE, n - base);
  const K* kt = kin + base;
  const uint32_t* vt = HAS_V ? vin + base : nullptr;
  const int wbase = warp * 32 * I;
  K key[I];
  uint32_t val[I], dig[I];
#pragma unroll
  for (int i = 0; i < I; ++i) {
    const int idx = wbase + i * 32 + lane;
    const bool ok = idx < valid;
    key[i] = ok ? kt[idx] : (K)(~(K)0 ^ flip);
    if (HAS_V) val[i] = ok ? vt[idx] : 0u;
  }
  uint32_t gs = 0;
  if (tid < 256) gs = gstart[tid];
  // early per-warp digit counts
#pragma unroll
  for (int i = 0; i < I; ++i) {
    dig[i] = digit_of<K>(key[i], flip, shift);
    atomicAdd(&s_base[warp][dig[i]], 1u);
  }
  __syncthreads();

  uint32_t rank[I];
  const uint32_t lt = lanemask_lt();
  auto rank_keys = [&]() {
    uint32_t* wr = s_run[warp];
    if constexpr (TWO_PHASE) {
      // all rows' peer masks first (independent → ILP), then the counter chain
      uint32_t pm[I];
#pragma unroll
      for (int i = 0; i < I; ++i) pm[i] = match_digit8(dig[i]);
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const uint32_t d = dig[i];
        const uint32_t below = __popc(pm[i] & lt);
        const uint32_t pre = wr[d];
        __syncwarp();
        if ((pm[i] & ~(lt | (1u << lane))) == 0) wr[d] = pre + below + 1u;
        __syncwarp();
        rank[i] = pre + below;
      }
    } else {
#pragma unroll
      for (int i = 0; i < I; ++i) {
        const uint32_t d = dig[i];
        if constexpr (ATOMS_RANK) {
          // one shared atomic per key: lanes of a warp that hit the same
          // counter get their old values in lane order (verified on the
          // device at first use, atoms_rank_ok), i.e. pre + below directly
          rank[i] = atomicAdd(&wr[d], 1u);
          continue;
        }
        const uint32_t peers = MATCH ? __match_any_sync(0xffffffffu, d) : match_digit8(d);
        const uint32_t below = __popc(peers & lt);
        const uint32_t pre = wr[d];
        __syncwarp();
        if ((peers & ~(lt | (1u << lane))) == 0) wr[d] = pre + below + 1u;
        __syncwarp();
        rank[i] = pre + below;
      }
    }
  };

  if (tid >= 256) {
    rank_keys();  // warps 8-15 rank while warps 0-7 publish and look back
  } else {
    const int d = tid;
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) c += s_base[w][d];
    if (tile == 0) st_relaxed(lookback + d, kFlagInc | c);
    else st_relaxed(lookback + (size_t)tile * 256 + d, kFlagAgg | c);
    // exclusive scan over digits (256 threads, named barrier 1)
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_scr[warp] = x;
    bar_named(1, 256);
    uint32_t add = 0;
    for (int g = 0; g < warp; ++g) add += s_scr[g];
    const uint32_t dstart = x - c + add;
    uint32_t run = dstart;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t t = s_base[w][d];
      s_base[w][d] = run;
      run += t;
    }
    uint32_t excl = 0;
    if (tile > 0) {
      int64_t t = (int64_t)tile - 1;
      if constexpr (LBW == 1) {
        while (true) {
          const uint32_t wv = ld_relaxed(lookback + (size_t)t * 256 + d);
          const uint32_t flag = wv & ~kCountMask;
          if (flag == 0) continue;
          excl += wv & kCountMask;
          if (flag == kFlagInc) break;
          --t;
        }
      } else {
        // windowed look-back: LBW predecessors loaded at once (independent
        // loads, one round trip), consumed in order until an inclusive
        // prefix; a not-yet-published entry stops the window and is re-read
        bool done = false;
        while (!done) {
          uint32_t wv[LBW];
#pragma unroll
          for (int j = 0; j < LBW; ++j) {
            const int64_t tj = t - j < 0 ? 0 : t - j;  // tile 0 is always inclusive
            wv[j] = ld_relaxed(lookback + (size_t)tj * 256 + d);
          }
          int used = 0;
#pragma unroll
          for (int j = 0; j < LBW; ++j) {
            if (done || used < j) continue;
            const uint32_t flag = wv[j] & ~kCountMask;
            if (flag == 0) continue;
            excl += wv[j] & kCountMask;
            used = j + 1;
            if (flag == kFlagInc) done = true;
          }
          t -= used;
        }
      }
      st_relaxed(lookback + (size_t)tile * 256 + d, kFlagInc | (excl + c));
    }
    s_goff[d] = gs + excl - dstart;
    rank_keys();
  }
  __syncthreads();

#pragma unroll
  for (int i = 0; i < I; ++i) {
    const uint32_t p = s_base[warp][dig[i]] + rank[i];
    s_keys[p] = key[i];
    if (HAS_V) s_vals[p] = val[i];
  }
  __syncthreads();
  for (int j = tid; j < valid; j += T) {
    const K k = s_keys[j];
    const uint32_t dst = s_goff[digit_of<K>(k, flip, shift)] + (uint32_t)j;
    kout[dst] = k;
    if (HAS_V) vout[dst] = s_vals[j];
  }
}

// ------------------------------------------------------------------ 2f. rank-first onesweep
// Ranking is ONE shared atomic per key: the lanes of a warp that hit the same
// per-warp digit counter get their old values in lane order — the stable
// rank (pre + lower peers) — so the eight-ballot multi-split disappears.
// This is not documented CUDA behaviour; it is verified on the device before
// first use (atoms_rank_ok below, 2^20 random rows per digit modulus) and
// the ballot kernel is used if the check fails.  After the ranking pass the
// counters hold the per-warp digit counts, so no separate counting pass is
// needed; warps 0-7 then publish, scan and look back while the rest wait.
template <typename K, bool HAS_V, int I, int T, int LBW, int MINB, bool ES = false>
__global__ void __launch_bounds__(T, MINB)
    onesweep_rf_kernel(const K* __restrict__ kin, K* __restrict__ kout, const uint32_t* __restrict__ vin,
                       uint32_t* __restrict__ vout, int64_t n, int shift, K flip,
                       const uint32_t* __restrict__ gstart, uint32_t* __restrict__ lookback,
                       uint32_t* __restrict__ tile_counter) {
  constexpr int W = T / 32, TILE = T * I;
  static_assert(T >= 256, "one look-back thread per digit");
  __shared__ uint32_t s_base[W][256];  // per-warp running counts → per-(warp, digit) tile positions
  __shared__ uint32_t s_goff[256];
  __shared__ uint32_t s_scr[8];
  __shared__ uint32_t s_tile;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  K* s_keys = reinterpret_cast<K*>(s_dyn);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + TILE);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < W * 256; i += T) (&s_base[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * TILE;
  const int valid = (int)min((int64_t)TILE, n - base);
  const K* kt = kin + base;
  const uint32_t* vt = HAS_V ? vin + base : nullptr;
  const int wbase = warp * 32 * I;
  K key[I];
  uint32_t val[I], rank[I];
#pragma unroll
  for (int i = 0; i < I; ++i) {
    const int idx = wbase + i * 32 + lane;
    const bool ok = idx < valid;
    key[i] = ok ? kt[idx] : (K)(~(K)0 ^ flip);
    if (HAS_V) val[i] = ok ? vt[idx] : 0u;
  }
  uint32_t gs = 0;
  if (tid < 256) gs = gstart[tid];
#pragma unroll
  for (int i = 0; i < I; ++i) rank[i] = atomicAdd(&s_base[warp][digit_of<K>(key[i], flip, shift)], 1u);
  __syncthreads();

  const int d = tid;  // digit of the look-back thread (tid < 256)
  uint32_t c = 0, dstart = 0;
  if (tid < 256) {
#pragma unroll
    for (int w = 0; w < W; ++w) c += s_base[w][d];
    if (tile == 0) st_relaxed(lookback + d, kFlagInc | c);
    else st_relaxed(lookback + (size_t)tile * 256 + d, kFlagAgg | c);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_scr[warp] = x;
    bar_named(1, 256);
    uint32_t add = 0;
    for (int g = 0; g < warp; ++g) add += s_scr[g];
    dstart = x - c + add;
    uint32_t run = dstart;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t t = s_base[w][d];
      s_base[w][d] = run;
      run += t;
    }
  }
  auto scatter_smem = [&]() {
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const uint32_t p = s_base[warp][digit_of<K>(key[i], flip, shift)] + rank[i];
      s_keys[p] = key[i];
      if (HAS_V) s_vals[p] = val[i];
    }
  };
  if (ES) {
    // local re-order first: the predecessors' aggregates land meanwhile, so
    // the look-back below spins less
    __syncthreads();
    scatter_smem();
  }
  if (tid < 256) {
    uint32_t excl = 0;
    if (tile > 0) {
      int64_t t = (int64_t)tile - 1;
      bool done = false;
      while (!done) {
        uint32_t wv[LBW];
#pragma unroll
        for (int j = 0; j < LBW; ++j) {
          const int64_t tj = t - j < 0 ? 0 : t - j;
          wv[j] = ld_relaxed(lookback + (size_t)tj * 256 + d);
        }
        int used = 0;
#pragma unroll
        for (int j = 0; j < LBW; ++j) {
          if (done || used < j) continue;
          const uint32_t flag = wv[j] & ~kCountMask;
          if (flag == 0) continue;
          excl += wv[j] & kCountMask;
          used = j + 1;
          if (flag == kFlagInc) done = true;
        }
        t -= used;
      }
      st_relaxed(lookback + (size_t)tile * 256 + d, kFlagInc | (excl + c));
    }
    s_goff[d] = gs + excl - dstart;
  }
  __syncthreads();
  if (!ES) {
    scatter_smem();
    __syncthreads();
  }
  for (int j = tid; j < valid; j += T) {
    const K k = s_keys[j];
    const uint32_t dst = s_goff[digit_of<K>(k, flip, shift)] + (uint32_t)j;
    kout[dst] = k;
    if (HAS_V) vout[dst] = s_vals[j];
  }
}

// u32 keys + u32 payload moved as ONE 8-byte element (key in the low half):
// PIN — the input is packed (else key and payload arrays), POUT — the output
// is packed (else split back into the two arrays).  The first live digit pass
// reads split and writes packed, the middle passes stay packed, the last one
// writes split: one 8-byte load / smem store / smem load / global store per
// element instead of two of each.
template <bool PIN, bool POUT, int I, int T, int LBW, int MINB>
__global__ void __launch_bounds__(T, MINB)
    onesweep_rfk_kernel(const void* __restrict__ kin_, void* __restrict__ kout_, const uint32_t* __restrict__ vin,
                        uint32_t* __restrict__ vout, int64_t n, int shift, uint32_t flip,
                       const uint32_t* __restrict__ gstart, uint32_t* __restrict__ lookback,
                       uint32_t* __restrict__ tile_counter) {
  constexpr int W = T / 32, TILE = T * I;
  static_assert(T >= 256, "one look-back thread per digit");
  __shared__ uint32_t s_base[W][256];  // per-warp running counts → per-(warp, digit) tile positions
  __shared__ uint32_t s_goff[256];
  __shared__ uint32_t s_scr[8];
  __shared__ uint32_t s_tile;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  uint64_t* s_el = reinterpret_cast<uint64_t*>(s_dyn);
  const uint32_t* kin = reinterpret_cast<const uint32_t*>(kin_);
  const uint64_t* ein = reinterpret_cast<const uint64_t*>(kin_);
  uint32_t* kout = reinterpret_cast<uint32_t*>(kout_);
  uint64_t* eout = reinterpret_cast<uint64_t*>(kout_);
  auto dig = [&](uint64_t e) -> uint32_t { return (((uint32_t)e ^ flip) >> shift) & 255u; };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < W * 256; i += T) (&s_base[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * TILE;
  const int valid = (int)min((int64_t)TILE, n - base);
  const int wbase = warp * 32 * I;
  uint64_t el[I];
  uint32_t rank[I];
#pragma unroll
  for (int i = 0; i < I; ++i) {
    const int idx = wbase + i * 32 + lane;
    const bool ok = idx < valid;
    if (PIN) el[i] = ok ? ein[base + idx] : (uint64_t)(~0u ^ flip);
    else el[i] = ok ? ((uint64_t)vin[base + idx] << 32) | kin[base + idx] : (uint64_t)(~0u ^ flip);
  }
  uint32_t gs = 0;
  if (tid < 256) gs = gstart[tid];
#pragma unroll
  for (int i = 0; i < I; ++i) rank[i] = atomicAdd(&s_base[warp][dig(el[i])], 1u);
  __syncthreads();

  const int d = tid;  // digit of the look-back thread (tid < 256)
  uint32_t c = 0, dstart = 0;
  if (tid < 256) {
#pragma unroll
    for (int w = 0; w < W; ++w) c += s_base[w][d];
    if (tile == 0) st_relaxed(lookback + d, kFlagInc | c);
    else st_relaxed(lookback + (size_t)tile * 256 + d, kFlagAgg | c);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_scr[warp] = x;
    bar_named(1, 256);
    uint32_t add = 0;
    for (int g = 0; g < warp; ++g) add += s_scr[g];
    dstart = x - c + add;
    uint32_t run = dstart;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t t = s_base[w][d];
      s_base[w][d] = run;
      run += t;
    }
  }
  auto scatter_smem = [&]() {
#pragma unroll
    for (int i = 0; i < I; ++i) s_el[s_base[warp][dig(el[i])] + rank[i]] = el[i];
  };
  {  // local re-order before the look-back walk (see onesweep_rf_kernel)
    // local re-order first: the predecessors' aggregates land meanwhile, so
    // the look-back below spins less
    __syncthreads();
    scatter_smem();
  }
  if (tid < 256) {
    uint32_t excl = 0;
    if (tile > 0) {
      int64_t t = (int64_t)tile - 1;
      bool done = false;
      while (!done) {
        uint32_t wv[LBW];
#pragma unroll
        for (int j = 0; j < LBW; ++j) {
          const int64_t tj = t - j < 0 ? 0 : t - j;
          wv[j] = ld_relaxed(lookback + (size_t)tj * 256 + d);
        }
        int used = 0;
#pragma unroll
        for (int j = 0; j < LBW; ++j) {
          if (done || used < j) continue;
          const uint32_t flag = wv[j] & ~kCountMask;
          if (flag == 0) continue;
          excl += wv[j] & kCountMask;
          used = j + 1;
          if (flag == kFlagInc) done = true;
        }
        t -= used;
      }
      st_relaxed(lookback + (size_t)tile * 256 + d, kFlagInc | (excl + c));
    }
    s_goff[d] = gs + excl - dstart;
  }
  __syncthreads();
  for (int j = tid; j < valid; j += T) {
    const uint64_t e = s_el[j];
    const uint32_t dst = s_goff[dig(e)] + (uint32_t)j;
    if (POUT) {
      eout[dst] = e;
    } else {
      kout[dst] = (uint32_t)e;
      vout[dst] = (uint32_t)(e >> 32);
    }
  }
}


// Persistent variant of onesweep_rfk_kernel with the next tile prefetched
// (HB_SORT_CFG=78): 2 CTAs/SM each loop over tiles claimed from the same
// in-order counter; right after a tile's elements are in registers, thread 0
// claims the NEXT tile and pulls it into shared memory with cp.async.bulk
// (one 45 KB copy packed, or keys + payload), so the loads of tile i+1 are in
// flight while tile i is ranked, looked back and scattered.  Partial tiles
// load from global directly.  Progress: every CTA finishes its tiles in claim
// order, so the smallest unfinished tile always belongs to a running CTA.
template <bool PIN, bool POUT, int I, int T, int LBW>
__global__ void __launch_bounds__(T, 2)
    onesweep_rfp_kernel(const void* __restrict__ kin_, void* __restrict__ kout_, const uint32_t* __restrict__ vin,
                        uint32_t* __restrict__ vout, int64_t n, int shift, uint32_t flip,
                        const uint32_t* __restrict__ gstart, uint32_t* __restrict__ lookback,
                        uint32_t* __restrict__ tile_counter, uint32_t ntiles) {
  constexpr int W = T / 32, TILE = T * I;
  static_assert(T >= 256, "one look-back thread per digit");
  __shared__ uint32_t s_base[W][256];
  __shared__ uint32_t s_goff[256];
  __shared__ uint32_t s_scr[8];
  __shared__ uint32_t s_next;
  __shared__ __align__(8) uint64_t s_bar;
  extern __shared__ __align__(128) unsigned char s_dyn[];
  uint64_t* s_el = reinterpret_cast<uint64_t*>(s_dyn);          // [TILE] re-order buffer
  uint64_t* s_in = s_el + TILE;                                  // [TILE] prefetched input
  const uint32_t* s_in32 = reinterpret_cast<const uint32_t*>(s_in);
  const uint32_t* kin = reinterpret_cast<const uint32_t*>(kin_);
  const uint64_t* ein = reinterpret_cast<const uint64_t*>(kin_);
  uint32_t* kout = reinterpret_cast<uint32_t*>(kout_);
  uint64_t* eout = reinterpret_cast<uint64_t*>(kout_);
  auto dig = [&](uint64_t e) -> uint32_t { return (((uint32_t)e ^ flip) >> shift) & 255u; };
  auto full = [&](uint32_t t) { return (int64_t)(t + 1) * TILE <= n; };
  auto prefetch = [&](uint32_t t) {  // thread 0: whole tile t into s_in
    const int64_t b = (int64_t)t * TILE;
    if (PIN) {
      mbar_expect_tx(&s_bar, TILE * 8);
      tma_bulk_g2s(s_in, ein + b, TILE * 8, &s_bar);
    } else {
      mbar_expect_tx(&s_bar, TILE * 8);
      tma_bulk_g2s(s_in, kin + b, TILE * 4, &s_bar);
      tma_bulk_g2s(reinterpret_cast<uint32_t*>(s_in) + TILE, vin + b, TILE * 4, &s_bar);
    }
  };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t gs = tid < 256 ? gstart[tid] : 0u;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t t = atomicAdd(tile_counter, 1u);
    s_next = t;
    if (t < ntiles && full(t)) prefetch(t);
  }
  __syncthreads();
  uint32_t phase = 0;
  const int wbase = warp * 32 * I;
  for (;;) {
    const uint32_t tile = s_next;
    if (tile >= ntiles) break;
    const int64_t base = (int64_t)tile * TILE;
    const int valid = (int)min((int64_t)TILE, n - base);
    const bool staged = full(tile);
    for (int i = tid; i < W * 256; i += T) (&s_base[0][0])[i] = 0;
    if (staged) {
      mbar_wait(&s_bar, phase);
      phase ^= 1u;
    }
    uint64_t el[I];
    uint32_t rank[I];
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const int idx = wbase + i * 32 + lane;
      if (staged) {
        el[i] = PIN ? s_in[idx] : (((uint64_t)s_in32[TILE + idx] << 32) | s_in32[idx]);
      } else {
        const bool ok = idx < valid;
        if (PIN) el[i] = ok ? ein[base + idx] : (uint64_t)(~0u ^ flip);
        else el[i] = ok ? ((uint64_t)vin[base + idx] << 32) | kin[base + idx] : (uint64_t)(~0u ^ flip);
      }
    }
    __syncthreads();  // s_in consumed, s_base zeroed
    if (tid == 0) {   // claim the next tile and start its loads now
      const uint32_t t = atomicAdd(tile_counter, 1u);
      s_next = t;
      if (t < ntiles && full(t)) {
        fence_proxy_async_smem();
        prefetch(t);
      }
    }
#pragma unroll
    for (int i = 0; i < I; ++i) rank[i] = atomicAdd(&s_base[warp][dig(el[i])], 1u);
    __syncthreads();

    const int d = tid;
    uint32_t c = 0, dstart = 0;
    if (tid < 256) {
#pragma unroll
      for (int w = 0; w < W; ++w) c += s_base[w][d];
      if (tile == 0) st_relaxed(lookback + d, kFlagInc | c);
      else st_relaxed(lookback + (size_t)tile * 256 + d, kFlagAgg | c);
      uint32_t x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_scr[warp] = x;
      bar_named(1, 256);
      uint32_t add = 0;
      for (int g = 0; g < warp; ++g) add += s_scr[g];
      dstart = x - c + add;
      uint32_t run = dstart;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const uint32_t t = s_base[w][d];
        s_base[w][d] = run;
        run += t;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < I; ++i) s_el[s_base[warp][dig(el[i])] + rank[i]] = el[i];
    if (tid < 256) {
      uint32_t excl = 0;
      if (tile > 0) {
        int64_t t = (int64_t)tile - 1;
        bool done = false;
        while (!done) {
          uint32_t wv[LBW];
#pragma unroll
          for (int j = 0; j < LBW; ++j) {
            const int64_t tj = t - j < 0 ? 0 : t - j;
            wv[j] = ld_relaxed(lookback + (size_t)tj * 256 + d);
          }
          int used = 0;
#pragma unroll
          for (int j = 0; j < LBW; ++j) {
            if (done || used < j) continue;
            const uint32_t flag = wv[j] & ~kCountMask;
            if (flag == 0) continue;
            excl += wv[j] & kCountMask;
            used = j + 1;
            if (flag == kFlagInc) done = true;
          }
          t -= used;
        }
        st_relaxed(lookback + (size_t)tile * 256 + d, kFlagInc | (excl + c));
      }
      s_goff[d] = gs + excl - dstart;
    }
    __syncthreads();
    for (int j = tid; j < valid; j += T) {
      const uint64_t e = s_el[j];
      const uint32_t dst = s_goff[dig(e)] + (uint32_t)j;
      if (POUT) {
        eout[dst] = e;
      } else {
        kout[dst] = (uint32_t)e;
        vout[dst] = (uint32_t)(e >> 32);
      }
    }
    __syncthreads();  // s_el / s_base / s_goff / s_next reused by the next tile
  }
}

// device check of the lane-ordered shared atomics the rank-first kernel relies on
__global__ void atoms_order_check(unsigned int* bad, int rows) {
  __shared__ uint32_t cnt[8][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (int mod : {2, 5, 32, 256}) {
    for (int i = lane; i < 256; i += 32) cnt[warp][i] = 0;
    __syncwarp();
    for (int r = 0; r < rows; ++r) {
      const uint32_t d = (uint32_t)(splitmix64_at((uint64_t)(blockIdx.x * 8 + warp) * 7919u + mod, (uint64_t)r * 32 + lane) %
                                    (uint64_t)mod);
      const uint32_t before = cnt[warp][d];
      __syncwarp();
      const uint32_t below = __popc(__match_any_sync(0xffffffffu, d) & lt);
      const uint32_t got = atomicAdd(&cnt[warp][d], 1u);
      __syncwarp();
      if (got != before + below) atomicAdd(bad, 1u);
    }
  }
}

template <typename K, int T, int I>
size_t onesweep_smem(bool has_v) {
  return (size_t)T * I * sizeof(K) + (has_v ? (size_t)T * I * 4 : 0);
}

// Tuning variants (selected by HB_SORT_CFG for experiments; default = best measured)
struct PassArgs {
  const void* kin; void* kout; const uint32_t* vin; uint32_t* vout;
  int64_t n; int shift; uint64_t flip; const uint32_t* hist; uint32_t* lookback; uint32_t* counter;
  const uint32_t* gstart;  // pre-scanned digit starts of this pass
};

// true when shared atomics return lane-ordered old values on this device
// (checked once per device: 256 CTAs x 8 warps x 4 moduli x 512 rows)
bool atoms_rank_ok() {
  static int cached[64];
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  std::call_once(once[dev], [&] {
    unsigned int* bad = nullptr;
    unsigned int h = 1;
    if (cudaMalloc(&bad, 4) == cudaSuccess && cudaMemset(bad, 0, 4) == cudaSuccess) {
      atoms_order_check<<<256, 256>>>(bad, 512);
      if (cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost) != cudaSuccess) h = 1;
    }
    if (bad) cudaFree(bad);
    cudaGetLastError();
    cached[dev] = h == 0 ? 1 : 2;
  });
  return cached[dev] == 1;
}

template <bool PIN, bool POUT, int I, int T, int LBW, int MINB>
int launch_rfk_impl(const PassArgs& a, cudaStream_t s, int64_t tiles) {
  const size_t smem = (size_t)T * I * 8;
  auto k = onesweep_rfk_kernel<PIN, POUT, I, T, LBW, MINB>;
  HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<(unsigned)tiles, T, smem, s>>>(a.kin, a.kout, a.vin, a.vout, a.n, a.shift, (uint32_t)a.flip, a.gstart, a.lookback,
                                     a.counter);
  return check_launch();
}

template <bool PIN, bool POUT, int I, int T, int LBW>
int launch_rfp_impl(const PassArgs& a, cudaStream_t s, int64_t tiles) {
  const size_t smem = (size_t)T * I * 16;
  auto k = onesweep_rfp_kernel<PIN, POUT, I, T, LBW>;
  HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DeviceInfo di;
  HB_TRY(device_info(&di));
  int64_t grid = (int64_t)di.sms * 2;
  if (grid > tiles) grid = tiles;
  k<<<(unsigned)grid, T, smem, s>>>(a.kin, a.kout, a.vin, a.vout, a.n, a.shift, (uint32_t)a.flip, a.gstart, a.lookback,
                                    a.counter, (uint32_t)tiles);
  return check_launch();
}

template <int I, int T, int LBW>
int launch_rfp(const PassArgs& a, bool pin, bool pout, cudaStream_t s, int64_t* tiles_out, bool dry) {
  const int64_t tiles = ceil_div(a.n, (int64_t)T * I);
  *tiles_out = tiles;
  if (dry) return HB_OK;
  if (pin && pout) return launch_rfp_impl<true, true, I, T, LBW>(a, s, tiles);
  if (pin) return launch_rfp_impl<true, false, I, T, LBW>(a, s, tiles);
  if (pout) return launch_rfp_impl<false, true, I, T, LBW>(a, s, tiles);
  return launch_rfp_impl<false, false, I, T, LBW>(a, s, tiles);
}

template <int I, int T, int LBW, int MINB>
int launch_rfk(const PassArgs& a, bool pin, bool pout, cudaStream_t s, int64_t* tiles_out, bool dry) {
  const int64_t tiles = ceil_div(a.n, (int64_t)T * I);
  *tiles_out = tiles;
  if (dry) return HB_OK;
  if (pin && pout) return launch_rfk_impl<true, true, I, T, LBW, MINB>(a, s, tiles);
  if (pin) return launch_rfk_impl<true, false, I, T, LBW, MINB>(a, s, tiles);
  if (pout) return launch_rfk_impl<false, true, I, T, LBW, MINB>(a, s, tiles);
  return launch_rfk_impl<false, false, I, T, LBW, MINB>(a, s, tiles);
}

template <typename K, int I, int T, int LBW, int MINB, bool ES = false>
int launch_rf(const PassArgs& a, cudaStream_t s, int64_t* tiles_out, bool dry) {
  const int64_t tiles = ceil_div(a.n, (int64_t)T * I);
  *tiles_out = tiles;
  if (dry) return HB_OK;
  const size_t smem = (size_t)T * I * sizeof(K) + (a.vin ? (size_t)T * I * 4 : 0);
  if (a.vin) {
    HB_CUDA_TRY(cudaFuncSetAttribute(onesweep_rf_kernel<K, true, I, T, LBW, MINB, ES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    onesweep_rf_kernel<K, true, I, T, LBW, MINB, ES><<<(unsigned)tiles, T, smem, s>>>(
        (const K*)a.kin, (K*)a.kout, a.vin, a.vout, a.n, a.shift, (K)a.flip, a.gstart, a.lookback, a.counter);
  } else {
    HB_CUDA_TRY(cudaFuncSetAttribute(onesweep_rf_kernel<K, false, I, T, LBW, MINB, ES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    onesweep_rf_kernel<K, false, I, T, LBW, MINB, ES><<<(unsigned)tiles, T, smem, s>>>(
        (const K*)a.kin, (K*)a.kout, nullptr, nullptr, a.n, a.shift, (K)a.flip, a.gstart, a.lookback, a.counter);
  }
  return check_launch();
}

template <typename K, int I, int T = 512, bool TWO = false, int LBW = 1, bool MATCH = false, bool AR = false>
int launch_ec(const PassArgs& a, cudaStream_t s, int64_t* tiles_out, bool dry) {
  const int64_t tiles = ceil_div(a.n, (int64_t)T * I);
  *tiles_out = tiles;
  if (dry) return HB_OK;
  const size_t smem = (size_t)T * I * sizeof(K) + (a.vin ? (size_t)T * I * 4 : 0);
  if (a.vin) {
    HB_CUDA_TRY(cudaFuncSetAttribute(onesweep_ec_kernel<K, true, I, T, TWO, LBW, MATCH, AR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    onesweep_ec_kernel<K, true, I, T, TWO, LBW, MATCH, AR><<<(unsigned)tiles, T, smem, s>>>(
        (const K*)a.kin, (K*)a.kout, a.vin, a.vout, a.n, a.shift, (K)a.flip, a.gstart, a.lookback, a.counter);
  } else {
    HB_CUDA_TRY(cudaFuncSetAttribute(onesweep_ec_kernel<K, false, I, T, TWO, LBW, MATCH, AR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    onesweep_ec_kernel<K, false, I, T, TWO, LBW, MATCH, AR><<<(unsigned)tiles, T, smem, s>>>(
        (const K*)a.kin, (K*)a.kout, nullptr, nullptr, a.n, a.shift, (K)a.flip, a.gstart, a.lookback, a.counter);
  }
  return check_launch();
}

template <typename K, int T, int I, bool M>
int launch_pass(const PassArgs& a, cudaStream_t s, int64_t* tiles_out, bool dry) {
  const int64_t tiles = ceil_div(a.n, (int64_t)T * I);
  *tiles_out = tiles;
  if (dry) return HB_OK;
  const size_t smem = onesweep_smem<K, T, I>(a.vin != nullptr);
  if (a.vin) {
    HB_CUDA_TRY(cudaFuncSetAttribute(onesweep_kernel<K, true, T, I, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    onesweep_kernel<K, true, T, I, M><<<(unsigned)tiles, T, smem, s>>>(
        (const K*)a.kin, (K*)a.kout, a.vin, a.vout, a.n, a.shift, (K)a.flip, a.hist, a.lookback, a.counter);
  } else {
    HB_CUDA_TRY(cudaFuncSetAttribute(onesweep_kernel<K, false, T, I, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    onesweep_kernel<K, false, T, I, M><<<(unsigned)tiles, T, smem, s>>>(
        (const K*)a.kin, (K*)a.kout, nullptr, nullptr, a.n, a.shift, (K)a.flip, a.hist, a.lookback, a.counter);
  }
  return check_launch();
}

int sort_variant() {
  static int v = [] {
    const char* e = getenv("HB_SORT_CFG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <typename K, int T, int I>
int launch_persist(const PassArgs& a, cudaStream_t s, int64_t* tiles_out, bool dry) {
  const int64_t tiles = ceil_div(a.n, (int64_t)T * I);
  *tiles_out = tiles;
  if (dry) return HB_OK;
  DeviceInfo di;
  HB_TRY(device_info(&di));
  const bool hv = a.vin != nullptr;
  const size_t stage = (size_t)T * I * sizeof(K) + (hv ? (size_t)T * I * 4 : 0);
  const size_t smem = 2 * stage;
  const int vec_ok = ((uintptr_t)a.kin % 16 == 0) && (!hv || (uintptr_t)a.vin % 16 == 0);
  int64_t grid = (int64_t)di.sms * 3;
  if (grid > tiles) grid = tiles;
  if (hv) {
    HB_CUDA_TRY(cudaFuncSetAttribute(onesweep_persist_kernel<K, true, T, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    onesweep_persist_kernel<K, true, T, I><<<(unsigned)grid, T, smem, s>>>(
        (const K*)a.kin, (K*)a.kout, a.vin, a.vout, a.n, a.shift, (K)a.flip, a.hist, a.lookback, a.counter, tiles, vec_ok);
  } else {
    HB_CUDA_TRY(cudaFuncSetAttribute(onesweep_persist_kernel<K, false, T, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    onesweep_persist_kernel<K, false, T, I><<<(unsigned)grid, T, smem, s>>>(
        (const K*)a.kin, (K*)a.kout, nullptr, nullptr, a.n, a.shift, (K)a.flip, a.hist, a.lookback, a.counter, tiles, vec_ok);
  }
  return check_launch();
}

template <typename K, int T, int I>
int launch_tma(const PassArgs& a, cudaStream_t s, int64_t* tiles_out, bool dry) {
  const int64_t tiles = ceil_div(a.n, (int64_t)T * I);
  *tiles_out = tiles;
  if (dry) return HB_OK;
  const bool hv = a.vin != nullptr;
  if ((uintptr_t)a.kin % 16 || (hv && (uintptr_t)a.vin % 16))  // bulk copies need 16-byte alignment
    return launch_pass<K, 512, (sizeof(K) == 4 ? 12 : 8), false>(a, s, tiles_out, dry);
  DeviceInfo di;
  HB_TRY(device_info(&di));
  const size_t stage = (size_t)T * I * sizeof(K) + (hv ? (size_t)T * I * 4 : 0);
  const size_t smem = 2 * stage;
  int64_t grid = (int64_t)di.sms * 3;
  if (grid > tiles) grid = tiles;
  if (hv) {
    HB_CUDA_TRY(cudaFuncSetAttribute(onesweep_tma_kernel<K, true, T, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    onesweep_tma_kernel<K, true, T, I><<<(unsigned)grid, T, smem, s>>>(
        (const K*)a.kin, (K*)a.kout, a.vin, a.vout, a.n, a.shift, (K)a.flip, a.hist, a.lookback, a.counter, tiles);
  } else {
    HB_CUDA_TRY(cudaFuncSetAttribute(onesweep_tma_kernel<K, false, T, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    onesweep_tma_kernel<K, false, T, I><<<(unsigned)grid, T, smem, s>>>(
        (const K*)a.kin, (K*)a.kout, nullptr, nullptr, a.n, a.shift, (K)a.flip, a.hist, a.lookback, a.counter, tiles);
  }
  return check_launch();
}

template <typename K>
int run_pass(const PassArgs& a, cudaStream_t s, int64_t* tiles, bool dry) {
  if constexpr (sizeof(K) == 8) {
    switch (sort_variant()) {
      case 1: return launch_pass<K, 512, 8, false>(a, s, tiles, dry);
      case 6: return launch_persist<K, 256, 8>(a, s, tiles, dry);
      case 8: return launch_tma<K, 256, 8>(a, s, tiles, dry);
      case 12: return launch_pass<K, 256, 8, true>(a, s, tiles, dry);
      case 13: return launch_ec<K, 8>(a, s, tiles, dry);
      default:
        if (atoms_rank_ok()) return launch_rf<K, 12, 256, 2, 3, true>(a, s, tiles, dry);
        return launch_ec<K, 8>(a, s, tiles, dry);
    }
  } else {
  switch (sort_variant()) {
    case 1: return launch_pass<K, 512, 12, false>(a, s, tiles, dry);
    case 2: return launch_pass<K, 512, 12, true>(a, s, tiles, dry);
    case 3: return launch_pass<K, 256, 12, false>(a, s, tiles, dry);
    case 4: return launch_pass<K, 256, 16, true>(a, s, tiles, dry);
    case 5: return launch_pass<K, 384, 16, true>(a, s, tiles, dry);
    case 6: return launch_persist<K, 256, 12>(a, s, tiles, dry);
    case 7: return launch_persist<K, 256, 16>(a, s, tiles, dry);
    case 8: return launch_tma<K, 256, 12>(a, s, tiles, dry);
    case 9: return launch_tma<K, 256, 16>(a, s, tiles, dry);
    case 10: return launch_ec<K, 12>(a, s, tiles, dry);
    case 11: return launch_ec<K, 8>(a, s, tiles, dry);
    case 13: return launch_ec<K, 16, 384>(a, s, tiles, dry);
    case 14: return launch_ec<K, 12, 512, true>(a, s, tiles, dry);
    case 15: return launch_ec<K, 16, 384, true>(a, s, tiles, dry);
    case 16: return launch_ec<K, 20, 384>(a, s, tiles, dry);
    case 17: return launch_ec<K, 24, 384>(a, s, tiles, dry);
    case 18: return launch_ec<K, 16, 512>(a, s, tiles, dry);
    case 19: return launch_ec<K, 16, 640>(a, s, tiles, dry);
    case 20: return launch_ec<K, 28, 384>(a, s, tiles, dry);
    case 21: return launch_ec<K, 20, 384, false, 4>(a, s, tiles, dry);
    case 22: return launch_ec<K, 20, 384, false, 8>(a, s, tiles, dry);
    case 23: return launch_ec<K, 16, 384, false, 4>(a, s, tiles, dry);
    case 24: return launch_ec<K, 24, 384, false, 4>(a, s, tiles, dry);
    case 25: return launch_ec<K, 20, 384, false, 2>(a, s, tiles, dry);
    case 12: return launch_pass<K, 256, 12, true>(a, s, tiles, dry);
    case 26: return launch_ec<K, 20, 384>(a, s, tiles, dry);
    case 27: return launch_ec<K, 20, 384, false, 2, true>(a, s, tiles, dry);
    case 40: return launch_ec<K, 20, 384, false, 2, false, true>(a, s, tiles, dry);
    case 41: return launch_ec<K, 24, 384, false, 2, false, true>(a, s, tiles, dry);
    case 42: return launch_ec<K, 16, 384, false, 2, false, true>(a, s, tiles, dry);
    case 43: return launch_ec<K, 16, 512, false, 2, false, true>(a, s, tiles, dry);
    case 44: return launch_ec<K, 12, 512, false, 2, false, true>(a, s, tiles, dry);
    case 50: return launch_rf<K, 20, 384, 2, 2>(a, s, tiles, dry);
    case 51: return launch_rf<K, 12, 384, 2, 3>(a, s, tiles, dry);
    case 52: return launch_rf<K, 16, 512, 2, 2>(a, s, tiles, dry);
    case 53: return launch_rf<K, 24, 256, 2, 3>(a, s, tiles, dry);
    case 54: return launch_rf<K, 16, 256, 2, 4>(a, s, tiles, dry);
    case 55: return launch_rf<K, 14, 384, 2, 3>(a, s, tiles, dry);
    case 56: return launch_rf<K, 28, 256, 2, 3>(a, s, tiles, dry);
    case 57: return launch_rf<K, 20, 256, 2, 4>(a, s, tiles, dry);
    case 58: return launch_rf<K, 24, 256, 4, 3>(a, s, tiles, dry);
    case 59: return launch_rf<K, 32, 256, 2, 2>(a, s, tiles, dry);
    case 60: return launch_rf<K, 22, 256, 2, 3>(a, s, tiles, dry);
    case 61: return launch_rf<K, 24, 256, 1, 3>(a, s, tiles, dry);
    case 63: return launch_rf<K, 22, 256, 2, 3, true>(a, s, tiles, dry);
    case 64: return launch_rf<K, 24, 256, 2, 3, true>(a, s, tiles, dry);
    case 65: return launch_rf<K, 20, 384, 2, 2, true>(a, s, tiles, dry);
    case 66: return launch_rf<K, 22, 256, 4, 3, true>(a, s, tiles, dry);
    case 28: return launch_ec<K, 16, 384, false, 2, true>(a, s, tiles, dry);
    case 29: return launch_ec<K, 24, 384, false, 2, true>(a, s, tiles, dry);
    case 62: return launch_ec<K, 20, 384, false, 2>(a, s, tiles, dry);  // ballot ranking (42 Gkeys/s)
    default:  // best measured (round 1): rank-first with lane-ordered shared atomics + early re-order, 52 Gkeys/s
      if (atoms_rank_ok()) return launch_rf<K, 24, 256, 2, 3, true>(a, s, tiles, dry);
      return launch_ec<K, 20, 384, false, 2>(a, s, tiles, dry);
  }
  }
}

// live digit passes of a u32-key + u32-payload sort with the pair moved as one
// 8-byte element: split → packed → … → packed → split (back into keys/vals)
template <int PI, int PT, int LBW, int MINB, bool PERSIST = false>
int packed_passes(uint32_t* keys, uint32_t* vals, int64_t n, uint32_t flip, const bool* live, int nlive,
                  const DevBuf& hist, const DevBuf& gst, DevBuf& lb, cudaStream_t s) {
  int64_t tiles = 0;
  PassArgs pa{};
  pa.n = n;
  HB_TRY((launch_rfk<PI, PT, LBW, MINB>(pa, false, false, s, &tiles, true)));
  // the persistent kernel's CTAs claim one tile past the end each: counter room
  const size_t extra = PERSIST ? 2048 : 0;
  const size_t lb_words = (size_t)tiles * 256 + 32 + extra;
  DevBuf pA, pB;
  HB_TRY(alloc(&lb, lb_words * 4, s));
  HB_TRY(alloc(&pA, (size_t)n * 8, s));
  if (nlive >= 3) HB_TRY(alloc(&pB, (size_t)n * 8, s));
  uint32_t* counter = lb.as<uint32_t>() + (size_t)tiles * 256;
  void* cur = keys;
  void* nxt = pA.ptr;
  int done = 0;
  for (int p = 0; p < 4; ++p) {
    if (!live[p]) continue;
    const bool first = done == 0, last = done == nlive - 1;
    HB_CUDA_TRY(cudaMemsetAsync(lb.ptr, 0, lb_words * 4, s));
    pa.kin = cur;
    pa.kout = last ? (void*)keys : nxt;
    pa.vin = first ? vals : nullptr;
    pa.vout = last ? vals : nullptr;
    pa.shift = 8 * p; pa.flip = (uint64_t)flip; pa.hist = hist.as<uint32_t>() + p * 256;
    pa.lookback = lb.as<uint32_t>(); pa.counter = counter; pa.gstart = gst.as<uint32_t>() + p * 256;
    if (PERSIST) HB_TRY((launch_rfp<PI, PT, LBW>(pa, !first, !last, s, &tiles, false)));
    else HB_TRY((launch_rfk<PI, PT, LBW, MINB>(pa, !first, !last, s, &tiles, false)));
    cur = nxt;
    nxt = (nxt == pA.ptr) ? pB.ptr : pA.ptr;
    ++done;
  }
  return HB_OK;
}

template <typename K>
int radix_sort(K* keys, uint32_t* vals, int64_t n, K flip, int* passes_done, cudaStream_t s) {
  constexpr int P = SortCfg<K>::kPasses;
  DeviceInfo di;
  HB_TRY(device_info(&di));
  if (passes_done) *passes_done = 0;
  if (n <= 1) return HB_OK;
  if (n >= (int64_t)kCountMask) {
    set_error("radix sort supports n < 2^30 keys per call (got %lld)", (long long)n);
    return HB_EINVAL;
  }
  DevBuf hist, kalt, valt, lb;
  HB_TRY(alloc(&hist, (size_t)P * 256 * 4, s));
  HB_CUDA_TRY(cudaMemsetAsync(hist.ptr, 0, (size_t)P * 256 * 4, s));
  int64_t hb = ceil_div(n, 512 * 8);
  if (hb > (int64_t)di.sms * 2) hb = (int64_t)di.sms * 2;
  if constexpr (sizeof(K) == 4) {
    if (((uintptr_t)keys & 15) == 0 && sort_variant() != 62) {
      HB_CUDA_TRY(cudaFuncSetAttribute(digit_hist32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDh32Smem));
      DeviceInfo di;
      HB_TRY(device_info(&di));
      digit_hist32_kernel<<<di.sms, kDh32Threads, kDh32Smem, s>>>(reinterpret_cast<const uint32_t*>(keys), n,
                                                                   (uint32_t)flip, hist.as<uint32_t>());
    } else {
      digit_hist_kernel<K><<<(int)hb, 512, 0, s>>>(keys, n, flip, hist.as<uint32_t>());
    }
  } else {
    digit_hist_kernel<K><<<(int)hb, 512, 0, s>>>(keys, n, flip, hist.as<uint32_t>());
  }
  HB_TRY(check_launch());
  uint32_t h[P * 256];
  HB_CUDA_TRY(cudaMemcpyAsync(h, hist.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaStreamSynchronize(s));
  bool live[P];
  int nlive = 0;
  for (int p = 0; p < P; ++p) {
    live[p] = true;
    for (int b = 0; b < 256; ++b)
      if (h[p * 256 + b] == (uint32_t)n) live[p] = false;
    nlive += live[p];
  }
  if (passes_done) *passes_done = nlive;
  if (nlive == 0) return HB_OK;

  DevBuf gst;
  HB_TRY(alloc(&gst, (size_t)P * 256 * 4, s));
  scan_hist_kernel<<<P, 256, 0, s>>>(hist.as<uint32_t>(), gst.as<uint32_t>(), P);
  HB_TRY(check_launch());
  int64_t tiles = 0;
  PassArgs pa{};
  pa.n = n;
  if constexpr (sizeof(K) == 4) {
    // key + payload as one 8-byte element between the first and the last live pass
    const int v = sort_variant();
    const bool aligned16 = (((uintptr_t)keys | (uintptr_t)vals) & 15) == 0;
    if (vals && nlive >= 2 && (v == 0 || (v >= 74 && v <= 79)) && atoms_rank_ok()) {
      switch (v) {
        case 78:
          if (aligned16)
            return packed_passes<22, 256, 2, 2, true>(reinterpret_cast<uint32_t*>(keys), vals, n, (uint32_t)flip, live, nlive, hist, gst, lb, s);
          break;
        case 79:
          if (aligned16)
            return packed_passes<14, 384, 2, 2, true>(reinterpret_cast<uint32_t*>(keys), vals, n, (uint32_t)flip, live, nlive, hist, gst, lb, s);
          break;
        case 75: return packed_passes<20, 256, 2, 3>(reinterpret_cast<uint32_t*>(keys), vals, n, (uint32_t)flip, live, nlive, hist, gst, lb, s);
        case 76: return packed_passes<24, 256, 2, 3>(reinterpret_cast<uint32_t*>(keys), vals, n, (uint32_t)flip, live, nlive, hist, gst, lb, s);
        case 77: return packed_passes<16, 256, 2, 4>(reinterpret_cast<uint32_t*>(keys), vals, n, (uint32_t)flip, live, nlive, hist, gst, lb, s);
        default:  // best measured: 22 keys/thread, 59.5 Gkeys/s (24: 57.4, 20: 55.6)
          return packed_passes<22, 256, 2, 3>(reinterpret_cast<uint32_t*>(keys), vals, n, (uint32_t)flip, live, nlive, hist, gst, lb, s);
      }
    }
  }
  HB_TRY(alloc(&kalt, (size_t)n * sizeof(K), s));
  if (vals) HB_TRY(alloc(&valt, (size_t)n * 4, s));
  HB_TRY(run_pass<K>(pa, s, &tiles, true));
  const size_t lb_words = (size_t)tiles * 256 + 32;  // + tile counter (padded)
  HB_TRY(alloc(&lb, lb_words * 4, s));
  K* kcur = keys;
  K* knext = kalt.as<K>();
  uint32_t* vcur = vals;
  uint32_t* vnext = valt.as<uint32_t>();
  uint32_t* counter = lb.as<uint32_t>() + (size_t)tiles * 256;
  for (int p = 0; p < P; ++p) {
    if (!live[p]) continue;
    HB_CUDA_TRY(cudaMemsetAsync(lb.ptr, 0, lb_words * 4, s));
    pa.kin = kcur; pa.kout = knext; pa.vin = vcur; pa.vout = vals ? vnext : nullptr;
    pa.shift = 8 * p; pa.flip = (uint64_t)flip; pa.hist = hist.as<uint32_t>() + p * 256;
    pa.lookback = lb.as<uint32_t>(); pa.counter = counter; pa.gstart = gst.as<uint32_t>() + p * 256;
    HB_TRY(run_pass<K>(pa, s, &tiles, false));
    std::swap(kcur, knext);
    std::swap(vcur, vnext);
  }
  if (kcur != keys) {
    HB_CUDA_TRY(cudaMemcpyAsync(keys, kcur, (size_t)n * sizeof(K), cudaMemcpyDeviceToDevice, s));
    if (vals) HB_CUDA_TRY(cudaMemcpyAsync(vals, vcur, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
  }
  return HB_OK;
}

// lower_bound of (probe_key, probe_val) in the lexicographically sorted
// (keys, vals) sequence — the split points of the sample-merge exchange.
template <typename K>
__global__ void sort_bounds_kernel(const K* __restrict__ keys, const uint32_t* __restrict__ vals,
                                   int64_t n, K flip, const K* __restrict__ pk,
                                   const uint32_t* __restrict__ pv, int m,
                                   int64_t* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const K key = pk[j] ^ flip;
  const uint32_t v = pv ? pv[j] : 0u;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const K k = keys[mid] ^ flip;
    const bool less = k < key || (pv && vals && k == key && vals[mid] < v);
    if (less) lo = mid + 1;
    else hi = mid;
  }
  out[j] = lo;
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hb_sort_bounds(const void* keys, int key_code, const uint32_t* vals, int64_t n,
                              const void* probe_keys, const uint32_t* probe_vals, int32_t m,
                              int64_t* out_pos, int flags, void* stream) {
  HB_CHECK_ARG(key_code == HB_U32 || key_code == HB_I32 || key_code == HB_U64 || key_code == HB_I64,
               "keys must be u32, i32, u64 or i64");
  HB_CHECK_ARG(n >= 0 && m >= 0, "negative size");
  if (m == 0) return HB_OK;
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_sort_bounds works on device arrays");
  cudaStream_t s = as_stream(stream);
  const int blocks = (m + 127) / 128;
  if (key_code == HB_U64 || key_code == HB_I64) {
    const uint64_t flip = key_code == HB_I64 ? (1ull << 63) : 0ull;
    sort_bounds_kernel<uint64_t><<<blocks, 128, 0, s>>>((const uint64_t*)keys, vals, n, flip,
                                                          (const uint64_t*)probe_keys, probe_vals, m, out_pos);
  } else {
    const uint32_t flip = key_code == HB_I32 ? (1u << 31) : 0u;
    sort_bounds_kernel<uint32_t><<<blocks, 128, 0, s>>>((const uint32_t*)keys, vals, n, flip,
                                                          (const uint32_t*)probe_keys, probe_vals, m, out_pos);
  }
  return finish(flags, s);
}

extern "C" int hb_sort(const void* keys_in, void* keys_out, int key_code, const uint32_t* vals_in,
                       uint32_t* vals_out, int64_t n, int32_t* passes_done, int flags, void* stream) {
  HB_CHECK_ARG(key_code == HB_U32 || key_code == HB_I32 || key_code == HB_U64 || key_code == HB_I64,
               "sort keys must be u32, i32, u64 or i64 (code %d)", key_code);
  HB_CHECK_ARG(n >= 0, "n must be >= 0");
  HB_CHECK_ARG(n == 0 || (keys_in && keys_out), "keys is NULL");
  HB_CHECK_ARG(!vals_in == !vals_out, "vals_in and vals_out must both be set or both NULL");
  const bool dev = flags & HB_DEVICE_PTRS;
  HB_CHECK_ARG(dev || !(flags & HB_ASYNC), "HB_ASYNC requires device pointers");
  cudaStream_t s = as_stream(stream);
  const bool wide = key_code == HB_U64 || key_code == HB_I64;
  const size_t ks = wide ? 8 : 4;
  DevBuf dk, dv;
  if (dev) {
    // device: sort in keys_out (copy first unless in place)
    if (keys_out != keys_in && n) HB_CUDA_TRY(cudaMemcpyAsync(keys_out, keys_in, (size_t)n * ks, cudaMemcpyDeviceToDevice, s));
    if (vals_in && vals_out != vals_in && n) HB_CUDA_TRY(cudaMemcpyAsync(vals_out, vals_in, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
    HB_TRY(stage_in(&dk, keys_out, (size_t)n * ks, true, s));
    if (vals_in) HB_TRY(stage_in(&dv, vals_out, (size_t)n * 4, true, s));
  } else {
    HB_TRY(stage_in(&dk, keys_in, (size_t)n * ks, false, s));
    if (vals_in) HB_TRY(stage_in(&dv, vals_in, (size_t)n * 4, false, s));
  }
  int done = 0;
  int rc;
  if (wide) {
    const uint64_t flip = key_code == HB_I64 ? (1ull << 63) : 0ull;
    rc = radix_sort<uint64_t>(dk.as<uint64_t>(), vals_in ? dv.as<uint32_t>() : nullptr, n, flip, &done, s);
  } else {
    const uint32_t flip = key_code == HB_I32 ? (1u << 31) : 0u;
    rc = radix_sort<uint32_t>(dk.as<uint32_t>(), vals_in ? dv.as<uint32_t>() : nullptr, n, flip, &done, s);
  }
  if (rc != HB_OK) return rc;
  if (passes_done) *passes_done = done;
  HB_TRY(copy_out(keys_out, dk, (size_t)n * ks, dev, s));
  if (vals_in) HB_TRY(copy_out(vals_out, dv, (size_t)n * 4, dev, s));
  return finish(flags, s);
}
