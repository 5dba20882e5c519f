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
#include <string.h>

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
// INM — the input is key and payload arrays (0), packed (1), or list
// ranking's level-1 log (2: log_slot_pair turns each slot into its packed
// pair on the load, prefix = the ranked sublist starts); OUTM — the output is
// packed (1) or split back into the two arrays (0).  The first live digit
// pass reads split and writes packed, the middle passes stay packed, the
// last one writes split: one 8-byte load / smem store / smem load / global
// store per element instead of two of each.
template <int INM, int OUTM, int I, int T, int LBW, int MINB>
__global__ void __launch_bounds__(T, MINB)
    onesweep_rfk_kernel(const void* __restrict__ kin_, void* __restrict__ kout_, const uint32_t* __restrict__ vin,
                        uint32_t* __restrict__ vout, int64_t n, int shift, uint32_t flip,
                       const uint32_t* __restrict__ gstart, uint32_t* __restrict__ lookback,
                       uint32_t* __restrict__ tile_counter, const int64_t* __restrict__ prefix,
                       uint32_t* __restrict__ clear, uint32_t* __restrict__ clear_counter) {
  static_assert(OUTM == 0 || OUTM == 1, "output split (0) or packed (1)");
  static_assert(INM != 2 || (T * I) % kLogChunkSlots == 0, "log tiles are whole chunks");
  constexpr bool POUT = OUTM == 1;
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
  // the next pass's look-back words (the other buffer, idle during this
  // pass) are zeroed tile by tile: no memset kernel between passes
  if (clear != nullptr && tid < 256) {
    clear[(size_t)tile * 256 + tid] = 0u;
    if (tile == 0 && tid == 0) *clear_counter = 0u;
  }
  const int64_t base = (int64_t)tile * TILE;
  const int valid = (int)min((int64_t)TILE, n - base);
  const int wbase = warp * 32 * I;
  uint64_t el[I];
  uint32_t rank[I];
#pragma unroll
  for (int i = 0; i < I; ++i) {
    const int idx = wbase + i * 32 + lane;
    const bool ok = idx < valid;
    if (INM == 2) el[i] = log_slot_pair(ok ? ein[base + idx] : (uint64_t)kLogEmpty << 32, prefix);
    else if (INM == 1) el[i] = ok ? ein[base + idx] : (uint64_t)(~0u ^ flip);
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

// ------------------------------------------------------------------ host side
struct PassArgs {
  const void* kin; void* kout; const uint32_t* vin; uint32_t* vout;
  int64_t n; int shift; uint64_t flip; const uint32_t* hist; uint32_t* lookback; uint32_t* counter;
  uint32_t* clear = nullptr; uint32_t* clear_counter = nullptr;  // rfk: the next pass's words, zeroed in-pass
  const uint32_t* gstart;  // pre-scanned digit starts of this pass
  const int64_t* prefix;   // INM 2 (log input): ranked sublist starts
};

bool production_rank_selftest();

// true when shared atomics return lane-ordered old values on this device:
// checked once per device, first on the bare pattern (256 CTAs x 8 warps x 4
// moduli x 512 rows), then through the production kernels themselves
// (production_rank_selftest: duplicate-heavy keys with an index payload
// through every atomics-ranked pass shape, stability checked on the device).
// Any violation selects the ballot ranking for the process.
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
    cached[dev] = (h == 0 && production_rank_selftest()) ? 1 : 2;
  });
  return cached[dev] == 1;
}

// Ranking method of a call: the lane-ordered shared-atomic ranking (fast,
// verified per device) unless the caller asks for the ballot multi-split
// (HB_SORT_BALLOT), the environment forces it (HB_SORT_RANK=ballot), or the
// device check failed.
bool use_atomics_rank(int flags) {
  static const bool env_ballot = [] {
    const char* e = getenv("HB_SORT_RANK");
    return e && strcmp(e, "ballot") == 0;
  }();
  return !(flags & HB_SORT_BALLOT) && !env_ballot && atoms_rank_ok();
}

// u32 key + u32 payload moved as one 8-byte element: 22 keys/thread, 256
// threads, 3 CTAs/SM (measured best: 59.5 Gkeys/s; 24: 57.4, 20: 55.6);
// look-back window 3 predecessors per round trip (2^28 pairs: window 1 / 2 /
// 3 / 4 / 5 / 6 = 4.75 / 4.36 / 4.29 / 4.32 / 4.34 / 4.38 ms,
// profiles/micro_sort_lookback_reset_r02.txt)
constexpr int kPkI = 22, kPkT = 256, kPkLbw = 3, kPkMinB = 3;

template <int INM, int OUTM>
int launch_rfk(const PassArgs& a, cudaStream_t s, int64_t tiles) {
  const size_t smem = (size_t)kPkT * kPkI * 8;
  auto k = onesweep_rfk_kernel<INM, OUTM, kPkI, kPkT, kPkLbw, kPkMinB>;
  HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<(unsigned)tiles, kPkT, smem, s>>>(a.kin, a.kout, a.vin, a.vout, a.n, a.shift, (uint32_t)a.flip, a.gstart,
                                        a.lookback, a.counter, a.prefix, a.clear, a.clear_counter);
  return check_launch();
}

// Separate key / payload arrays.  Rank-first (atomics) tiles: u32 24 keys x
// 256 threads, u64 12 x 256; ballot tiles: u32 20 x 384, u64 8 x 512.
template <typename K>
struct PassShape {
  static constexpr int rf_i = sizeof(K) == 4 ? 24 : 12, rf_t = 256;
  static constexpr int ec_i = sizeof(K) == 4 ? 20 : 8, ec_t = sizeof(K) == 4 ? 384 : 512, ec_lbw = sizeof(K) == 4 ? 2 : 1;
  static int64_t tiles(int64_t n, bool atoms) { return ceil_div(n, atoms ? (int64_t)rf_i * rf_t : (int64_t)ec_i * ec_t); }
};

template <typename K, bool HAS_V>
int launch_pass(const PassArgs& a, bool atoms, cudaStream_t s) {
  using Sh = PassShape<K>;
  const int64_t tiles = Sh::tiles(a.n, atoms);
  if (atoms) {
    const size_t smem = (size_t)Sh::rf_t * Sh::rf_i * (sizeof(K) + (HAS_V ? 4 : 0));
    auto k = onesweep_rf_kernel<K, HAS_V, Sh::rf_i, Sh::rf_t, 3, 3, true>;  // look-back window 3 (as the packed pass)
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)tiles, Sh::rf_t, smem, s>>>((const K*)a.kin, (K*)a.kout, a.vin, a.vout, a.n, a.shift, (K)a.flip,
                                              a.gstart, a.lookback, a.counter);
  } else {
    const size_t smem = (size_t)Sh::ec_t * Sh::ec_i * (sizeof(K) + (HAS_V ? 4 : 0));
    auto k = onesweep_ec_kernel<K, HAS_V, Sh::ec_i, Sh::ec_t, false, Sh::ec_lbw>;
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)tiles, Sh::ec_t, smem, s>>>((const K*)a.kin, (K*)a.kout, a.vin, a.vout, a.n, a.shift, (K)a.flip,
                                              a.gstart, a.lookback, a.counter);
  }
  return check_launch();
}

// Look-back words of consecutive onesweep passes: two buffers of `words`
// (tiles·256 flags + the padded tile counter); pass k uses buffer k % 2 and
// zeroes the other one tile by tile for pass k + 1, so only the first
// buffer needs a memset (one per sort instead of one per pass).
struct LookbackPair {
  uint32_t* base = nullptr;
  size_t words = 0;
  int64_t tiles = 0;
  void set(int k, bool more, PassArgs& pa) const {
    uint32_t* cur = base + (size_t)(k & 1) * words;
    uint32_t* oth = base + (size_t)((k + 1) & 1) * words;
    pa.lookback = cur;
    pa.counter = cur + (size_t)tiles * 256;
    pa.clear = more ? oth : nullptr;
    pa.clear_counter = more ? oth + (size_t)tiles * 256 : nullptr;
  }
};

int lookback_pair(DevBuf& lb, int64_t tiles, LookbackPair* out, cudaStream_t s) {
  out->tiles = tiles;
  out->words = (size_t)tiles * 256 + 32;
  HB_TRY(alloc(&lb, 2 * out->words * 4, s));
  out->base = lb.as<uint32_t>();
  HB_CUDA_TRY(cudaMemsetAsync(out->base, 0, out->words * 4, s));
  return HB_OK;
}

// live digit passes of a u32-key + u32-payload sort with the pair moved as one
// 8-byte element: split → packed → … → packed → split (back into keys/vals)
int packed_passes(uint32_t* keys, uint32_t* vals, int64_t n, uint32_t flip, const bool* live, int nlive,
                  const DevBuf& hist, const DevBuf& gst, DevBuf& lb, cudaStream_t s) {
  const int64_t tiles = ceil_div(n, (int64_t)kPkT * kPkI);
  DevBuf pA, pB;
  LookbackPair lbp;
  HB_TRY(lookback_pair(lb, tiles, &lbp, s));
  HB_TRY(alloc(&pA, (size_t)n * 8, s));
  if (nlive >= 3) HB_TRY(alloc(&pB, (size_t)n * 8, s));
  PassArgs pa{};
  pa.n = n;
  void* cur = keys;
  void* nxt = pA.ptr;
  int done = 0;
  for (int p = 0; p < 4; ++p) {
    if (!live[p]) continue;
    const bool first = done == 0, last = done == nlive - 1;
    lbp.set(done, !last, pa);
    pa.kin = cur;
    pa.kout = last ? (void*)keys : nxt;
    pa.vin = first ? vals : nullptr;
    pa.vout = last ? vals : nullptr;
    pa.shift = 8 * p; pa.flip = (uint64_t)flip; pa.hist = hist.as<uint32_t>() + p * 256;
    pa.gstart = gst.as<uint32_t>() + p * 256;
    if (first && last) return HB_EINVAL;  // nlive >= 2 on this path
    if (first) HB_TRY((launch_rfk<0, 1>(pa, s, tiles)));
    else if (last) HB_TRY((launch_rfk<1, 0>(pa, s, tiles)));
    else HB_TRY((launch_rfk<1, 1>(pa, s, tiles)));
    cur = nxt;
    nxt = (nxt == pA.ptr) ? pB.ptr : pA.ptr;
    ++done;
  }
  return HB_OK;
}

// Order packed (payload << 32 | key) pairs by the key bits [shift0,
// shift0 + 8 * passes): `passes` packed digit passes, hist = their digit
// histograms (row p for the digit at shift0 + 8p), already counted by the
// producer of `pairs`.  With log_prefix, `pairs` is list ranking's level-1
// log and the first pass reads each slot as its packed pair (INM 2).  The
// passes ping-pong between `pairs` and `alt` (n pairs, the caller's); the
// result lands in *sorted (one of the two).  Needs the atomics ranking
// (stable); returns HB_ENOSYS when it is not in use so the caller takes the
// general path.
int sort_pairs_bits(uint64_t* pairs, int64_t n, const uint32_t* hist, int shift0, int passes,
                    const int64_t* log_prefix, uint64_t* alt, uint64_t** sorted, cudaStream_t s) {
  if (!use_atomics_rank(0)) return HB_ENOSYS;
  if (n >= (int64_t)kCountMask) {
    set_error("radix sort supports n < 2^30 keys per call (got %lld)", (long long)n);
    return HB_EINVAL;
  }
  if (passes < 1 || passes > 4 || shift0 < 0 || shift0 + 8 * passes > 32) return HB_EINVAL;
  const int64_t tiles = ceil_div(n, (int64_t)kPkT * kPkI);
  DevBuf gst, lb;
  HB_TRY(alloc(&gst, (size_t)passes * 256 * 4, s));
  scan_hist_kernel<<<passes, 256, 0, s>>>(hist, gst.as<uint32_t>(), passes);
  HB_TRY(check_launch());
  LookbackPair lbp;
  HB_TRY(lookback_pair(lb, tiles, &lbp, s));
  PassArgs pa{};
  pa.n = n;
  pa.flip = 0;
  void* cur = pairs;
  void* nxt = alt;
  for (int p = 0; p < passes; ++p) {
    lbp.set(p, p + 1 < passes, pa);
    pa.kin = cur;
    pa.kout = nxt;
    pa.vin = nullptr;
    pa.vout = nullptr;
    pa.shift = shift0 + 8 * p;
    pa.hist = hist + p * 256;
    pa.gstart = gst.as<uint32_t>() + p * 256;
    pa.prefix = log_prefix;
    if (p == 0 && log_prefix) HB_TRY((launch_rfk<2, 1>(pa, s, tiles)));
    else HB_TRY((launch_rfk<1, 1>(pa, s, tiles)));
    std::swap(cur, nxt);
  }
  *sorted = static_cast<uint64_t*>(cur);
  return HB_OK;
}

// `flags`: HB_SORT_BALLOT selects the ballot ranking; with HB_ASYNC and no
// passes_done the digit histogram is not read back (no host sync): every
// digit position is sorted (a constant digit's pass is the identity).
template <typename K>
int radix_sort_impl(K* keys, uint32_t* vals, int64_t n, K flip, int* passes_done, int flags, bool atoms,
                    cudaStream_t s) {
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
  if (sizeof(K) == 4 && ((uintptr_t)keys & 15) == 0) {
    HB_CUDA_TRY(cudaFuncSetAttribute(digit_hist32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDh32Smem));
    digit_hist32_kernel<<<di.sms, kDh32Threads, kDh32Smem, s>>>(reinterpret_cast<const uint32_t*>(keys), n,
                                                                 (uint32_t)flip, hist.as<uint32_t>());
  } else {
    int64_t hb = ceil_div(n, 512 * 8);
    if (hb > (int64_t)di.sms * 2) hb = (int64_t)di.sms * 2;
    digit_hist_kernel<K><<<(int)hb, 512, 0, s>>>(keys, n, flip, hist.as<uint32_t>());
  }
  HB_TRY(check_launch());
  bool live[P];
  int nlive = 0;
  const bool no_sync = (flags & HB_ASYNC) && !passes_done && sizeof(K) == 4;
  if (no_sync) {
    for (int p = 0; p < P; ++p) live[p] = true;
    nlive = P;
  } else {
    uint32_t h[P * 256];
    HB_CUDA_TRY(cudaMemcpyAsync(h, hist.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    for (int p = 0; p < P; ++p) {
      live[p] = true;
      for (int b = 0; b < 256; ++b)
        if (h[p * 256 + b] == (uint32_t)n) live[p] = false;
      nlive += live[p];
    }
  }
  if (passes_done) *passes_done = nlive;
  if (nlive == 0) return HB_OK;

  DevBuf gst;
  HB_TRY(alloc(&gst, (size_t)P * 256 * 4, s));
  scan_hist_kernel<<<P, 256, 0, s>>>(hist.as<uint32_t>(), gst.as<uint32_t>(), P);
  HB_TRY(check_launch());
  if constexpr (sizeof(K) == 4) {
    if (vals && nlive >= 2 && atoms)
      return packed_passes(reinterpret_cast<uint32_t*>(keys), vals, n, (uint32_t)flip, live, nlive, hist, gst, lb, s);
  }
  HB_TRY(alloc(&kalt, (size_t)n * sizeof(K), s));
  if (vals) HB_TRY(alloc(&valt, (size_t)n * 4, s));
  const int64_t tiles = PassShape<K>::tiles(n, atoms);
  const size_t lb_words = (size_t)tiles * 256 + 32;  // + tile counter (padded)
  HB_TRY(alloc(&lb, lb_words * 4, s));
  PassArgs pa{};
  pa.n = n;
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
    HB_TRY((vals ? launch_pass<K, true>(pa, atoms, s) : launch_pass<K, false>(pa, atoms, s)));
    std::swap(kcur, knext);
    std::swap(vcur, vnext);
  }
  if (kcur != keys) {
    HB_CUDA_TRY(cudaMemcpyAsync(keys, kcur, (size_t)n * sizeof(K), cudaMemcpyDeviceToDevice, s));
    if (vals) HB_CUDA_TRY(cudaMemcpyAsync(vals, vcur, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
  }
  return HB_OK;
}

template <typename K>
int radix_sort(K* keys, uint32_t* vals, int64_t n, K flip, int* passes_done, int flags, cudaStream_t s) {
  return radix_sort_impl<K>(keys, vals, n, flip, passes_done, flags, use_atomics_rank(flags), s);
}

// ---- the production-path stability self-test (run once per device)
template <typename K>
__global__ void selftest_fill(K* keys, uint32_t* vals, int64_t n, uint64_t seed, uint64_t mod, int shift_hi) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = splitmix64_at(seed, (uint64_t)i + 1);
    K k = (K)(r % mod);
    if (shift_hi > 0) k |= (K)((r >> 32) % mod) << shift_hi;  // a second live digit far from the first
    keys[i] = k;
    vals[i] = (uint32_t)i;
  }
}
template <typename K>
__global__ void selftest_check(const K* keys, const uint32_t* vals, int64_t n, unsigned int* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool ok = keys[i - 1] < keys[i] || (keys[i - 1] == keys[i] && vals[i - 1] < vals[i]);
    if (!ok) atomicAdd(bad, 1u);
  }
}
template <typename K>
bool selftest_case(uint64_t mod, int shift_hi, bool sync_path, cudaStream_t s) {
  const int64_t n = ((int64_t)1 << 20) + 7;  // ragged last tile
  DevBuf keys, vals, bad;
  if (alloc(&keys, (size_t)n * sizeof(K), s) != HB_OK || alloc(&vals, (size_t)n * 4, s) != HB_OK ||
      alloc(&bad, 4, s) != HB_OK)
    return false;
  selftest_fill<K><<<256, 256, 0, s>>>(keys.as<K>(), vals.as<uint32_t>(), n, 0x5eed0000ull + mod, mod, shift_hi);
  int passes = 0;
  if (radix_sort_impl<K>(keys.as<K>(), vals.as<uint32_t>(), n, (K)0, sync_path ? &passes : nullptr,
                         sync_path ? 0 : HB_ASYNC, true, s) != HB_OK)
    return false;
  unsigned int h = 1;
  if (cudaMemsetAsync(bad.ptr, 0, 4, s) != cudaSuccess) return false;
  selftest_check<K><<<256, 256, 0, s>>>(keys.as<K>(), vals.as<uint32_t>(), n, bad.as<unsigned int>());
  if (cudaMemcpyAsync(&h, bad.ptr, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return false;
  return h == 0;
}

// Duplicate-heavy keys (2..256 distinct values per live digit) with an index
// payload through every pass shape the atomics ranking drives: u32 one live
// digit (onesweep_rf_kernel), u32 all four digits (packed onesweep_rfk
// kernels: split → packed → packed → split), u32 two live digits, u64 keys.
bool production_rank_selftest() {
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return false;
  bool ok = selftest_case<uint32_t>(3, 0, true, s) && selftest_case<uint32_t>(2, 0, false, s) &&
            selftest_case<uint32_t>(256, 0, false, s) && selftest_case<uint32_t>(5, 24, true, s) &&
            selftest_case<uint64_t>(7, 40, true, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  cudaGetLastError();
  return ok;
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

// list ranking's node sort (csrc/listrank.cu)
int sort_pairs_bits_ext(uint64_t* pairs, int64_t n, const uint32_t* hist, int shift0, int passes,
                        const int64_t* log_prefix, uint64_t* alt, uint64_t** sorted, cudaStream_t s) {
  return sort_pairs_bits(pairs, n, hist, shift0, passes, log_prefix, alt, sorted, s);
}
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
    rc = radix_sort<uint64_t>(dk.as<uint64_t>(), vals_in ? dv.as<uint32_t>() : nullptr, n, flip,
                              passes_done ? &done : nullptr, flags, s);
  } else {
    const uint32_t flip = key_code == HB_I32 ? (1u << 31) : 0u;
    rc = radix_sort<uint32_t>(dk.as<uint32_t>(), vals_in ? dv.as<uint32_t>() : nullptr, n, flip,
                              passes_done ? &done : nullptr, dev ? flags : (flags & ~HB_ASYNC), s);
  }
  if (rc != HB_OK) return rc;
  if (passes_done) *passes_done = done;
  HB_TRY(copy_out(keys_out, dk, (size_t)n * ks, dev, s));
  if (vals_in) HB_TRY(copy_out(vals_out, dv, (size_t)n * 4, dev, s));
  return finish(flags, s);
}
