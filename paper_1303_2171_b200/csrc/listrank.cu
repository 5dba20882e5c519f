// listrank.cu — list ranking (replaces the ranking of list_rank_with_stats /
// list_rank_hybrid, reference kernels_irregular.py:377-508: rank[i] = distance
// of node i from the head; the result is independent of the algorithm, so the
// output equals the reference's bit for bit).
//
// Fast path (hb_list_rank): recursive sparse ruling set (Helman-JaJa) with
// Wyllie pointer jumping at the top.
//   level 1: every node whose index is a multiple of K (plus the list head)
//            starts a sublist; one thread per sublist walks its successors
//            until the next sublist head, writing (sublist id, local weighted
//            offset) packed into the 64-bit output slot of each node it passes
//            and the sublist's (next sublist, length);
//   level 2+: the same on the list of sublists (weighted by their lengths)
//            until at most kBase nodes remain;
//   top:     one CTA ranks the remaining list in shared memory by Wyllie
//            pointer jumping (suffix sums → prefix = total - suffix) and checks
//            that the chain from the head covers every node (broken lists and
//            cycles → HB_ESTRUCT, the reference's StructuralError);
//   back down: rank = prefix[sublist] + local offset, one coalesced pass per
//            level.
// The walk is a chain of dependent random 4-byte reads (one 32-byte sector
// per node): it is bound by DRAM sector throughput, not bytes.
#include <stdlib.h>

#include <algorithm>
#include <climits>
#include <vector>

#include "common.cuh"

namespace hb {
int sort_pairs_bits_ext(uint64_t* pairs, int64_t n, const uint32_t* hist, int shift0, int passes,
                        const int64_t* log_prefix, uint64_t* alt, uint64_t** sorted, cudaStream_t s);
namespace {

#ifndef HB_LR_K
#define HB_LR_K 64
#endif
constexpr int kK = HB_LR_K;   // sublist spacing (node index multiple)
constexpr int kBase = 4096;   // top level size ranked in one CTA

// Validation: out[0] += tails (succ == -1), out[1] += out-of-range successors.
// 16-byte loads, four in flight per thread (a pure read stream of n * sizeof(S) bytes).
template <typename S>
__global__ void lr_check_kernel(const S* __restrict__ succ, int64_t n,
                                unsigned long long* __restrict__ out) {
  constexpr int V = 16 / sizeof(S), U = 4;  // successors per 16-byte load, loads in flight
  unsigned long long tails = 0, bad = 0;
  auto test = [&](int64_t s) {
    tails += (s == -1);
    bad += (s < -1 || s >= n);
  };
  const int64_t nv = ((uintptr_t)succ & 15) ? 0 : n / V;  // whole 16-byte vectors (a caller's view may be unaligned)
  const uint4* sv = reinterpret_cast<const uint4*>(succ);
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += T * U) {
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) w[u] = i + u * T < nv ? __ldcs(sv + i + u * T) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u * T >= nv) continue;
      const S* e = reinterpret_cast<const S*>(&w[u]);
#pragma unroll
      for (int k = 0; k < V; ++k) test((int64_t)e[k]);
    }
  }
  for (int64_t i = nv * V + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T) test((int64_t)succ[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    tails += __shfl_xor_sync(0xffffffffu, tails, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (tails) atomicAdd(out, tails);
    if (bad) atomicAdd(out + 1, bad);
  }
}

// Sublist heads of a level with spacing 2^ks: node indices that are
// multiples of 2^ks, plus the list head.  Level 1 (the input list) uses
// kK = 64 — the layout hb_lr_layout publishes; the levels above use
// kUpperShift (shorter sublists: those walks are few, so their time is the
// longest sublist's, ~2^ks * ln(sublists) dependent steps).
constexpr int kKShift = 6;
static_assert((1 << kKShift) == kK, "kK is a power of two");
#ifndef HB_LR_UPPER_SHIFT
#define HB_LR_UPPER_SHIFT 3  // levels >= 2 of a 2^28-node list: spacing 64 -> 536 us, 8 -> 339, 4 -> 365 (ncu, cold)
#endif
constexpr int kUpperShift = HB_LR_UPPER_SHIFT;
__device__ __forceinline__ bool is_head(int64_t v, int64_t head, int ks) {
  return (v & ((1ll << ks) - 1)) == 0 || v == head;
}

// sublist id of a head node: v / 2^ks for multiples of 2^ks, `extra` for the list head otherwise
__device__ __forceinline__ int64_t sub_id(int64_t v, int64_t head, int64_t extra, int ks) {
  return (v & ((1ll << ks) - 1)) == 0 ? v >> ks : extra;
}

// Sublist walks.  tmp[v] = (sublist << 32) | local offset; nxt[j] = next
// sublist or -1; len[j] = weight sum.  Each thread claims sublists from a
// global counter (or the static stride t, t+T, ...) and keeps kChains of them
// in flight; the loop is flattened (a finished walk immediately starts the
// thread's next sublist), so lanes never idle waiting for the longest walk of
// their warp.  With 2048 threads per SM one dependent chain per thread
// already fills the random-access path, and the single-chain loop is the
// leanest (kChains = 1 measured fastest).
#ifndef HB_LR_CHAINS
#define HB_LR_CHAINS 1  // measured with dynamic claiming: 1 / 2 / 3 / 4 / 8 chains = 13.24 / 12.97 / 12.76 / 12.62 / 12.0 Gnodes/s
#endif
constexpr int kChains = HB_LR_CHAINS;
constexpr int64_t kWalkBlocksPer10Sm = 36;  // level-1 log walk: 3.6 blocks of 128 threads per SM

// The level-1 walk's two hot global counters (sublist claims, log-chunk
// claims) sit 256 bytes apart in one small stream-ordered allocation.  How
// fast the walk runs depended on where they landed — in one 128-byte line
// 24.4 ms per 2^28-node call, 256 B or 64 KB apart 15.4-15.6 ms, 4 KB apart
// 18.6 ms, and 14.9-17.3 ms as the pair moved through one 2 MB page — until
// log chunks were claimed in pairs (kChunkClaim): 14.9-15.1 ms wherever
// they land (profiles/micro_lr_chains_r02.txt).
constexpr size_t kCtrJobs = 0, kCtrChunks = 256 / 8, kCtrBytes = 512;  // u64 slots, bytes

// Successor reads are random: load them L2-only (.cg).  The read-only
// (.nc / __ldg) path promotes every L1 miss to a full 128-byte line, i.e.
// four 32-byte sectors of DRAM traffic for one useful 4-byte successor.
__device__ __forceinline__ int64_t ld_succ(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int64_t ld_succ(const int64_t* p) {
  int64_t v;
  asm volatile("ld.global.cg.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void st_stream(uint64_t* p, uint64_t v) {
  asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename S, bool WEIGHTED>
__global__ void __launch_bounds__(128)
    lr_walk_kernel(const S* __restrict__ succ, const int64_t* __restrict__ w, int64_t n, int64_t head,
                   int64_t nsub, int64_t extra, uint64_t* __restrict__ tmp, int64_t* __restrict__ nxt,
                   int64_t* __restrict__ len, unsigned long long* __restrict__ err,
                   unsigned long long* __restrict__ jobs, int ks) {
  // jobs != nullptr: sublists are claimed from a global counter as chains
  // free up (dynamic balance: a thread's walks are geometric-length, so a
  // static stride leaves stragglers); else the static stride t, t+T, ...
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  int64_t job = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // next sublist to start
  int64_t j[kChains], cur[kChains], acc[kChains], steps[kChains];
  auto start = [&](int c) {
    for (;;) {
      const int64_t jj = jobs ? (int64_t)atomicAdd(jobs, 1ull) : job;
      if (jj >= nsub) break;
      job += T;
      const int64_t h = jj == extra ? head : jj << ks;
      if (h >= n) {
        nxt[jj] = -1;
        len[jj] = 0;
        continue;
      }
      tmp[h] = (uint64_t)jj << 32;
      j[c] = jj;
      acc[c] = WEIGHTED ? w[h] : 1;
      cur[c] = ld_succ(succ + h);
      steps[c] = 0;
      return;
    }
    j[c] = -1;
  };
#pragma unroll
  for (int c = 0; c < kChains; ++c) start(c);
  while (true) {
    bool any = false;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (j[c] < 0) continue;
      any = true;
      const int64_t v = cur[c];
      if (v == -1 || is_head(v, head, ks) || steps[c] > n) {
        if (steps[c] > n) atomicAdd(err, 1ull);  // cycle without a sublist head
        nxt[j[c]] = (v == -1 || steps[c] > n) ? -1 : sub_id(v, head, extra, ks);
        // a runaway walk reports more weight than the whole list holds, so a
        // chain check on the summaries alone (sharded ranking) still fails
        len[j[c]] = steps[c] > n ? n + 1 : acc[c];
        start(c);
        continue;
      }
      st_stream(tmp + v, ((uint64_t)j[c] << 32) | (uint64_t)(uint32_t)acc[c]);
      acc[c] += WEIGHTED ? w[v] : 1;
      cur[c] = ld_succ(succ + v);
      ++steps[c];
    }
    if (!any) break;
  }
}

// ---------------------------------------------------------------- level-0 log walk
// The level-0 walk of the plain path writes (sublist, offset) to a RANDOM
// node slot per node.  On B200 a scattered 8-byte store costs a sector
// read-modify-write in DRAM (HBM3e has no write mask) and the L2 does not
// merge separate partial stores to one sector, however local they are
// (profiles/micro_scatter_window_r02.txt): ~55 B of DRAM traffic per node.
// The log walk instead appends (node, offset) to per-thread 32-entry chunks
// of a sequential log (chunk ids from one counter; each chunk opens with a
// marker holding its sublist id, and every walk start writes a marker).
// The walk also counts the node sort's digit histograms.  After the sublist
// chain is ranked, the library's radix sort orders the log by the node bits
// above 2^13-node buckets — coalesced passes, the first reading each log
// slot as its packed (rank, node) pair (log_slot_pair) — and
// lr_bucket_finish_kernel writes each bucket's ranks into rank[] through
// shared memory.  (Without the atomics ranking: lr_log_pairs_kernel, a full
// key sort and lr_widen_kernel.)
constexpr int kLogChunk = kLogChunkSlots;  // the log format: common.cuh
constexpr int kChunkClaim = 2;  // log chunks per counter claim
constexpr uint32_t kMarkBit = kLogMark;
constexpr uint32_t kEmptyHi = kLogEmpty;
constexpr int64_t kLogMin = 1 << 20;  // smaller lists: the plain walk (everything fits in L2)

template <typename S>
__global__ void __launch_bounds__(128)
    lr_walk_log_kernel(const S* __restrict__ succ, int64_t n, int64_t head, int64_t nsub, int64_t extra,
                       uint64_t* __restrict__ log, unsigned long long* __restrict__ chunk_ctr, int64_t max_chunks,
                       int64_t* __restrict__ nxt, int64_t* __restrict__ len, unsigned long long* __restrict__ err,
                       unsigned long long* __restrict__ jobs, uint32_t* __restrict__ hist, int hshift, int hpasses) {
  // Entries are held back in registers and stored 4 at a time (one full
  // 32-byte sector as two 16-byte stores issued together): a sector filled
  // entry by entry over microseconds would be evicted part-written and cost
  // a DRAM read-modify-write (no write mask on HBM3e).  Chunks are 256-byte
  // aligned, so every group of 4 slots is one sector.
  // the node sort's digit histograms (digits at hshift + 8d, d < hpasses) of
  // every slot written, so the sort needs no counting pass over the log
  __shared__ uint32_t hcount[2][256];
  for (int i = threadIdx.x; i < 2 * 256; i += blockDim.x) (&hcount[0][0])[i] = 0;
  __syncthreads();
  auto count = [&](uint32_t hi, uint32_t times) {
    const uint32_t key = (hi & kMarkBit) ? 0xffffffffu : hi;
    atomicAdd(&hcount[0][(key >> hshift) & 255u], times);
    if (hpasses > 1) atomicAdd(&hcount[1][(key >> (hshift + 8)) & 255u], times);
  };
  int64_t cbase = 0;
  int fill = kLogChunk;  // no chunk yet
  bool overflow = false;
  uint64_t b0 = 0, b1 = 0, b2 = 0, b3 = 0;
  int nb = 0;
  auto push = [&](uint64_t e) {  // next slot of the current chunk
    count((uint32_t)(e >> 32), 1u);
    if (nb == 0) b0 = e;
    else if (nb == 1) b1 = e;
    else if (nb == 2) b2 = e;
    else b3 = e;
    ++nb;
    ++fill;
    if (nb == 4) {
      uint64_t* p = log + cbase + fill - 4;
      asm volatile("st.global.cs.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(b0), "l"(b1) : "memory");
      asm volatile("st.global.cs.v2.u64 [%0], {%1, %2};" ::"l"(p + 2), "l"(b2), "l"(b3) : "memory");
      nb = 0;
    }
  };
  // Chunks are claimed kChunkClaim at a time.  One at a time, the chunk and
  // sublist counters take ~13M returning atomics per 2^28-node walk, enough
  // to queue at their L2 slices, and the walk then runs 14.9-17.6 ms
  // depending on which slices the counters land on; claiming chunks in pairs
  // makes it 14.9 ms wherever they land (claiming sublists in pairs instead
  // is slower, 18.6 ms; profiles/micro_lr_chains_r02.txt).
  int64_t spare = -1, spare_end = -1;  // claimed chunks not yet opened: [spare, spare_end)
  auto put = [&](uint64_t e, uint32_t j) {
    if (fill == kLogChunk) {
      int64_t c = spare;
      if (c >= 0) {
        if (++spare >= spare_end) spare = -1;
      } else {
        c = (int64_t)atomicAdd(chunk_ctr, (unsigned long long)kChunkClaim);
        if (c >= max_chunks) {
          overflow = true;
          return;
        }
        spare_end = c + kChunkClaim < max_chunks ? c + kChunkClaim : max_chunks;
        spare = c + 1 < spare_end ? c + 1 : -1;
      }
      cbase = c * kLogChunk;
      fill = 0;
      push((uint64_t)(kMarkBit | j) << 32);
    }
    push(e);
  };
  auto walk = [&](int64_t jj) {
    const int64_t h = jj == extra ? head : jj * kK;
    if (h >= n) {
      nxt[jj] = -1;
      len[jj] = 0;
      return;
    }
    const uint32_t j = (uint32_t)jj;
    if (fill < kLogChunk && fill > 0) push((uint64_t)(kMarkBit | j) << 32);  // a new walk inside the chunk: its marker
    put((uint64_t)h << 32, j);
    int64_t acc = 1, steps = 0;
    int64_t v = ld_succ(succ + h);
    while (v != -1 && !is_head(v, head, kKShift) && steps <= n) {
      put(((uint64_t)v << 32) | (uint64_t)(uint32_t)acc, j);
      ++acc;
      ++steps;
      v = ld_succ(succ + v);
    }
    if (steps > n) atomicAdd(err, 1ull);  // cycle without a sublist head
    nxt[jj] = (v == -1 || steps > n) ? -1 : sub_id(v, head, extra, kKShift);
    len[jj] = steps > n ? n + 1 : acc;
  };
  for (;;) {
    const int64_t jj = (int64_t)atomicAdd(jobs, 1ull);
    if (jj >= nsub || overflow) break;
    walk(jj);
  }
  if (overflow) atomicAdd(err, 1ull);
  if (!overflow) {
    while (fill > 0 && fill < kLogChunk) push((uint64_t)kEmptyHi << 32);  // pad (and flush) the last chunk
    for (; spare >= 0 && spare < spare_end; ++spare) {  // claimed chunks never opened: all padding
      const ulonglong2 pad = make_ulonglong2((uint64_t)kEmptyHi << 32, (uint64_t)kEmptyHi << 32);
      ulonglong2* p = reinterpret_cast<ulonglong2*>(log + spare * kLogChunk);
#pragma unroll
      for (int k = 0; k < kLogChunk / 2; ++k) __stcs(p + k, pad);
      count(kEmptyHi, kLogChunk);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < hpasses * 256; i += blockDim.x) {
    const uint32_t c = (&hcount[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

// log slot → (key = node, val = prefix[sublist] + offset); markers and
// padding → key 0xffffffff (sorted behind every node)
__global__ void lr_log_pairs_kernel(const uint64_t* __restrict__ log, int64_t slots, const int64_t* __restrict__ prefix,
                                    uint32_t* __restrict__ key, uint32_t* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const uint32_t le = (2u << lane) - 1u;  // lanes <= me
  // warps cover whole chunks (32 slots): blockDim is a multiple of 32, slots of kLogChunk
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i - lane < slots;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t e = i < slots ? __ldcs(reinterpret_cast<const unsigned long long*>(log) + i) : ((uint64_t)kEmptyHi << 32);
    const uint32_t hi = (uint32_t)(e >> 32);
    const bool mark = (hi & kMarkBit) && hi != kEmptyHi;
    const uint32_t mb = __ballot_sync(0xffffffffu, mark);
    const int src = 31 - __clz(mb & le);
    const uint32_t j = __shfl_sync(0xffffffffu, hi & ~kMarkBit, src < 0 ? 0 : src);
    if (i < slots) {
      const bool node = !(hi & kMarkBit);
      key[i] = node ? hi : 0xffffffffu;
      val[i] = node ? (uint32_t)(prefix[j] + (int64_t)(uint32_t)e) : 0u;
    }
  }
}

// The node sort's finish.  The pairs are ordered by the node bits above BB
// (and the markers / padding, key 0xffffffff, behind every node), and a
// valid list has exactly one pair per node, so positions [b * 2^BB,
// (b + 1) * 2^BB) hold exactly the nodes of bucket b: one CTA per bucket
// places their ranks in shared memory by the low node bits and writes the
// bucket's slice of rank[] coalesced.  This replaces the LSD passes over the
// low bits (a random 8-byte store to rank[] would cost a DRAM sector
// read-modify-write, micro_scatter_window_r02.txt).  BB = 13 (64 KB of
// shared memory per CTA), 14 where that saves a digit pass (2^29 nodes).
constexpr int kBucketThreads = 512;
template <int BB>
__global__ void __launch_bounds__(kBucketThreads) lr_bucket_finish_kernel(const uint64_t* __restrict__ pairs, int64_t n,
                                                                          int64_t* __restrict__ rank,
                                                                          unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) int64_t s_rank[];
  constexpr int S = 1 << BB;
  const int64_t lo = (int64_t)blockIdx.x * S;
  const int cnt = (int)min((int64_t)S, n - lo);
  const ulonglong2* src = reinterpret_cast<const ulonglong2*>(pairs + lo);
  bool bad = false;
  // 16-byte loads (lo is a multiple of 8192 pairs); a ragged last bucket's odd tail pair alone
  for (int i = threadIdx.x; 2 * i < cnt; i += kBucketThreads) {
    ulonglong2 two;
    if (2 * i + 1 < cnt) {
      two = __ldcs(src + i);
    } else {
      two.x = __ldcs(reinterpret_cast<const unsigned long long*>(pairs) + lo + 2 * i);
      two.y = ~0ull;
    }
    const uint32_t k0 = (uint32_t)two.x, k1 = (uint32_t)two.y;
    if ((int64_t)(k0 >> BB) != (int64_t)blockIdx.x) bad = true;
    else s_rank[k0 & (S - 1)] = (int64_t)(two.x >> 32);
    if (2 * i + 1 < cnt) {
      if ((int64_t)(k1 >> BB) != (int64_t)blockIdx.x) bad = true;
      else s_rank[k1 & (S - 1)] = (int64_t)(two.y >> 32);
    }
  }
  if (bad) atomicAdd(err, 1ull);
  __syncthreads();
  longlong2* dst = reinterpret_cast<longlong2*>(rank + lo);
  for (int i = threadIdx.x; 2 * i < cnt; i += kBucketThreads) {
    if (2 * i + 1 < cnt) __stcs(dst + i, make_longlong2(s_rank[2 * i], s_rank[2 * i + 1]));
    else rank[lo + 2 * i] = s_rank[2 * i];
  }
}

__global__ void lr_widen_kernel(const uint32_t* __restrict__ val, int64_t n, int64_t* __restrict__ rank) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    rank[i] = (int64_t)val[i];
}

// rank[v] = prefix[sublist] + local
__global__ void lr_expand_kernel(const uint64_t* __restrict__ tmp, int64_t n,
                                 const int64_t* __restrict__ prefix, int64_t* __restrict__ out) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t t = tmp[v];
    out[v] = prefix[t >> 32] + (int64_t)(t & 0xffffffffull);
  }
}

// Top level, one CTA: weighted Wyllie pointer jumping in shared memory.
// prefix[j] = sum of len over the chain from `head` up to (excluding) j.
// status[0] = chain total from head, status[1] = 1 if a cycle was found.
__global__ void __launch_bounds__(1024)
    lr_top_kernel(const int64_t* __restrict__ nxt_in, const int64_t* __restrict__ len, int64_t m,
                  int64_t head, int64_t* __restrict__ prefix, int64_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char top_smem[];
  int64_t(*val)[kBase] = reinterpret_cast<int64_t(*)[kBase]>(top_smem);
  int32_t(*nxt)[kBase] = reinterpret_cast<int32_t(*)[kBase]>(top_smem + 2 * kBase * sizeof(int64_t));
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    nxt[0][i] = (int32_t)nxt_in[i];
    val[0][i] = len[i];
  }
  __syncthreads();
  int cur = 0;
  int rounds = 0;
  while ((1ll << rounds) < 2 * m) {
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const int32_t nx = nxt[cur][i];
      if (nx >= 0) {
        val[cur ^ 1][i] = val[cur][i] + val[cur][nx];
        nxt[cur ^ 1][i] = nxt[cur][nx];
      } else {
        val[cur ^ 1][i] = val[cur][i];
        nxt[cur ^ 1][i] = -1;
      }
    }
    __syncthreads();
    cur ^= 1;
    ++rounds;
  }
  // val = suffix sums; a remaining successor means a cycle
  __shared__ int cyc;
  if (threadIdx.x == 0) cyc = 0;
  __syncthreads();
  const int64_t total = val[cur][head];
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    if (nxt[cur][i] >= 0) cyc = 1;
    prefix[i] = total - val[cur][i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    status[0] = total;
    status[1] = cyc;
  }
}

constexpr size_t kTopSmem = 2 * kBase * (sizeof(int64_t) + sizeof(int32_t));

struct Level {
  DevBuf tmp, nxt, len, ranked;
  int64_t n = 0, nsub = 0, extra = -1, head = 0;
  // level 0 with the log walk
  bool logged = false;
  DevBuf log, ctr, key, hist;
  int64_t max_chunks = 0;
  int sort_shift = 0, sort_passes = 0, bucket_bits = 0;  // the node sort (bucket finish)
  int ks = 0;  // sublist spacing 2^ks
};

// Rank the list `succ` (n nodes, first node `head`): out_rank[v] = sum of the
// weights of the nodes before v on the chain (w0 == nullptr: unit weights,
// i.e. the distance from the head).  The chain must cover weight `expect`
// in total (n for unit weights), else HB_ESTRUCT.
template <typename S>
int rank_levels(const S* succ, const int64_t* w0, int64_t n, int64_t head, int64_t expect, int64_t* out_rank,
                cudaStream_t s) {
  DeviceInfo di;
  HB_TRY(device_info(&di));
  DevBuf err, st;
  HB_TRY(alloc(&err, 8, s));
  HB_CUDA_TRY(cudaMemsetAsync(err.ptr, 0, 8, s));
  std::vector<Level*> levels;
  struct Cleanup {
    std::vector<Level*>& v;
    ~Cleanup() {
      for (auto* l : v) delete l;
    }
  } cleanup{levels};

  // descend: level 0 walks the input list, later levels walk the sublist lists
  const int64_t* w = w0;
  const void* cur_succ = succ;
  bool first = true;
  int64_t cur_n = n, cur_head = head;
  while (cur_n > kBase) {
    Level* L = new Level();
    levels.push_back(L);
    L->n = cur_n;
    L->head = cur_head;
    const int ks = first ? kKShift : kUpperShift;  // sublist spacing 2^ks
    L->ks = ks;
    const int64_t regular = ceil_div(cur_n, (int64_t)1 << ks);
    L->extra = (cur_head & (((int64_t)1 << ks) - 1)) == 0 ? -1 : regular;
    L->nsub = regular + (L->extra >= 0 ? 1 : 0);
    L->logged = first && w0 == nullptr && cur_n >= kLogMin && cur_n <= (1ll << 29);  // sort size < 2^30
    if (L->logged) {
      // every full chunk holds >= 31 node / walk-start entries; plus one partial chunk per thread
      L->max_chunks = (cur_n + L->nsub) / (kLogChunk - 1) + (int64_t)di.sms * 16 * 128 * kChunkClaim + 64;
      // log + the sort's second buffer allocated together, up front: the same
      // allocation pattern every call keeps the stream-ordered pool from growing
      HB_TRY(alloc(&L->log, (size_t)L->max_chunks * kLogChunk * 8, s));
      HB_TRY(alloc(&L->key, (size_t)L->max_chunks * kLogChunk * 8, s));
      HB_TRY(alloc(&L->ctr, 8, s));
      HB_CUDA_TRY(cudaMemsetAsync(L->ctr.ptr, 0, 8, s));
      // The node sort orders the (rank, node) pairs by the node bits above a
      // 2^bucket_bits-node bucket (2^13; 2^14 where that saves a pass) and up
      // to bit nb, nodes < 2^nb: markers and padding (key 0xffffffff) have
      // bit nb set and sort behind every node.
      int nb = 1;
      while (((int64_t)1 << nb) < cur_n) ++nb;
      L->bucket_bits = 13;
      L->sort_passes = std::max(1, (nb + 1 - 13 + 7) / 8);
      if (L->sort_passes > 1 && (nb + 1 - 14 + 7) / 8 < L->sort_passes) {
        L->bucket_bits = 14;
        --L->sort_passes;
      }
      L->sort_shift = nb + 1 - 8 * L->sort_passes;
      HB_TRY(alloc(&L->hist, 2 * 256 * 4, s));
      HB_CUDA_TRY(cudaMemsetAsync(L->hist.ptr, 0, 2 * 256 * 4, s));
    } else if (first) {
      L->tmp.ptr = out_rank;  // packed (sublist, offset) lives in the output until expanded
      L->tmp.owned = false;
    } else {
      HB_TRY(alloc(&L->tmp, (size_t)cur_n * 8, s));
    }
    HB_TRY(alloc(&L->nxt, (size_t)L->nsub * 8, s));
    HB_TRY(alloc(&L->len, (size_t)L->nsub * 8, s));
    int64_t blocks = ceil_div(L->nsub, 128 * kChains);
    if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;  // 2048 resident threads / SM
    DevBuf jobs;  // dynamic sublist claiming (+1 % over a static stride: 12.62 vs 12.49 Gnodes/s)
    HB_TRY(alloc(&jobs, kCtrBytes, s));  // [kCtrJobs] sublist claims, [kCtrChunks] log-chunk claims
    HB_CUDA_TRY(cudaMemsetAsync(jobs.ptr, 0, kCtrBytes, s));
    if (L->logged) {
      // Fewer walks in flight than the SMs could hold: 3.6 blocks of 128
      // per SM (~68K walks) from 2^27 nodes up — 14.9 vs 16.9 ms per
      // 2^28-node call and 29.5 vs 33.3 ms at 2^29 against one walk per
      // resident thread; 4 blocks/SM is faster in some processes (14.6) and
      // 16.8-17.2 ms in others, 3.6 was 14.9-15.1 in every process measured — and
      // 6 blocks/SM below 2^27 (3.67 vs 4.06 ms at 2^26, 1.42 vs 1.54 at
      // 2^24; neutral at 2^20-2^22).  profiles/micro_lr_chains_r02.txt.
      blocks = std::min<int64_t>(blocks, cur_n >= ((int64_t)1 << 27) ? (int64_t)di.sms * kWalkBlocksPer10Sm / 10
                                                                      : (int64_t)di.sms * 6);
      unsigned long long* ctr = jobs.as<unsigned long long>();
      lr_walk_log_kernel<S><<<(int)blocks, 128, 0, s>>>(
          (const S*)cur_succ, cur_n, cur_head, L->nsub, L->extra, L->log.as<uint64_t>(),
          ctr + kCtrChunks, L->max_chunks, L->nxt.as<int64_t>(), L->len.as<int64_t>(),
          err.as<unsigned long long>(), ctr + kCtrJobs, L->hist.as<uint32_t>(), L->sort_shift, L->sort_passes);
      // the chunk count the pairs pass reads back
      HB_CUDA_TRY(cudaMemcpyAsync(L->ctr.ptr, ctr + kCtrChunks, 8, cudaMemcpyDeviceToDevice, s));
    } else if (first && w0 != nullptr) {
      lr_walk_kernel<S, true><<<(int)blocks, 128, 0, s>>>(
          (const S*)cur_succ, w0, cur_n, cur_head, L->nsub, L->extra, L->tmp.as<uint64_t>(),
          L->nxt.as<int64_t>(), L->len.as<int64_t>(), err.as<unsigned long long>(), jobs.as<unsigned long long>(), ks);
    } else if (first) {
      lr_walk_kernel<S, false><<<(int)blocks, 128, 0, s>>>(
          (const S*)cur_succ, nullptr, cur_n, cur_head, L->nsub, L->extra, L->tmp.as<uint64_t>(),
          L->nxt.as<int64_t>(), L->len.as<int64_t>(), err.as<unsigned long long>(), jobs.as<unsigned long long>(), ks);
    } else {
      lr_walk_kernel<int64_t, true><<<(int)blocks, 128, 0, s>>>(
          (const int64_t*)cur_succ, w, cur_n, cur_head, L->nsub, L->extra, L->tmp.as<uint64_t>(),
          L->nxt.as<int64_t>(), L->len.as<int64_t>(), err.as<unsigned long long>(), jobs.as<unsigned long long>(), ks);
    }
    HB_TRY(check_launch());
    cur_succ = L->nxt.ptr;
    w = L->len.as<int64_t>();
    cur_head = L->extra >= 0 ? L->extra : cur_head >> ks;
    cur_n = L->nsub;
    first = false;
  }

  // top level
  DevBuf top_nxt, top_len, top_prefix;
  if (first) {  // the whole list is small: rank it directly (unit weights)
    HB_TRY(alloc(&top_nxt, (size_t)cur_n * 8, s));
    HB_TRY(alloc(&top_len, (size_t)cur_n * 8, s));
    std::vector<int64_t> ones((size_t)cur_n, 1);
    if (w0 != nullptr)
      HB_CUDA_TRY(cudaMemcpyAsync(ones.data(), w0, (size_t)cur_n * 8, cudaMemcpyDeviceToHost, s));
    std::vector<int64_t> nx((size_t)cur_n);
    std::vector<S> sh((size_t)cur_n);
    HB_CUDA_TRY(cudaMemcpyAsync(sh.data(), succ, (size_t)cur_n * sizeof(S), cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < cur_n; ++i) nx[(size_t)i] = (int64_t)sh[(size_t)i];
    HB_CUDA_TRY(cudaMemcpyAsync(top_nxt.ptr, nx.data(), (size_t)cur_n * 8, cudaMemcpyHostToDevice, s));
    HB_CUDA_TRY(cudaMemcpyAsync(top_len.ptr, ones.data(), (size_t)cur_n * 8, cudaMemcpyHostToDevice, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
  } else {
    top_nxt.ptr = const_cast<void*>(cur_succ);
    top_len.ptr = const_cast<int64_t*>(w);
  }
  HB_TRY(alloc(&top_prefix, (size_t)cur_n * 8, s));
  HB_TRY(alloc(&st, 16, s));
  HB_CUDA_TRY(cudaFuncSetAttribute(lr_top_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTopSmem));
  lr_top_kernel<<<1, 1024, kTopSmem, s>>>(top_nxt.as<int64_t>(), top_len.as<int64_t>(), cur_n, cur_head,
                                   top_prefix.as<int64_t>(), st.as<int64_t>());
  HB_TRY(check_launch());
  int64_t status[2] = {0, 0};
  unsigned long long errs = 0;
  HB_CUDA_TRY(cudaMemcpyAsync(status, st.ptr, 16, cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaMemcpyAsync(&errs, err.ptr, 8, cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaStreamSynchronize(s));
  if (errs || status[1]) {
    set_error("list contains a cycle");
    return HB_ESTRUCT;
  }
  if (status[0] > expect) {
    set_error("list contains a cycle");
    return HB_ESTRUCT;
  }
  if (status[0] != expect) {
    set_error("chain covers %lld of %lld nodes (broken list)", (long long)status[0], (long long)expect);
    return HB_ESTRUCT;
  }

  // ascend: expand every level's packed offsets
  const int64_t* prefix = top_prefix.as<int64_t>();
  if (first) {
    // rank = prefix of the unit-weight top list
    HB_CUDA_TRY(cudaMemcpyAsync(out_rank, prefix, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
    return HB_OK;
  }
  for (int li = (int)levels.size() - 1; li >= 0; --li) {
    Level* L = levels[(size_t)li];
    int64_t* dst;
    if (li == 0) {
      dst = out_rank;
    } else {
      HB_TRY(alloc(&L->ranked, (size_t)L->n * 8, s));
      dst = L->ranked.as<int64_t>();
    }
    if (L->logged) {
      unsigned long long used = 0;
      HB_CUDA_TRY(cudaMemcpyAsync(&used, L->ctr.ptr, 8, cudaMemcpyDeviceToHost, s));
      HB_CUDA_TRY(cudaStreamSynchronize(s));
      const int64_t slots = (int64_t)std::min<unsigned long long>(used, (unsigned long long)L->max_chunks) * kLogChunk;
      {  // the node sort over the bits above the buckets — its first pass reads the log — and the bucket finish
        uint64_t* sorted = nullptr;
        const int rc = sort_pairs_bits_ext(L->log.as<uint64_t>(), slots, L->hist.as<uint32_t>(), L->sort_shift,
                                           L->sort_passes, prefix, L->key.as<uint64_t>(), &sorted, s);
        if (rc == HB_OK) {
          const int bb = L->bucket_bits;
          const size_t smem = sizeof(int64_t) << bb;
          auto k = bb == 14 ? lr_bucket_finish_kernel<14> : lr_bucket_finish_kernel<13>;
          HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          HB_CUDA_TRY(cudaMemsetAsync(err.ptr, 0, 8, s));
          k<<<(unsigned)ceil_div(L->n, (int64_t)1 << bb), kBucketThreads, smem, s>>>(sorted, L->n, dst,
                                                                                     err.as<unsigned long long>());
          HB_TRY(check_launch());
          unsigned long long bad = 0;
          HB_CUDA_TRY(cudaMemcpyAsync(&bad, err.ptr, 8, cudaMemcpyDeviceToHost, s));
          HB_CUDA_TRY(cudaStreamSynchronize(s));
          if (bad) {
            set_error("node sort: %llu bucket(s) hold a foreign node (internal error)", bad);
            return HB_ECUDA;
          }
          prefix = dst;
          continue;
        }
        if (rc != HB_ENOSYS) return rc;
      }
      int64_t pb = ceil_div(slots, 256);
      if (pb > (int64_t)di.sms * 16) pb = (int64_t)di.sms * 16;
      uint32_t* key = L->key.as<uint32_t>();  // (node, rank) as two u32 arrays in the sort buffer
      uint32_t* val = key + slots;
      // general path (ballot-ranked sorts): (node, rank) as two arrays, sort, widen
      lr_log_pairs_kernel<<<(int)pb, 256, 0, s>>>(L->log.as<uint64_t>(), slots, prefix, key, val);
      HB_TRY(check_launch());
      // order the pairs by node: the first n keys are 0..n-1 (a valid list has
      // one log entry per node; the chain check above guarantees it)
      HB_TRY(hb_sort(key, key, HB_U32, val, val, slots, nullptr, HB_DEVICE_PTRS | HB_ASYNC, s));
      int64_t wb = ceil_div(L->n, 256);
      if (wb > (int64_t)di.sms * 16) wb = (int64_t)di.sms * 16;
      lr_widen_kernel<<<(int)wb, 256, 0, s>>>(val, L->n, dst);
      HB_TRY(check_launch());
      prefix = dst;
      continue;
    }
    int64_t blocks = ceil_div(L->n, 256);
    if (blocks > (int64_t)di.sms * 32) blocks = (int64_t)di.sms * 32;
    lr_expand_kernel<<<(int)blocks, 256, 0, s>>>(L->tmp.as<uint64_t>(), L->n, prefix, dst);
    HB_TRY(check_launch());
    prefix = dst;
  }
  return HB_OK;
}

// Sharded ranking, expansion: own sublists [lo, hi) → rank, others → 0
// (the packed slots of nodes walked by other ranks still hold the 0xFF..
// fill, sublist id 0xffffffff, which no rank owns).
__global__ void lr_expand_part_kernel(int64_t* __restrict__ io, int64_t n, const int64_t* __restrict__ prefix,
                                      int64_t lo, int64_t hi) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t t = (uint64_t)io[v];
    const int64_t j = (int64_t)(t >> 32);
    io[v] = (j >= lo && j < hi) ? prefix[j] + (int64_t)(t & 0xffffffffull) : 0;
  }
}

// the same expansion into int32 ranks (n < 2^31): the all-reduce that
// merges the ranks of all GPUs then moves half the bytes
__global__ void lr_expand_part32_kernel(const int64_t* __restrict__ packed, int64_t n,
                                        const int64_t* __restrict__ prefix, int64_t lo, int64_t hi,
                                        int32_t* __restrict__ out) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t t = (uint64_t)packed[v];
    const int64_t j = (int64_t)(t >> 32);
    out[v] = (j >= lo && j < hi) ? (int32_t)(prefix[j] + (int64_t)(t & 0xffffffffull)) : 0;
  }
}

__global__ void widen_i32_kernel(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)in[i];
}

void lr_layout(int64_t n, int64_t head, int64_t* nsub, int64_t* sub_head) {
  const int64_t regular = ceil_div(n, kK);
  const bool extra = head % kK != 0;
  *nsub = regular + (extra ? 1 : 0);
  *sub_head = extra ? regular : head / kK;
}

// validate_list's range check + tail count (kernels_irregular.py:377-393)
template <typename S>
int check_list(const S* succ, int64_t n, cudaStream_t s) {
  DeviceInfo di;
  HB_TRY(device_info(&di));
  DevBuf chk;
  HB_TRY(alloc(&chk, 16, s));
  HB_CUDA_TRY(cudaMemsetAsync(chk.ptr, 0, 16, s));
  int64_t blocks = ceil_div(n, 256);
  if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
  lr_check_kernel<S><<<(int)blocks, 256, 0, s>>>(succ, n, chk.as<unsigned long long>());
  HB_TRY(check_launch());
  unsigned long long c[2] = {0, 0};
  HB_CUDA_TRY(cudaMemcpyAsync(c, chk.ptr, 16, cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaStreamSynchronize(s));
  if (c[1]) {
    set_error("successor index out of range");
    return HB_ESTRUCT;
  }
  if (c[0] != 1) {
    set_error(c[0] == 0 ? "list contains a cycle" : "list has %llu tails (broken list)", c[0]);
    return HB_ESTRUCT;
  }
  return HB_OK;
}

// Sharded ranking, level 1: walk the sublists with ids in [lo, hi) only.
template <typename S>
int walk_part(const S* succ, int64_t n, int64_t head, int64_t lo, int64_t hi, uint64_t* packed, int64_t* nxt,
              int64_t* len, cudaStream_t s) {
  HB_TRY(check_list<S>(succ, n, s));
  DeviceInfo di;
  HB_TRY(device_info(&di));
  int64_t nsub, sub_head;
  lr_layout(n, head, &nsub, &sub_head);
  const int64_t extra = head % kK != 0 ? nsub - 1 : -1;
  HB_CUDA_TRY(cudaMemsetAsync(packed, 0xff, (size_t)n * 8, s));
  if (hi <= lo) return HB_OK;
  DevBuf err, jobs;
  HB_TRY(alloc(&err, 8, s));
  HB_TRY(alloc(&jobs, 8, s));
  const unsigned long long start = (unsigned long long)lo;
  HB_CUDA_TRY(cudaMemsetAsync(err.ptr, 0, 8, s));
  HB_CUDA_TRY(cudaMemcpyAsync(jobs.ptr, &start, 8, cudaMemcpyHostToDevice, s));
  int64_t blocks = ceil_div(hi - lo, 128 * kChains);
  if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
  lr_walk_kernel<S, false><<<(int)blocks, 128, 0, s>>>(succ, nullptr, n, head, hi, extra, packed, nxt, len,
                                                       err.as<unsigned long long>(), jobs.as<unsigned long long>(), kKShift);
  HB_TRY(check_launch());
  return HB_OK;
}

// succ[order[i]] = order[i+1], succ[order[n-1]] = -1 (gen_list, datasets.py:58-63)
template <typename S>
__global__ void link_order_kernel(const int32_t* __restrict__ order, int64_t n, S* __restrict__ succ) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    succ[order[i]] = i + 1 < n ? (S)order[i + 1] : (S)-1;
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hb_link_order(const int32_t* order, int64_t n, void* succ, int succ_code, int flags,
                             void* stream) {
  HB_CHECK_ARG(succ_code == HB_I32 || succ_code == HB_I64, "succ must be int32 or int64");
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_link_order works on device arrays");
  HB_CHECK_ARG(n >= 0 && n < (1ll << 31), "n out of range");
  if (n == 0) return HB_OK;
  DeviceInfo di;
  HB_TRY(device_info(&di));
  cudaStream_t s = as_stream(stream);
  int64_t blocks = ceil_div(n, 256);
  if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
  if (succ_code == HB_I32) link_order_kernel<int32_t><<<(int)blocks, 256, 0, s>>>(order, n, (int32_t*)succ);
  else link_order_kernel<int64_t><<<(int)blocks, 256, 0, s>>>(order, n, (int64_t*)succ);
  return finish(flags, s);
}

extern "C" int hb_list_rank(const void* succ, int succ_code, int64_t n, int64_t head, int64_t* rank,
                            int flags, void* stream) {
  HB_CHECK_ARG(succ_code == HB_I32 || succ_code == HB_I64, "succ must be int32 or int64");
  HB_CHECK_ARG(n >= 1, "list must have at least one node");
  HB_CHECK_ARG(succ && rank, "NULL pointer");
  if (head < 0 || head >= n) {
    set_error("head out of range");
    return HB_ESTRUCT;
  }
  HB_CHECK_ARG(n < (1ll << 31), "lists of up to 2^31-1 nodes are supported");
  const bool dev = flags & HB_DEVICE_PTRS;
  cudaStream_t s = as_stream(stream);
  const size_t se = succ_code == HB_I32 ? 4 : 8;
  DevBuf d_succ, d_rank, chk;
  HB_TRY(stage_in(&d_succ, succ, (size_t)n * se, dev, s));
  HB_TRY(stage_out(&d_rank, rank, (size_t)n * 8, dev, s));
  // structural pre-check (validate_list's range check + tail count)
  DeviceInfo di;
  HB_TRY(device_info(&di));
  HB_TRY(alloc(&chk, 16, s));
  HB_CUDA_TRY(cudaMemsetAsync(chk.ptr, 0, 16, s));
  int64_t blocks = ceil_div(n, 256);
  if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
  if (succ_code == HB_I32) lr_check_kernel<int32_t><<<(int)blocks, 256, 0, s>>>(d_succ.as<int32_t>(), n, chk.as<unsigned long long>());
  else lr_check_kernel<int64_t><<<(int)blocks, 256, 0, s>>>(d_succ.as<int64_t>(), n, chk.as<unsigned long long>());
  HB_TRY(check_launch());
  unsigned long long c[2] = {0, 0};
  HB_CUDA_TRY(cudaMemcpyAsync(c, chk.ptr, 16, cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaStreamSynchronize(s));
  if (c[1]) {
    set_error("successor index out of range");
    return HB_ESTRUCT;
  }
  if (c[0] != 1) {
    set_error(c[0] == 0 ? "list contains a cycle" : "list has %llu tails (broken list)", c[0]);
    return HB_ESTRUCT;
  }
  int rc = succ_code == HB_I32 ? rank_levels<int32_t>(d_succ.as<int32_t>(), nullptr, n, head, n, d_rank.as<int64_t>(), s)
                               : rank_levels<int64_t>(d_succ.as<int64_t>(), nullptr, n, head, n, d_rank.as<int64_t>(), s);
  if (rc != HB_OK) return rc;
  HB_TRY(copy_out(rank, d_rank, (size_t)n * 8, dev, s));
  return finish(flags, s);
}

extern "C" int hb_lr_layout(int64_t n, int64_t head, int64_t* nsub, int64_t* sub_head) {
  HB_CHECK_ARG(n >= 1 && head >= 0 && head < n, "bad list size / head");
  HB_CHECK_ARG(nsub && sub_head, "NULL pointer");
  lr_layout(n, head, nsub, sub_head);
  return HB_OK;
}

extern "C" int hb_lr_walk_part(const void* succ, int succ_code, int64_t n, int64_t head, int64_t sub_lo,
                               int64_t sub_hi, int64_t* packed, int64_t* sub_nxt, int64_t* sub_len, int flags,
                               void* stream) {
  HB_CHECK_ARG(succ_code == HB_I32 || succ_code == HB_I64, "succ must be int32 or int64");
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "the sharded ranking works on device arrays");
  HB_CHECK_ARG(n >= 1 && n < (1ll << 31), "lists of 1 .. 2^31-1 nodes are supported");
  HB_CHECK_ARG(succ && packed && sub_nxt && sub_len, "NULL pointer");
  if (head < 0 || head >= n) {
    set_error("head out of range");
    return HB_ESTRUCT;
  }
  int64_t nsub, sub_head;
  lr_layout(n, head, &nsub, &sub_head);
  HB_CHECK_ARG(0 <= sub_lo && sub_lo <= sub_hi && sub_hi <= nsub, "sublist range out of [0, %lld]", (long long)nsub);
  cudaStream_t s = as_stream(stream);
  int rc = succ_code == HB_I32
               ? walk_part<int32_t>((const int32_t*)succ, n, head, sub_lo, sub_hi, (uint64_t*)packed, sub_nxt, sub_len, s)
               : walk_part<int64_t>((const int64_t*)succ, n, head, sub_lo, sub_hi, (uint64_t*)packed, sub_nxt, sub_len, s);
  if (rc != HB_OK) return rc;
  return finish(flags, s);
}

extern "C" int hb_lr_finish_part32(const int64_t* sub_nxt, const int64_t* sub_len, int64_t nsub,
                                   int64_t sub_head, int64_t n, int64_t sub_lo, int64_t sub_hi,
                                   const int64_t* packed, int32_t* rank32, int flags, void* stream) {
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "the sharded ranking works on device arrays");
  HB_CHECK_ARG(n >= 1 && n <= (int64_t)INT32_MAX + 1 && nsub >= 1 && sub_head >= 0 && sub_head < nsub,
               "bad sublist layout (int32 ranks need n <= 2^31)");
  HB_CHECK_ARG(0 <= sub_lo && sub_lo <= sub_hi && sub_hi <= nsub, "sublist range out of range");
  HB_CHECK_ARG(sub_nxt && sub_len && packed && rank32, "NULL pointer");
  cudaStream_t s = as_stream(stream);
  DevBuf prefix;
  HB_TRY(alloc(&prefix, (size_t)nsub * 8, s));
  HB_TRY(rank_levels<int64_t>(sub_nxt, sub_len, nsub, sub_head, n, prefix.as<int64_t>(), s));
  DeviceInfo di;
  HB_TRY(device_info(&di));
  int64_t blocks = ceil_div(n, 256);
  if (blocks > (int64_t)di.sms * 32) blocks = (int64_t)di.sms * 32;
  lr_expand_part32_kernel<<<(int)blocks, 256, 0, s>>>(packed, n, prefix.as<int64_t>(), sub_lo, sub_hi, rank32);
  return finish(flags, s);
}

extern "C" int hb_widen_i32(const int32_t* in, int64_t n, int64_t* out, int flags, void* stream) {
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_widen_i32 works on device arrays");
  HB_CHECK_ARG(n >= 0 && (n == 0 || (in && out)), "bad arguments");
  if (n == 0) return HB_OK;
  cudaStream_t s = as_stream(stream);
  DeviceInfo di;
  HB_TRY(device_info(&di));
  int64_t blocks = ceil_div(n, 256);
  if (blocks > (int64_t)di.sms * 32) blocks = (int64_t)di.sms * 32;
  widen_i32_kernel<<<(int)blocks, 256, 0, s>>>(in, n, out);
  return finish(flags, s);
}

extern "C" int hb_lr_finish_part(const int64_t* sub_nxt, const int64_t* sub_len, int64_t nsub, int64_t sub_head,
                                 int64_t n, int64_t sub_lo, int64_t sub_hi, int64_t* rank, int flags, void* stream) {
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "the sharded ranking works on device arrays");
  HB_CHECK_ARG(n >= 1 && nsub >= 1 && sub_head >= 0 && sub_head < nsub, "bad sublist layout");
  HB_CHECK_ARG(0 <= sub_lo && sub_lo <= sub_hi && sub_hi <= nsub, "sublist range out of range");
  HB_CHECK_ARG(sub_nxt && sub_len && rank, "NULL pointer");
  cudaStream_t s = as_stream(stream);
  DevBuf prefix;
  HB_TRY(alloc(&prefix, (size_t)nsub * 8, s));
  // rank the sublist chain weighted by the sublist lengths: it must cover all n nodes
  HB_TRY(rank_levels<int64_t>(sub_nxt, sub_len, nsub, sub_head, n, prefix.as<int64_t>(), s));
  DeviceInfo di;
  HB_TRY(device_info(&di));
  int64_t blocks = ceil_div(n, 256);
  if (blocks > (int64_t)di.sms * 32) blocks = (int64_t)di.sms * 32;
  lr_expand_part_kernel<<<(int)blocks, 256, 0, s>>>(rank, n, prefix.as<int64_t>(), sub_lo, sub_hi);
  return finish(flags, s);
}
