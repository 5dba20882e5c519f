// ARCHIVED EXPERIMENT (round 2) — not built into libhb200.so.  Measured
// 134 us per SpMV at the 1M config vs 77 us for spmv_sell_kernel; see
// profiles/micro_spmv_gather_ceiling_r02.txt for the measurements and why
// the design cannot beat the row-ordered kernel by more than ~10-17 %.  To
// rebuild it, copy it into paper_1303_2171_b200/csrc/ and bind the three
// hb_spmv_plan_* entry points (scripts/experiments/test_spmv_colorder.py is
// its parity test: all cases bit-exact on B200).
// spmv_cor.cu — the bit-exact SpMV (reference _csr_range_matvec,
// kernels_irregular.py:206-211) over a COLUMN-ORDERED ROUNDS plan.
//
// Why: on a random sparse matrix every nonzero gathers one x value from a
// random 128-byte line.  The SM's L1 serves about one line (wavefront) per
// clock, gathers and shared-memory accesses alike: a warp gather of 32
// random lines costs 32, of 32 columns inside a 300-column window ~18
// (profiles/micro_gather_lines_r02.txt; LSU and TMA gather4 share that
// ceiling, micro_gather_mix_r02.txt).  The row-per-lane kernels (spmv.cu)
// pay 32 lines per 32 nonzeros.  Processing each SM's nonzeros in COLUMN
// order gives the warp-level locality, at the price of one shared
// read-modify-write of the row sum per nonzero.
//
// Plan (built once per device matrix + row range, on the device):
//   * the rows [row0,row1) are dealt to nc = #SM CTAs round-robin (balanced
//     nnz on the nnz-sorted matrix spmv_preprocess emits); when one CTA's rows
//     exceed kCorRmax, the range is cut into chunks processed one after the
//     other (virtual CTA v = chunk·nc + cta);
//   * each virtual CTA's nonzeros are sorted by column and dealt into ROUNDS of
//     ≤ kCorT entries by a greedy list scheduler: an entry goes to the first
//     round that is ≥ the current fill round, lies after the round of the
//     same row's previous entry, and has room.  So within a round the rows
//     are distinct, and every row's entries sit in strictly increasing rounds
//     in column order — the reference's left-to-right summation order;
//   * entry = (values f64, pk u32 = local row << shift | column − round's
//     first column) — 12 bytes per nonzero like CSR; round header = {start,
//     first column, count}.
// Kernel: one CTA per SM, thread t takes entry t of every round; the row sums
// live in shared memory; round r's products are added after a CTA barrier
// (rounds r−1's adds are done), products and gathers are issued 2 and 4
// rounds ahead.  Every product is one rounded fp64 multiply, every row summed
// from +0.0 with rounded adds in column order: bit-identical to the
// reference's `np.bincount(row_of, weights=values*x[col])`.
#include <stdlib.h>

#include <algorithm>
#include <memory>
#include <vector>

#include "common.cuh"

namespace hb {
namespace {

constexpr int kCorT = 1024;      // threads per CTA == entries per round
constexpr int kCorD = 4;         // rounds whose x gathers + values are in flight ahead of the adds
constexpr int kCorU = 2 * kCorD; // rounds whose packed entries are in flight (register ring)
constexpr int64_t kCorRmax = 8192;  // rows per CTA per chunk: 64 KB of fp64 row sums
constexpr int kCorRing = 1024;   // scheduler: rounds an entry may be deferred ahead of the fill round
constexpr int kCorSlotBits = 11; // scheduler output: round << 11 | slot in round
constexpr int kCorPf = 8;        // rounds of the entry stream prefetched into L2 ahead of its loads

struct CorRound {
  int64_t start;     // first entry
  uint32_t colbase;  // column of the round's first entry (its smallest)
  uint32_t count;    // entries (1..kCorT)
};

struct SpmvPlan {
  int dev = -1;
  int64_t row0 = 0, row1 = 0, nnz = 0, rounds = 0, rpc = 0;
  int nc = 0, chunks = 0, shift = 0;
  int64_t* round_ptr = nullptr;  // nc·chunks + 1
  CorRound* hdr = nullptr;
  uint32_t* pk = nullptr;
  double* val = nullptr;
  ~SpmvPlan() {
    if (round_ptr) cudaFree(round_ptr);
    if (hdr) cudaFree(hdr);
    if (pk) cudaFree(pk);
    if (val) cudaFree(val);
  }
};

__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// x: allocated in L1 (neighbouring columns of a round share lines), kept in L2
__device__ __forceinline__ double ld_x(const double* a, uint64_t pol) {
  double d;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(d) : "l"(a), "l"(pol));
  return d;
}
// the entry stream: read once, no L1 allocation, first out of L2
__device__ __forceinline__ double ld_sv(const double* a, uint64_t pol) {
  double d;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(d) : "l"(a), "l"(pol));
  return d;
}
__device__ __forceinline__ double ld_x_na(const double* a) {
  double d;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(d) : "l"(a));
  return d;
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t ld_sp(const uint32_t* a, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}

// ---------------------------------------------------------------- plan build
// row gr → (virtual CTA, local row): chunk c = off / (nc·rpc), then dealt
// round-robin over the chunk's nc CTAs
__device__ __forceinline__ void cor_place(int64_t off, int nc, int64_t rpc, int64_t* v, int64_t* l) {
  const int64_t per = (int64_t)nc * rpc;
  const int64_t c = off / per, w = off - c * per;
  *v = c * nc + w % nc;
  *l = w / nc;
}

// warp per row: key = (virtual CTA << 32 | column), payload = entry index,
// lrow[e] = the row's local index
__global__ void cor_keys_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t row0,
                                int64_t row1, int nc, int64_t rpc, uint64_t* __restrict__ keys,
                                uint32_t* __restrict__ eidx, uint32_t* __restrict__ lrow) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t base = rp[row0];
  for (int64_t r = row0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < row1; r += warps) {
    int64_t v, l;
    cor_place(r - row0, nc, rpc, &v, &l);
    const int64_t a = rp[r], b = rp[r + 1];
    for (int64_t j = a + lane; j < b; j += 32) {
      const int64_t e = j - base;
      keys[e] = ((uint64_t)v << 32) | (uint32_t)col[j];
      eidx[e] = (uint32_t)e;
      lrow[e] = (uint32_t)l;
    }
  }
}

__global__ void cor_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx, int64_t n,
                               uint32_t* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// seg[v] = first sorted position of virtual CTA v (lower bound of v << 32)
__global__ void cor_segments(const uint64_t* __restrict__ keys, int64_t n, int64_t nv, int64_t* __restrict__ seg) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= nv; v += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t want = (uint64_t)v << 32;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < want) lo = mid + 1;
      else hi = mid;
    }
    seg[v] = lo;
  }
}

// The greedy round scheduler, one warp per virtual CTA (lane 0 decides, the
// warp stages the entry stream through shared memory in batches).  Writes
// ts[p] = round << 11 | slot, per-round counts / first columns into the
// segment's own index range (rounds ≤ entries), rounds per CTA.  err = 1
// when an entry would have to be deferred ≥ kCorRing rounds (a very long row
// inside one CTA's share) — the caller then keeps the SELL kernel.
constexpr int kSchedBatch = 2048;
__global__ void __launch_bounds__(32) cor_schedule_kernel(const uint64_t* __restrict__ keys,
                                                          const uint32_t* __restrict__ lrow_s,
                                                          const int64_t* __restrict__ seg, int64_t rpc,
                                                          uint32_t* __restrict__ ts, uint32_t* __restrict__ rcount,
                                                          uint32_t* __restrict__ rcol, int64_t* __restrict__ nrounds,
                                                          int* __restrict__ err) {
  extern __shared__ uint32_t sm[];
  uint32_t* last = sm;                  // rpc: round of each row's latest entry + 1 (0 = none)
  uint32_t* fill = last + rpc;          // kCorRing
  uint32_t* colb = fill + kCorRing;     // kCorRing
  uint32_t* b_row = colb + kCorRing;    // kSchedBatch
  uint32_t* b_col = b_row + kSchedBatch;
  uint32_t* b_ts = b_col + kSchedBatch;
  const int lane = threadIdx.x;
  const int64_t v = blockIdx.x;
  const int64_t a = seg[v], b = seg[v + 1];
  for (int64_t i = lane; i < rpc; i += 32) last[i] = 0;
  for (int i = lane; i < kCorRing; i += 32) fill[i] = 0;
  __syncwarp();
  uint32_t cur = 0, top = 0;  // fill round; rounds used = top
  bool bad = false;
  for (int64_t p0 = a; p0 < b; p0 += kSchedBatch) {
    const int cnt = (int)min((int64_t)kSchedBatch, b - p0);
    for (int i = lane; i < cnt; i += 32) {
      b_row[i] = lrow_s[p0 + i];
      b_col[i] = (uint32_t)keys[p0 + i];
    }
    __syncwarp();
    if (lane == 0 && !bad) {
      for (int i = 0; i < cnt; ++i) {
        const uint32_t r = b_row[i];
        uint32_t t = max(cur, last[r]);
        while (t - cur < (uint32_t)kCorRing && fill[t % kCorRing] == (uint32_t)kCorT) ++t;
        if (t - cur >= (uint32_t)kCorRing || t >= (1u << (32 - kCorSlotBits)) - 1u) {
          bad = true;
          break;
        }
        const uint32_t s = fill[t % kCorRing]++;
        if (s == 0) colb[t % kCorRing] = b_col[i];
        last[r] = t + 1;
        b_ts[i] = (t << kCorSlotBits) | s;
        if (t + 1 > top) top = t + 1;
        while (fill[cur % kCorRing] == (uint32_t)kCorT) {  // retire full rounds
          rcount[a + cur] = kCorT;
          rcol[a + cur] = colb[cur % kCorRing];
          fill[cur % kCorRing] = 0;
          ++cur;
        }
      }
    }
    bad = __shfl_sync(0xffffffffu, bad, 0);
    __syncwarp();
    if (bad) break;
    for (int i = lane; i < cnt; i += 32) ts[p0 + i] = b_ts[i];
    __syncwarp();
  }
  if (lane == 0) {
    if (bad) {
      atomicExch(err, 1);
      nrounds[v] = 0;
      return;
    }
    for (uint32_t t = cur; t < top; ++t) {  // partially filled tail rounds (all non-empty)
      rcount[a + t] = fill[t % kCorRing];
      rcol[a + t] = colb[t % kCorRing];
    }
    nrounds[v] = top;
  }
}

// round_ptr = exclusive scan of rounds per virtual CTA (nv is small: #SM x chunks)
__global__ void cor_scan_rounds(const int64_t* __restrict__ nrounds, int64_t nv, int64_t* __restrict__ round_ptr) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t run = 0;
  for (int64_t v = 0; v < nv; ++v) {
    round_ptr[v] = run;
    run += nrounds[v];
  }
  round_ptr[nv] = run;
}

// one warp per virtual CTA: round starts (entries keep the CTA's segment
// [seg[v], seg[v+1]) of the output), headers, and the start of each round
// written back over rcount for the fill kernel (as an offset into the segment)
__global__ void cor_headers(const int64_t* __restrict__ seg, const int64_t* __restrict__ round_ptr,
                            const int64_t* __restrict__ nrounds, int64_t nv, uint32_t* __restrict__ rcount,
                            const uint32_t* __restrict__ rcol, CorRound* __restrict__ hdr) {
  const int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (v >= nv || (threadIdx.x & 31) != 0) return;
  const int64_t a = seg[v], nr = nrounds[v], base = round_ptr[v];
  uint32_t run = 0;
  for (int64_t t = 0; t < nr; ++t) {
    const uint32_t c = rcount[a + t];
    CorRound h;
    h.start = a + run;
    h.colbase = rcol[a + t];
    h.count = c;
    hdr[base + t] = h;
    rcount[a + t] = run;  // now: the round's start within the segment
    run += c;
  }
}

__global__ void cor_fill_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ e_s,
                                const uint32_t* __restrict__ lrow_s, const uint32_t* __restrict__ ts,
                                const int64_t* __restrict__ seg, const uint32_t* __restrict__ rstart,
                                const uint32_t* __restrict__ rcol, const double* __restrict__ values, int64_t n,
                                int shift, uint32_t* __restrict__ pk, double* __restrict__ val, int* __restrict__ err) {
  const uint32_t dmax = shift >= 32 ? 0xffffffffu : ((1u << shift) - 1u);
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[p];
    const int64_t v = (int64_t)(k >> 32);
    const uint32_t col = (uint32_t)k;
    const uint32_t t = ts[p] >> kCorSlotBits, s = ts[p] & ((1u << kCorSlotBits) - 1u);
    const int64_t a = seg[v];
    const int64_t q = a + rstart[a + t] + s;
    const uint32_t d = col - rcol[a + t];
    if (d > dmax) atomicExch(err, 2);
    pk[q] = shift >= 32 ? d : ((lrow_s[p] << shift) | d);
    val[q] = values[e_s[p]];
  }
}

// ---------------------------------------------------------------- the SpMV
constexpr int kCorH = 512;  // round headers staged in a shared ring (refilled 256 at a time)

template <typename Q, int EXP>
__global__ void __launch_bounds__(kCorT, 1)
    spmv_cor_kernel(const int64_t* __restrict__ round_ptr, const CorRound* __restrict__ hdr,
                    const uint32_t* __restrict__ pk, const double* __restrict__ sval, const double* __restrict__ x,
                    int64_t row0, int64_t row1, int64_t rpc, int chunks, int shift, const Q* __restrict__ perm,
                    double* __restrict__ y) {
  extern __shared__ double acc[];  // rpc row sums
  __shared__ CorRound s_hdr[kCorH];
  const int tid = threadIdx.x;
  const int nc = gridDim.x;
  const uint64_t keep = pol_evict_last(), once = pol_evict_first();
  const uint32_t dmask = shift >= 32 ? 0xffffffffu : ((1u << shift) - 1u);
  for (int c = 0; c < chunks; ++c) {
    const int64_t v = (int64_t)c * nc + blockIdx.x;
    for (int64_t l = tid; l < rpc; l += kCorT) acc[l] = 0.0;
    const int64_t R0 = round_ptr[v], R1 = round_ptr[v + 1];
    for (int i = tid; i < kCorH && R0 + i < R1; i += kCorT) s_hdr[i] = hdr[R0 + i];
    // the CTA's entries are one contiguous stream in round order: thread 0
    // keeps ~kCorPf rounds of it prefetched into L2, so the register-ring
    // loads below see L2 latency, not DRAM latency
    int64_t pf = 0, e_end = 0;
    auto prefetch_to = [&](int64_t upto) {
      upto = min(upto, e_end);
      while (pf < upto) {
        const int64_t a = pf & ~(int64_t)3, b = min(a + 2048, (upto + 3) & ~(int64_t)3);
        prefetch_l2(pk + a, (uint32_t)(b - a) * 4);
        prefetch_l2(sval + a, (uint32_t)(b - a) * 8);
        pf = b;
      }
    };
    if (tid == 0 && R1 > R0) {
      const CorRound hl = hdr[R1 - 1];
      pf = hdr[R0].start;
      e_end = hl.start + hl.count;
      prefetch_to(pf + (int64_t)kCorPf * kCorT);
    }
    __syncthreads();  // row sums zeroed, first headers staged
    double sink = 0.0;
    uint32_t epk[kCorU], actm = 0;  // packed entries of rounds r..r+U-1, active bits
    double ev[kCorD], xv[kCorD];     // values and gathered x of rounds r..r+D-1
    auto load_entry = [&](int s, int64_t r) {
      actm &= ~(1u << s);
      if (r < R1) {
        const CorRound& h = s_hdr[(r - R0) % kCorH];
        if ((uint32_t)tid < h.count) {
          actm |= 1u << s;
          epk[s] = ld_sp(pk + h.start + tid, once);
        }
      }
    };
    auto load_x = [&](int s, int64_t r) {
      if (actm & (1u << s)) {
        const CorRound& h = s_hdr[(r - R0) % kCorH];
        ev[s % kCorD] = ld_sv(sval + h.start + tid, once);
        if (EXP == 3) xv[s % kCorD] = ld_x_na(x + (h.colbase + (epk[s] & dmask)));
        else if (EXP == 4) xv[s % kCorD] = __ldg(x + (h.colbase + (epk[s] & dmask)));
        else if (EXP >= 7) xv[s % kCorD] = (double)(epk[s] & dmask);
        else xv[s % kCorD] = ld_x(x + (h.colbase + (epk[s] & dmask)), keep);
      }
    };
#pragma unroll
    for (int s = 0; s < kCorU; ++s) load_entry(s, R0 + s);
#pragma unroll
    for (int s = 0; s < kCorD; ++s) load_x(s, R0 + s);
    for (int64_t rb = R0; rb < R1; rb += kCorU) {
#pragma unroll
      for (int j = 0; j < kCorU; ++j) {
        const int64_t r = rb + j;
        if (r >= R1) break;
        if (actm & (1u << j)) {
          const uint32_t row = shift >= 32 ? 0u : (epk[j] >> shift);
          if (EXP == 6) sink = __dadd_rn(sink, __dmul_rn(ev[j % kCorD], xv[j % kCorD]) + row);
          else acc[row] = __dadd_rn(acc[row], __dmul_rn(ev[j % kCorD], xv[j % kCorD]));
        }
        // refill the header ring half that rounds < r have finished with
        // (its rounds' entries were loaded kCorU rounds ago)
        if (((r - R0) & (kCorH / 2 - 1)) == 0 && r > R0 && tid < kCorH / 2) {
          const int64_t rr = r + kCorH / 2 + tid;
          if (rr < R1) s_hdr[(rr - R0) % kCorH] = hdr[rr];
        }
        if (tid == 0 && EXP != 8 && EXP != 10) prefetch_to(pf + kCorT);
        if (EXP == 0 || EXP == 3 || EXP == 4 || EXP == 6 || EXP == 7 || EXP == 8) __syncthreads();  // this round's adds (and header refills) land before the next round's
        if (EXP == 2) asm volatile("bar.sync 0;" ::: "memory");
        load_entry(j, r + kCorU);
        load_x((j + kCorD) % kCorU, r + kCorD);
      }
    }
    if (EXP == 6 && sink == 1.2345) acc[0] = sink;
    __syncthreads();
    const int64_t cstart = (int64_t)c * nc * rpc;
    for (int64_t l = tid; l < rpc; l += kCorT) {
      const int64_t gr = row0 + cstart + l * nc + blockIdx.x;
      if (gr < row1) {
        if (perm) y[perm[gr]] = acc[l];
        else y[gr - row0] = acc[l];
      }
    }
    __syncthreads();
  }
}

inline int carveout_for(size_t smem) {
  const size_t max_smem = 228 * 1024;
  const int pct = (int)((smem * 100 + max_smem - 1) / max_smem);
  return pct > 100 ? 100 : pct;
}

}  // namespace
}  // namespace hb

extern "C" int hb_spmv_plan_build(const int32_t* row_ptr, const int32_t* col_idx, const double* values, int64_t row0,
                                  int64_t row1, int64_t cols, void** plan_out, int64_t* info, int flags,
                                  void* stream) {
  using namespace hb;
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_spmv_plan_build works on device arrays");
  HB_CHECK_ARG(row_ptr && plan_out && info, "NULL pointer");
  HB_CHECK_ARG(row0 >= 0 && row1 >= row0 && cols >= 0, "bad row range");
  *plan_out = nullptr;
  for (int i = 0; i < 8; ++i) info[i] = 0;
  cudaStream_t s = as_stream(stream);
  DeviceInfo di;
  HB_TRY(device_info(&di));
  int64_t ends[2] = {0, 0};
  HB_CUDA_TRY(cudaMemcpyAsync(&ends[0], row_ptr + row0, 4, cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaMemcpyAsync(&ends[1], row_ptr + row1, 4, cudaMemcpyDeviceToHost, s));
  HB_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t base = (int32_t)ends[0], nnz = (int32_t)ends[1] - (int32_t)ends[0];
  const int64_t rows = row1 - row0;
  if (rows == 0 || nnz < 0 || nnz >= ((int64_t)1 << 30) || cols > ((int64_t)1 << 32)) {
    info[6] = 1;  // not planned: caller keeps the SELL kernel
    return HB_OK;
  }
  auto plan = new SpmvPlan();
  std::unique_ptr<SpmvPlan> guard(plan);
  HB_CUDA_TRY(cudaGetDevice(&plan->dev));
  plan->row0 = row0;
  plan->row1 = row1;
  plan->nnz = nnz;
  plan->nc = (int)std::min<int64_t>(di.sms, rows);
  plan->chunks = (int)ceil_div(rows, (int64_t)plan->nc * kCorRmax);
  plan->rpc = ceil_div(rows, (int64_t)plan->nc * plan->chunks);
  int rb = 0;
  while (((int64_t)1 << rb) < plan->rpc) ++rb;
  plan->shift = 32 - rb;
  const int64_t nv = (int64_t)plan->nc * plan->chunks;
  HB_CUDA_TRY(cudaMalloc(&plan->round_ptr, (size_t)(nv + 1) * 8));
  // + 16 entries: the kernel's L2 prefetches round the stream's tail up to 16 bytes
  HB_CUDA_TRY(cudaMalloc(&plan->pk, (size_t)(nnz + 16) * 4));
  HB_CUDA_TRY(cudaMalloc(&plan->val, (size_t)(nnz + 16) * 8));
  if (nnz == 0) {
    HB_CUDA_TRY(cudaMemsetAsync(plan->round_ptr, 0, (size_t)(nv + 1) * 8, s));
  } else {
    DevBuf keys, keys_s, eidx, e_s, lrow, lrow_s, ts, rcount, rcol, seg, nrounds, errb;
    const size_t n = (size_t)nnz;
    HB_TRY(alloc(&keys, n * 8, s));
    HB_TRY(alloc(&keys_s, n * 8, s));
    HB_TRY(alloc(&eidx, n * 4, s));
    HB_TRY(alloc(&e_s, n * 4, s));
    HB_TRY(alloc(&lrow, n * 4, s));
    HB_TRY(alloc(&lrow_s, n * 4, s));
    HB_TRY(alloc(&ts, n * 4, s));
    HB_TRY(alloc(&rcount, n * 4, s));
    HB_TRY(alloc(&rcol, n * 4, s));
    HB_TRY(alloc(&seg, (size_t)(nv + 1) * 8, s));
    HB_TRY(alloc(&nrounds, (size_t)nv * 8, s));
    HB_TRY(alloc(&errb, 4, s));
    HB_CUDA_TRY(cudaMemsetAsync(errb.ptr, 0, 4, s));
    const int g = di.sms * 8;
    cor_keys_kernel<<<g, 256, 0, s>>>(row_ptr, col_idx, row0, row1, plan->nc, plan->rpc, keys.as<uint64_t>(),
                                      eidx.as<uint32_t>(), lrow.as<uint32_t>());
    HB_TRY(check_launch());
    HB_TRY(hb_sort(keys.ptr, keys_s.ptr, HB_U64, eidx.as<uint32_t>(), e_s.as<uint32_t>(), nnz, nullptr,
                   HB_DEVICE_PTRS | HB_ASYNC | HB_SORT_BALLOT, s));
    cor_gather_u32<<<g, 256, 0, s>>>(lrow.as<uint32_t>(), e_s.as<uint32_t>(), nnz, lrow_s.as<uint32_t>());
    cor_segments<<<(unsigned)ceil_div(nv + 1, 256), 256, 0, s>>>(keys_s.as<uint64_t>(), nnz, nv, seg.as<int64_t>());
    HB_TRY(check_launch());
    const size_t ssm = (size_t)plan->rpc * 4 + 2 * kCorRing * 4 + 3 * kSchedBatch * 4;
    HB_CUDA_TRY(cudaFuncSetAttribute(cor_schedule_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
    cor_schedule_kernel<<<(unsigned)nv, 32, ssm, s>>>(keys_s.as<uint64_t>(), lrow_s.as<uint32_t>(), seg.as<int64_t>(),
                                                      plan->rpc, ts.as<uint32_t>(), rcount.as<uint32_t>(),
                                                      rcol.as<uint32_t>(), nrounds.as<int64_t>(), errb.as<int>());
    HB_TRY(check_launch());
    cor_scan_rounds<<<1, 1, 0, s>>>(nrounds.as<int64_t>(), nv, plan->round_ptr);
    int herr = 0;
    HB_CUDA_TRY(cudaMemcpyAsync(&plan->rounds, plan->round_ptr + nv, 8, cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaMemcpyAsync(&herr, errb.ptr, 4, cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    if (herr != 0) {
      info[6] = 2;  // a row too long for the round scheduler's window
      return HB_OK;
    }
    HB_CUDA_TRY(cudaMalloc(&plan->hdr, (size_t)std::max<int64_t>(plan->rounds, 1) * sizeof(CorRound)));
    cor_headers<<<(unsigned)ceil_div(nv, 8), 256, 0, s>>>(seg.as<int64_t>(), plan->round_ptr, nrounds.as<int64_t>(),
                                                           nv, rcount.as<uint32_t>(), rcol.as<uint32_t>(), plan->hdr);
    cor_fill_kernel<<<g, 256, 0, s>>>(keys_s.as<uint64_t>(), e_s.as<uint32_t>(), lrow_s.as<uint32_t>(),
                                      ts.as<uint32_t>(), seg.as<int64_t>(), rcount.as<uint32_t>(), rcol.as<uint32_t>(),
                                      values + base, nnz, plan->shift, plan->pk, plan->val, errb.as<int>());
    HB_TRY(check_launch());
    HB_CUDA_TRY(cudaMemcpyAsync(&herr, errb.ptr, 4, cudaMemcpyDeviceToHost, s));
    HB_CUDA_TRY(cudaStreamSynchronize(s));
    if (herr != 0) {
      info[6] = 3;  // a round spans more columns than the packed entry holds
      return HB_OK;
    }
  }
  HB_CUDA_TRY(cudaStreamSynchronize(s));
  info[0] = plan->chunks;
  info[1] = plan->nc;
  info[2] = plan->rpc;
  info[3] = plan->rounds;
  info[4] = (int64_t)((nv + 1) * 8 + plan->rounds * sizeof(CorRound) + nnz * 12);
  info[5] = nnz;
  *plan_out = guard.release();
  return HB_OK;
}

extern "C" int hb_spmv_plan_run(const void* plan_, const double* x, const void* perm, int perm_code, double* y,
                                int flags, void* stream) {
  using namespace hb;
  HB_CHECK_ARG((flags & HB_DEVICE_PTRS) != 0, "hb_spmv_plan_run works on device arrays");
  HB_CHECK_ARG(plan_ && x && y, "NULL pointer");
  HB_CHECK_ARG(perm == nullptr || perm_code == HB_I32 || perm_code == HB_I64, "perm must be int32 or int64");
  const SpmvPlan* plan = reinterpret_cast<const SpmvPlan*>(plan_);
  int dev = -1;
  HB_CUDA_TRY(cudaGetDevice(&dev));
  HB_CHECK_ARG(dev == plan->dev, "SpMV plan belongs to device %d, current device is %d", plan->dev, dev);
  if (plan->row1 == plan->row0) return HB_OK;
  cudaStream_t s = as_stream(stream);
  const size_t smem = (size_t)plan->rpc * 8;
  if (perm == nullptr || perm_code == HB_I32) {
    static const int exp = getenv("HB_COR_EXP") ? atoi(getenv("HB_COR_EXP")) : 0;
    auto k = exp == 1 ? spmv_cor_kernel<int32_t, 1> : exp == 2 ? spmv_cor_kernel<int32_t, 2>
           : exp == 3 ? spmv_cor_kernel<int32_t, 3> : exp == 4 ? spmv_cor_kernel<int32_t, 4>
           : exp == 6 ? spmv_cor_kernel<int32_t, 6> : exp == 7 ? spmv_cor_kernel<int32_t, 7>
           : exp == 8 ? spmv_cor_kernel<int32_t, 8> : exp == 9 ? spmv_cor_kernel<int32_t, 9>
           : exp == 10 ? spmv_cor_kernel<int32_t, 10> : spmv_cor_kernel<int32_t, 0>;
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_for(smem + sizeof(CorRound) * kCorH + 1024)));
    k<<<plan->nc, kCorT, smem, s>>>(plan->round_ptr, plan->hdr, plan->pk, plan->val, x, plan->row0, plan->row1,
                                    plan->rpc, plan->chunks, plan->shift, reinterpret_cast<const int32_t*>(perm), y);
  } else {
    auto k = spmv_cor_kernel<int64_t, 0>;
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_for(smem + sizeof(CorRound) * kCorH + 1024)));
    k<<<plan->nc, kCorT, smem, s>>>(plan->round_ptr, plan->hdr, plan->pk, plan->val, x, plan->row0, plan->row1,
                                    plan->rpc, plan->chunks, plan->shift, reinterpret_cast<const int64_t*>(perm), y);
  }
  HB_TRY(check_launch());
  return finish(flags, s);
}

extern "C" int hb_spmv_plan_free(void* plan) {
  delete reinterpret_cast<hb::SpmvPlan*>(plan);
  return HB_OK;
}
