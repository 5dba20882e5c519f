/*
 * hb200.h — C ABI of libhb200.so, the B200 (sm_100a) kernels behind the
 * hybridbench work-partitioned hot path (arXiv 1303.2171).
 *
 * Every entry point replaces the DeviceB side of one reference `run_part`
 * (or the equivalent side function) in /root/reference/pkg/src/hybridbench/.
 * The citation above each declaration names the reference interface it
 * replaces.  The Python package paper_1303_2171_b200 binds these through
 * ctypes.CDLL (which releases the GIL, so the two `run_workshared` threads
 * really overlap, cf. worksharing.py:317-320); INTEGRATION.md shows the
 * binding a maintainer of the reference would add.
 *
 * Conventions
 *  - Plain pointers and sizes only.  `stream` is a cudaStream_t passed as
 *    void* (NULL = the legacy default stream of the current device).
 *  - `flags & HB_DEVICE_PTRS`: every data pointer is a device pointer on the
 *    current device.  Otherwise every data pointer is a HOST pointer (pinned
 *    or pageable) and the library stages it through its own device buffers;
 *    host↔device copies then happen inside the call.
 *  - `flags & HB_ASYNC` (device pointers only): return without synchronising
 *    the stream.  Checks that need a device→host read are then skipped.
 *  - Return value: HB_OK, or an HB_E* code; hb_last_error() gives a
 *    thread-local message.  The Python layer maps HB_EINVAL → ValueError,
 *    HB_ESTRUCT → StructuralError, everything else → HybridBenchError
 *    (reference hierarchy: errors.py:10-49).
 */
#ifndef HB200_H
#define HB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_OK 0
#define HB_EINVAL 1   /* argument / domain error      -> ValueError          */
#define HB_ESTRUCT 2  /* malformed structure          -> StructuralError     */
#define HB_ECUDA 3    /* CUDA runtime failure         -> HybridBenchError    */
#define HB_ENOMEM 4   /* device allocation failed     -> HybridBenchError    */
#define HB_ENOSYS 5   /* not supported on this device -> HybridBenchError    */

#define HB_DEVICE_PTRS 1
#define HB_ASYNC 2

/* element type codes for the histogram input (numpy dtype.kind/itemsize) */
#define HB_U8 1
#define HB_I8 2
#define HB_U16 3
#define HB_I16 4
#define HB_U32 5
#define HB_I32 6
#define HB_U64 7
#define HB_I64 8
#define HB_F64 9

/* ------------------------------------------------------------------ runtime */
int hb_version(void);
const char* hb_last_error(void);
/* Number of visible CUDA devices (0 if the driver has none). */
int hb_device_count(int* count);
/* SM count of the current device (grid sizing is a multiple of it). */
int hb_sm_count(int* count);
/* Synchronise `stream` and surface any pending CUDA error. */
int hb_stream_sync(void* stream);
/* Release cached device staging buffers of the current device. */
int hb_trim(void);

/* Device memory and streams for callers without a GPU framework (the
 * reference's own ctypes binding): select the device of
 * the calling thread, allocate / free device buffers, copy host <-> device
 * (stream-ordered; pass NULL for the legacy default stream; the copy is
 * complete on return unless flags & HB_ASYNC — then a page-locked host
 * buffer must stay untouched until hb_stream_sync; pageable buffers are
 * always consumed / filled before return), create / destroy streams.
 * Upload once, then run any entry point with HB_DEVICE_PTRS on the buffers
 * — the device-resident mode the benchmarks use.                         */
int hb_set_device(int device);
int hb_buf_alloc(size_t bytes, void** out);
int hb_buf_free(void* buf);
int hb_buf_upload(void* dst_device, const void* src_host, size_t bytes, int flags, void* stream);
int hb_buf_download(void* dst_host, const void* src_device, size_t bytes, int flags, void* stream);
int hb_stream_create(void** out);
int hb_stream_destroy(void* stream);

/* ---------------------------------------------------------------- generators
 * Device-side restatement of rng.py:45-51 (`splitmix64_array`): draw k
 * (1-based, k = k0+1 .. k0+n) of the stream `seed`, transformed:
 *   HB_GEN_RAW  u64 draw                         (splitmix64_array)
 *   HB_GEN_LOW8 u8  draw & 255                   (gen_hist_data / gen_image,
 *                                                 datasets.py:33-34, 104-106)
 *   HB_GEN_HI32 u32 draw >> 32                   (gen_sort_data, datasets.py:28-30)
 *   HB_GEN_MOD  i64 draw % bound                 (uniform_ints, rng.py:65-67)
 * `out` is a device pointer.  Bit-identical to the reference for every k.   */
#define HB_GEN_RAW 0
#define HB_GEN_LOW8 1
#define HB_GEN_HI32 2
#define HB_GEN_MOD 3
int hb_gen_splitmix(uint64_t seed, uint64_t k0, int64_t n, int kind, uint64_t bound,
                    void* out, void* stream);

/* ---------------------------------------------------------------- histogram
 * Replaces HistogramWorkload.run_part (kernels_regular.py:149-154): the bin
 * counts of `data[0:n]` (element type `dtype`), bin b = element value.
 * `bins_out` receives bin_count uint64 counts (ADDED to it when
 * flags & HB_ACCUMULATE, overwritten otherwise).  Elements outside
 * [0, bin_count) → HB_EINVAL, the reference's ValueError
 * (kernels_regular.py:137-138).  Supports 1 <= bin_count <= 49152.       */
#define HB_ACCUMULATE 4
int hb_hist(const void* data, int dtype, int64_t n, int32_t bin_count, uint64_t* bins_out,
            int flags, void* stream);


/* --------------------------------------------------------------------- SpMV
 * Replaces _csr_range_matvec / SpmvWorkload.run_part (kernels_irregular.py:
 * 206-211, 250-251): y = A[row0:row1] x over a CSR whose row_ptr entries are
 * absolute offsets into col_idx/values.  Index arrays are HB_I32 or HB_I64.
 *   perm == NULL: y[i-row0] = row i's sum         (the y_perm slice)
 *   perm != NULL: y[perm[i]] = row i's sum        (fused inverse permutation,
 *                                                  SpmvWorkload.merge :253-257)
 * mode HB_SPMV_SEQ: bit-identical to the reference (rounded products, rows
 * summed left to right, no FMA).  HB_SPMV_WARP: warp tree reduction,
 * within 1e-9 relative.  Host-pointer calls stage only the row range.     */
#define HB_SPMV_SEQ 0
#define HB_SPMV_WARP 1
#define HB_SPMV_MERGE 2  /* merge-path (load-balanced for any row lengths), within 1e-9 relative */
int hb_spmv_csr(const void* row_ptr, int ptr_code, const void* col_idx, int col_code,
                const double* values, int64_t row0, int64_t row1, int64_t cols, const double* x,
                const void* perm, int perm_code, double* y, int mode, int flags, void* stream);

/* SELL-32 copy of a device int32 CSR (the bit-exact SpMV's conflict-free
 * layout): tile t = rows [32t, 32t+32) stored column-major, its length the
 * longest row; tile_off (device, ntiles+1 int64) = element offsets.
 * hb_spmv_sell_build with sell_col == NULL sizes it (tile_off + *total_out,
 * host), then with sell_col/sell_val (total entries each) fills it.
 * hb_spmv_sell = hb_spmv_csr mode HB_SPMV_SEQ on that layout (row_ptr still
 * gives the row lengths), bit-identical.  Device pointers only.            */
int hb_spmv_sell_build(const int32_t* row_ptr, const int32_t* col_idx, const double* values, int64_t rows,
                       int64_t* tile_off, int32_t* sell_col, double* sell_val, int64_t* total_out, int flags,
                       void* stream);
int hb_spmv_sell(const int32_t* row_ptr, const int64_t* tile_off, const int32_t* sell_col, const double* sell_val,
                 int64_t row0, int64_t row1, const double* x, const void* perm, int perm_code, double* y, int flags,
                 void* stream);

/* CsrMatrix invariants (kernels_irregular.py:44-60) checked on the device:
 * *flags_out |= 1 bad row_ptr ends, 2 decreasing row_ptr, 4 column out of
 * range, 8 columns not strictly increasing within a row.                   */
/* Device spmv_preprocess (kernels_irregular.py:171-203): perm_out = the
 * stable argsort of the row lengths (hb_sort with a row-index payload),
 * new_row_ptr = exclusive scan of the sorted lengths, rows gathered into
 * new_col/new_values.  Index types follow ptr_code / col_code / perm_code.
 * Device pointers only.                                                    */
int hb_spmv_preprocess(const void* row_ptr, int ptr_code, const void* col_idx, int col_code,
                       const double* values, int64_t rows, void* perm_out, int perm_code,
                       void* new_row_ptr, void* new_col, double* new_values, int flags, void* stream);

int hb_csr_validate(const void* row_ptr, int ptr_code, const void* col_idx, int col_code,
                    int64_t rows, int64_t nnz, int64_t cols, uint32_t* flags_out, int flags,
                    void* stream);

/* Device gen_csr (datasets.py:37-55), bit-identical to the reference:
 * avg = max(1, round(density*cols)) (computed by the caller, Python's
 * round), seed_counts/rows/vals = mix_seed(seed, 1/2/3) (rng.py:54-57).
 * row_ptr (rows+1, ptr_code) is always written and *nnz_out returned; with
 * col_idx == values == NULL nothing else happens (sizing call), otherwise
 * col_idx/values (nnz_cap entries) receive the columns and values.  Rows of
 * up to 1020 nonzeros; device pointers only.                                */
int hb_gen_csr(int64_t rows, int64_t cols, int64_t avg, uint64_t seed_counts, uint64_t seed_rows,
               uint64_t seed_vals, void* row_ptr, int ptr_code, void* col_idx, int col_code, double* values,
               int64_t nnz_cap, int64_t* nnz_out, int flags, void* stream);

/* ---------------------------------------------------------------- bilateral
 * Replaces bilateral_rows / BilateralApplyWorkload.run_part
 * (kernels_regular.py:461-511): output rows [row0, row1) of the clamp-to-edge
 * LUT bilateral filter of the uint8 image img[height][width];
 * spatial[(2r+1)^2] row-major and range256[256] are the BilateralLut tables
 * (:447-458).  out is (row1-row0) x width, fp64 (out_code 64, bit-identical
 * to the reference) or fp32 (out_code 32, the fp64 result rounded).
 * flags & HB_FP32_ARITH: taps in fp32 (fp32 tables, FMA), within 1e-5
 * relative of the fp64 result (the tolerance north_star allows for filter
 * outputs) at about twice the fp64 kernel's rate.
 * Host-pointer calls stage only the strip plus its clamped halo rows.     */
#define HB_FP32_ARITH 16  /* filters: fp32 arithmetic (within 1e-5 relative of the fp64 result) */
int hb_bilateral_u8(const uint8_t* img, int32_t height, int32_t width, int32_t radius,
                    const double* spatial, const double* range256, int32_t row0, int32_t row1,
                    void* out, int out_code, int flags, void* stream);

/* -------------------------------------------------------------- convolution
 * Replaces convolve_rows / ConvolutionWorkload.run_part
 * (kernels_regular.py:359-414): output rows [row0, row1) of the clamp-to-edge
 * correlation of img[height][width] (in_code HB_U8 or HB_F64) with the
 * (2r+1)^2 row-major weights.  Bit-identical to the reference for fp64 output
 * (out_code 64): taps in row-major order, zero weights skipped, rounded fp64
 * multiply then add, no FMA.  out_code 32 rounds that result to fp32.
 * flags & HB_FP32_ARITH: fp32 taps with FMA, within 1e-5 relative of the
 * fp64 result (north_star's filter tolerance).  flags & HB_TAPS_DENSE: the
 * caller states that no weight is 0 (device-pointer calls then skip reading
 * the weights back to choose the branch-free kernel: no host wait, CUDA-graph
 * capturable); a wrong statement is the caller's error.
 * Host-pointer calls stage only the strip plus its clamped halo rows.     */
#define HB_TAPS_DENSE 32
int hb_convolve(const void* img, int in_code, int32_t height, int32_t width, int32_t radius,
                const double* weights, int32_t row0, int32_t row1, void* out, int out_code,
                int flags, void* stream);

/* --------------------------------------------------------------------- sort
 * Replaces the DeviceB side of sample_sort_hybrid (kernels_regular.py:239-310)
 * with an LSD radix sort (onesweep: one digit-histogram pass, then one
 * decoupled-look-back pass per 8-bit digit that is not constant).  Sorts
 * keys_in[0:n] into keys_out (the same pointer sorts in place; key_code
 * HB_U32/HB_I32/HB_U64/HB_I64).  When vals_in/vals_out are non-NULL the
 * uint32 payload is permuted alongside — stably, so a payload of 0..n-1
 * becomes the stable argsort.  *passes_done (optional) receives the number
 * of digit passes executed (0 ⇔ all keys equal).  n < 2^30 per call.
 * Ranking: one shared atomic per key, relying on lane-ordered old values
 * (verified on each device before first use — on the bare atomic pattern
 * and through the production pass kernels on duplicate-heavy keys with an
 * index payload, stability checked on the device; the ballot multi-split
 * runs when either check fails).  flags & HB_SORT_BALLOT (or HB_SORT_RANK=ballot in
 * the environment) selects the ballot multi-split, whose stability does not
 * depend on that behaviour — the library's own stable-argsort users
 * (device gen_list, spmv_preprocess) use it.  With HB_ASYNC and
 * passes_done == NULL (32-bit keys) the call never waits on the host: all
 * four digit positions are sorted.                                         */
#define HB_SORT_BALLOT 8  /* rank with the ballot multi-split instead of lane-ordered shared atomics */
int hb_sort(const void* keys_in, void* keys_out, int key_code, const uint32_t* vals_in,
            uint32_t* vals_out, int64_t n, int32_t* passes_done, int flags, void* stream);

/* Split points of the multi-GPU sample-merge: out_pos[j] =
 * number of (keys[i], vals[i]) lexicographically below (probe_keys[j],
 * probe_vals[j]) in the sorted sequence (key-only when either vals array is
 * NULL).  Device pointers only.                                             */
int hb_sort_bounds(const void* keys, int key_code, const uint32_t* vals, int64_t n,
                   const void* probe_keys, const uint32_t* probe_vals, int32_t m, int64_t* out_pos,
                   int flags, void* stream);

/* ------------------------------------------------------------- list ranking
 * Replaces the ranking of list_rank_with_stats / list_rank_hybrid
 * (kernels_irregular.py:377-508): rank[i] = distance of node i from `head`
 * along succ (succ[i] = next node or -1; HB_I32 or HB_I64), rank int64.
 * Includes validate_list's checks (:377-393): head/successor out of range,
 * cycles and broken lists return HB_ESTRUCT.  Recursive sparse ruling set
 * (Helman-JaJa) + Wyllie pointer jumping on the top level.               */
int hb_list_rank(const void* succ, int succ_code, int64_t n, int64_t head, int64_t* rank, int flags,
                 void* stream);

/* Device-side gen_list (datasets.py:58-63) second half: given `order`, the
 * stable argsort of the splitmix draws (hb_sort of the draws with an index
 * payload), link succ[order[i]] = order[i+1], tail -1.  Device pointers. */
int hb_link_order(const int32_t* order, int64_t n, void* succ, int succ_code, int flags, void* stream);

/* The reference's fractional-independent-set reduction and sublist-head
 * choice (kernels_irregular.py:396-448), run on the GPU for its statistics:
 * round_sizes[r] = live nodes at the start of round r (first round_cap
 * rounds), stats = {fis_rounds, reduced_size, removed_total, sublist_count}
 * — identical to the reference's ListRankStats for the same (list, seed,
 * sublists = 4 * total workers).  The list must be valid (hb_list_rank
 * first); non-convergence → HB_ESTRUCT.                                    */
int hb_list_fis_stats(const void* succ, int succ_code, int64_t n, int64_t head, uint64_t seed,
                      int32_t sublists, int64_t* round_sizes, int32_t round_cap, int64_t* stats,
                      int flags, void* stream);

/* -------------------------------------------------------- multi-GPU shards
 * One process per GPU; these are the device halves of the partition → run_part
 * → merge protocol (worksharing.py:297-359) when DeviceB is a group of G GPUs
 * (SURVEY §8e).  The collectives themselves are torch.distributed (NCCL over
 * NVLink) on the tensors these functions produce and consume.
 *
 * hb_partition_nnz: the device-side SpMV partitioner.  bounds_out[k] (HOST
 * array, parts+1 entries) = row0 + searchsorted(cum, k*total/parts, 'left')
 * over cum = row_ptr[row0..row1] - row_ptr[row0] in fp64 — SpmvWorkload's
 * split rule (kernels_irregular.py:243-245) at k/G.  With HB_DEVICE_PTRS
 * row_ptr is a device array and only the G+1 bounds leave the device.      */
int hb_partition_nnz(const void* row_ptr, int ptr_code, int64_t row0, int64_t row1, int32_t parts,
                     int64_t* bounds_out, int flags, void* stream);

/* dst[perm[i]] = src[i], i < n, 4- or 8-byte elements: SpmvWorkload.merge's
 * un-permute (kernels_irregular.py:253-257) applied to an all-gathered
 * y_perm.  Device pointers only.                                           */
int hb_scatter_perm(const void* src, int64_t n, int elem_bytes, const void* perm, int perm_code, void* dst,
                    int flags, void* stream);

/* Stable merge of nruns sorted runs keys[offsets[r] .. offsets[r+1]) (host
 * offsets array, offsets[0] = 0, offsets[nruns] = n) into keys_out, the
 * uint32 payload (optional) moved alongside; equal keys keep run order.  The
 * receive side of the multi-GPU sample-merge sort (runs arrive in rank
 * order).  Pairwise merge-path rounds; device pointers only, no aliasing.  */
int hb_merge_runs(const void* keys, int key_code, const uint32_t* vals, int64_t n, const int64_t* offsets,
                  int32_t nruns, void* keys_out, uint32_t* vals_out, int flags, void* stream);

/* Sharded list ranking (the sublist split of _rank_reduced,
 * kernels_irregular.py:431-478, mapped onto GPUs):
 *  hb_lr_layout      nsub sublists (every node index ≡ 0 mod 64, plus the
 *                    head) and the id of the head's sublist;
 *  hb_lr_walk_part   validates succ (like hb_list_rank), fills packed[n]
 *                    with 0xff, walks the sublists with ids in
 *                    [sub_lo, sub_hi): packed[v] = (sublist << 32 | offset)
 *                    for the nodes it passes, sub_nxt/sub_len[j] for its ids;
 *  (caller)          all-gathers sub_nxt / sub_len across the G ranks;
 *  hb_lr_finish_part ranks the sublist chain weighted by length (it must
 *                    cover all n nodes, else HB_ESTRUCT — on every rank
 *                    alike) and turns packed into ranks for the nodes of
 *                    sublists [sub_lo, sub_hi), 0 for all other nodes;
 *  (caller)          all-reduce (sum) of rank → every rank holds all ranks
 *                    (int32 ranks + hb_widen_i32 when n <= 2^31).
 * Device pointers only; n < 2^31.                                          */
int hb_lr_layout(int64_t n, int64_t head, int64_t* nsub, int64_t* sub_head);
int hb_lr_walk_part(const void* succ, int succ_code, int64_t n, int64_t head, int64_t sub_lo, int64_t sub_hi,
                    int64_t* packed, int64_t* sub_nxt, int64_t* sub_len, int flags, void* stream);
int hb_lr_finish_part(const int64_t* sub_nxt, const int64_t* sub_len, int64_t nsub, int64_t sub_head, int64_t n,
                      int64_t sub_lo, int64_t sub_hi, int64_t* rank, int flags, void* stream);
/* hb_lr_finish_part with int32 ranks (n <= 2^31): reads the packed walk
 * output and writes rank32 — the all-reduce then moves 4 bytes per node —
 * and hb_widen_i32 turns the reduced ranks back into the int64 result.    */
int hb_lr_finish_part32(const int64_t* sub_nxt, const int64_t* sub_len, int64_t nsub, int64_t sub_head, int64_t n,
                        int64_t sub_lo, int64_t sub_hi, const int64_t* packed, int32_t* rank32, int flags,
                        void* stream);
int hb_widen_i32(const int32_t* in, int64_t n, int64_t* out, int flags, void* stream);

/* ------------------------------------------------------- host (DeviceA)
 * The host share of a work-shared run on `workers` host threads, bit-identical
 * to the reference's numpy bodies (no GPU involved): histogram
 * (HistogramWorkload.run_part, kernels_regular.py:149-154), CSR row range
 * (_csr_range_matvec, kernels_irregular.py:206-211; y[i - row0], or
 * y[perm[i]] when perm is given — the un-permute of :224-227 fused in),
 * convolution rows (convolve_rows, kernels_regular.py:359-381; f64 out) and
 * bilateral rows (bilateral_rows, :461-486; f64 out).                      */
int hb_host_hist(const void* data, int dtype, int64_t n, int32_t bin_count, uint64_t* bins_out, int workers);
int hb_host_spmv_rows(const void* row_ptr, int ptr_code, const void* col_idx, int col_code,
                      const double* values, int64_t row0, int64_t row1, const double* x,
                      const void* perm, int perm_code, double* y, int workers);
int hb_host_conv_rows(const void* img, int in_code, int32_t height, int32_t width, int32_t radius,
                      const double* weights, int32_t row0, int32_t row1, double* out, int workers);
int hb_host_bilateral(const uint8_t* img, int32_t height, int32_t width, int32_t radius,
                      const double* spatial, const double* range256, int32_t row0, int32_t row1,
                      double* out, int workers);

#ifdef __cplusplus
}
#endif
#endif /* HB200_H */
