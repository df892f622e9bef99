/*
 * include/prefixscan_b200.h -- C-ABI of libprefixscan_b200.so, the B200
 * (sm_100a) prefix-sum path that sits behind the reference package's scan
 * entry points (/root/reference/pkg/src/prefixscan).
 *
 * The reference is pure Python + numba; it has no FFI of its own.  These
 * exports are the boundary a maintainer binds with ctypes,
 * one per reference kernel family on the hot path:
 *
 *   ps_scan            <- core.py:86-92   _scan_kernel        (+ core.py:118-126 sequential_inclusive_scan)
 *                         simd.py:75-101  _make_horizontal_kernel (+ simd.py:134-148 horizontal_scan)
 *                         core.py:109-115 _shift_right_kernel  (fused: exclusive != 0)
 *   ps_reduce          <- core.py:95-100  _accumulate_kernel   (+ core.py:129-132 sequential_accumulate)
 *                         simd.py:104-121 _make_simd_accumulate_kernel
 *   ps_add_offset      <- core.py:103-106 _increment_kernel    (+ core.py:135-138 sequential_increment)
 *   ps_scan_batched    <- simd.py:164-206 vertical pass kernels (row seeds in, row totals out)
 *   ps_scan_segmented  <- (no reference kernel; CSR-segment form of the per-chunk scans of simd.py:164-206)
 *   ps_scan_host       <- engine.py:219-248 ScanEngine.run on host buffers (end-to-end call:
 *                         host->device copy, scan, device->host copy, pipelined)
 *
 * Conventions
 * - extern "C", plain pointers and sizes, no exceptions cross the ABI.
 * - Every device call is asynchronous on `stream` (a cudaStream_t passed as
 *   void*; NULL = legacy default stream) except ps_scan_host, which blocks.
 * - Element counts and leading dimensions are in ELEMENTS.
 * - The accumulator ("acc") type of a dtype pair: int64 for signed integer
 *   input, uint64 for uint32 input, double for float32/float64 input.  Seeds,
 *   totals and deltas are acc-typed 8-byte values.
 * - Seeds: the carry-in of a scan is  seed_bits (host value, acc bits)
 *   + sum(seed_terms[0 .. n_seed_terms))  (device array, acc-typed) -- the
 *   device terms let a multi-GPU carry (allgathered shard totals) flow
 *   without a host round trip.
 * - Scratch: look-back descriptors.  Sized by ps_*_scratch_bytes, must be
 *   ZERO-FILLED when first allocated, and each launch on one scratch buffer
 *   needs a fresh `epoch` in [1, PS_EPOCH_MAX] strictly greater than the
 *   previous one (descriptors are epoch-tagged, so no per-call memset).  When
 *   the epochs run out, zero the buffer again and restart at 1.  (The first
 *   16 bytes of a batched scan's scratch are the rows kernel's row ticket;
 *   every launch leaves them at zero again.)  One scratch may serve every
 *   entry point in turn: the non-descriptor words kernels leave in it
 *   (segment and compaction bookkeeping) keep their two low bits 0, so they
 *   never pass for a published descriptor of a later epoch.
 * - Forward progress.  The persistent kernels (stream, rows, CSR regions, single-pass select)
 *   are cooperative launches of at most one resident grid, so every CTA a role waits on is
 *   running.  The look-back tiles kernels (small inputs) take tile ids from blockIdx and rely
 *   on the hardware dispatching CTAs in increasing linear order: a tile only ever waits on
 *   lower-numbered tiles, which are resident or finished by then -- the argument CUB's
 *   single-pass scan rests on; there is no atomic tile counter.  Cross-GPU waits
 *   (ps_scan_mailbox) give up after ~10 s and raise the caller's timeout flag instead of
 *   hanging.
 * - `in == out` (in place) is allowed; partial overlap is not.
 * - Return 0 on success, a PS_ERR_* (>0) on misuse, or a cudaError_t value
 *   offset by PS_ERR_CUDA_BASE on a CUDA failure.
 */
#ifndef PREFIXSCAN_B200_H
#define PREFIXSCAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes (same numbering as oracle/scan_oracle.h) */
#define PS_DTYPE_INT32 1
#define PS_DTYPE_INT64 2
#define PS_DTYPE_UINT32 3
#define PS_DTYPE_UINT64 4
#define PS_DTYPE_FLOAT32 5
#define PS_DTYPE_FLOAT64 6
#define PS_DTYPE_UINT8 7    /* flags only (ps_select): byte bitmap / bool */

/* multi-GPU schemes, named after plan.py:24-37 SchemeId */
#define PS_SCHEME_SCAN_INCREMENT 0   /* scan-then-fixup, 4n bytes  (SCAN_INCREMENT_EQUAL)   */
#define PS_SCHEME_ACCUMULATE_SCAN 1  /* reduce-then-scan, 3n bytes (ACCUMULATE_SCAN_EQUAL) */

#define PS_EPOCH_MAX 0x3FFFFFFFu

#define PS_OK 0
#define PS_ERR_DTYPE 1     /* unsupported (dtype_in, dtype_out) pair              */
#define PS_ERR_ARG 2       /* negative size, NULL or element-misaligned buffer, bad leading dimension */
#define PS_ERR_SCRATCH 3   /* scratch missing or smaller than ps_*_scratch_bytes   */
#define PS_ERR_EPOCH 4     /* epoch outside [1, PS_EPOCH_MAX]                      */
#define PS_ERR_OVERLAP 5   /* in/out partially overlap                             */
#define PS_ERR_CUDA_BASE 1000

/* Supported (dtype_in -> dtype_out) pairs:
 *   int32->int32, int32->int64, int64->int64, uint32->uint32, uint32->uint64,
 *   uint64->uint64, float32->float32, float32->float64, float64->float64 */
int ps_pair_supported(int dtype_in, int dtype_out);

/* Bytes of look-back scratch for a 1-D scan of n elements. */
size_t ps_scan_scratch_bytes(int64_t n, int dtype_in, int dtype_out);

/* Inclusive (exclusive == 0) or exclusive scan of in[0..n) into out[0..n).
 * total_out (device, acc-typed, nullable) receives seed + sum(in).
 * Replaces core.py:86-92 (+ exclusive: core.py:109-115, whose returned "last"
 * is *total_out). */
int ps_scan(const void *in, void *out, int64_t n, int dtype_in, int dtype_out, int exclusive,
            uint64_t seed_bits, const void *seed_terms, int64_t n_seed_terms, void *total_out,
            void *scratch, size_t scratch_bytes, uint32_t epoch, void *stream);

/* Bytes of scratch for ps_reduce. */
size_t ps_reduce_scratch_bytes(int64_t n, int dtype_in);

/* total_out (device, acc-typed) = seed_bits + sum(seed_terms) + sum(in[0..n)).
 * Read-only on `in`.  Deterministic summation order.  Replaces core.py:95-100. */
int ps_reduce(const void *in, int64_t n, int dtype_in, uint64_t seed_bits, const void *seed_terms,
              int64_t n_seed_terms, void *total_out, void *scratch, size_t scratch_bytes,
              void *stream);

/* buf[i] = buf[i] + delta, delta = delta_bits + sum(delta_terms), computed in
 * the acc type and stored back in the element type.  Replaces core.py:103-106. */
int ps_add_offset(void *buf, int64_t n, int dtype, uint64_t delta_bits, const void *delta_terms,
                  int64_t n_delta_terms, void *stream);

/* Bytes of scratch for ps_scan_batched. */
size_t ps_scan_batched_scratch_bytes(int64_t rows, int64_t cols, int dtype_in, int dtype_out);

/* rows independent scans: out[r*ld_out + c] = row_seeds[r] + sum_{c'<=c} in[r*ld_in + c']
 * (exclusive: c' < c).  row_seeds / row_totals: device, acc-typed, nullable. */
int ps_scan_batched(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                    int64_t ld_out, int dtype_in, int dtype_out, int exclusive,
                    const void *row_seeds, void *row_totals, void *scratch, size_t scratch_bytes,
                    uint32_t epoch, void *stream);

/* Bytes of scratch for ps_scan_segmented. */
size_t ps_scan_segmented_scratch_bytes(int64_t n, int dtype_in, int dtype_out);

/* Segmented scan over CSR segments of one contiguous buffer: segment s is
 * in[seg_offsets[s] .. seg_offsets[s+1]), seg_offsets (device int64, nseg+1
 * entries, non-decreasing, seg_offsets[0] == 0, seg_offsets[nseg] == n).
 * Every segment restarts at zero; seg_totals (device acc-typed, nullable)
 * receives each segment's sum (0 for an empty segment).  Large inputs run on
 * the shared-memory-region kernel (seg_stream.cuh: head bitmap pre-pass, one
 * HBM read and one write per element); for integer scans with 64-bit outputs
 * the totals are read back from `out` by a small kernel after the scan (the
 * inclusive value of a segment's last element), otherwise the scanners emit
 * them.  seg_totals must not overlap in / out. */
int ps_scan_segmented(const void *in, void *out, int64_t n, const int64_t *seg_offsets,
                      int64_t nseg, int dtype_in, int dtype_out, int exclusive, void *seg_totals,
                      void *scratch, size_t scratch_bytes, uint32_t epoch, void *stream);

/* Bytes of scratch for ps_shift_right. */
size_t ps_shift_right_scratch_bytes(int64_t n, int dtype);

/* out[0] = identity, out[i] = in[i-1]; *last_out (device, element-typed,
 * nullable) = in[n-1].  in == out allowed.  Replaces exclusive_from_inclusive
 * (core.py:141-151 / _shift_right_kernel core.py:109-115); the fused form is
 * ps_scan(..., exclusive=1, ...). */
int ps_shift_right(const void *in, void *out, int64_t n, int dtype, uint64_t identity_bits, void *last_out,
                   void *scratch, size_t scratch_bytes, void *stream);

/* row_totals[r] (device, acc-typed) = sum(in[r*ld_in .. r*ld_in+cols)).  Read-only.
 * Replaces simd.py:178-186 _vertical_pass1_accumulate. */
int ps_reduce_batched(const void *in, int64_t rows, int64_t cols, int64_t ld_in, int dtype_in, void *row_totals,
                      void *stream);

/* buf[r*ld + c] += row_deltas[r] (device, acc-typed).  rows <= 65535.
 * Replaces simd.py:189-195 _vertical_pass2_increment. */
int ps_add_offset_batched(void *buf, int64_t rows, int64_t cols, int64_t ld, int dtype, const void *row_deltas,
                          void *stream);

/* *total_out (device uint64) = seed + sum over w-blocks of (block sum mod 2^32)
 * + the scalar tail: the total the reference's horizontal kernel returns for
 * uint32 data (simd.py:84-99).  Read-only on `in`. */
int ps_reduce_wrapped_blocks(const void *in, int64_t n, int w, uint64_t seed_bits, void *total_out, void *stream);

/* Device workspace for ps_scan_host with the given chunk size. */
size_t ps_scan_host_workspace_bytes(int64_t chunk_elems, int dtype_in, int dtype_out);

/* Number of epochs ps_scan_host consumes (one per chunk). */
int64_t ps_scan_host_epochs(int64_t n, int64_t chunk_elems);

/* End-to-end scan of HOST buffers: chunked pipeline of H2D copy -> scan
 * seeded by the previous chunk's total -> D2H copy over three CUDA streams.
 * Page-locked buffers are copied directly; pageable ones go through a ring of
 * pinned bounce buffers filled and drained by host copy threads, overlapped
 * with the transfers of neighbouring chunks (in == out allowed).  Blocks until out_host and *total_host (acc-typed,
 * host, nullable) are written.  Epochs epoch .. epoch+ps_scan_host_epochs-1
 * are used on the scratch inside `workspace` (zero-filled when allocated). */
int ps_scan_host(const void *in_host, void *out_host, int64_t n, int dtype_in, int dtype_out,
                 int exclusive, uint64_t seed_bits, void *total_host, void *workspace,
                 size_t workspace_bytes, int64_t chunk_elems, uint32_t epoch, void *stream);

/* Page-lock a caller-owned host range in place (cudaHostRegister) so that
 * ps_scan_host / ps_scan_batched_host stream it at full PCIe rate without a
 * copy into a pinned buffer -- the reference's users pass plain numpy arrays
 * (core.py:118-126), which this turns into DMA-able memory.  *registered
 * (nullable) = 1 if this call registered the range, 0 if it already was page-
 * locked (nothing to undo).  ps_host_unregister undoes a registration;
 * ps_host_is_pinned reports 1 for page-locked (registered or cudaHostAlloc)
 * memory and 0 for pageable memory. */
int ps_host_register(void *ptr, size_t bytes, int *registered);
int ps_host_unregister(void *ptr);
int ps_host_is_pinned(const void *ptr);

/* Blelloch tree step functions on a power-of-two span, in place, element-typed
 * arithmetic in the reference's exact pairing (bit-identical float results):
 *   ps_tree_up_sweep   <- up_sweep   simd.py:327-334, :356-360 (root -> *root_out,
 *                         device, element-typed, nullable)
 *   ps_tree_down_sweep <- down_sweep simd.py:338-347, :363-367 (up-swept span ->
 *                         its exclusive scan)
 * PS_ERR_ARG unless n is a power of two (simd.py:370-372). */
int ps_tree_up_sweep(void *data, int64_t n, int dtype, void *root_out, void *stream);
int ps_tree_down_sweep(void *data, int64_t n, int dtype, void *stream);

/* Fused exchange of shard totals over NVLink / NVSwitch (SURVEY.md §8(e) option ii;
 * replaces the all-gather feeding the ledger fold, engine.py:329-331, across
 * GPUs).  Every GPU owns a mailbox of 2 x n_peers 16-byte slots (e.g. in
 * symmetric memory); slot (e & 1) * n_peers + h holds rank h's total of
 * exchange epoch e.  This call stores {epoch, *total} (device, acc-typed 8
 * bytes) into that slot of every peer's mailbox -- peer_mailboxes is a DEVICE
 * array of n_peers mapped base addresses -- as value store then flag store
 * with st.release.sys (the consumer polls the flag with ld.acquire.sys and only
 * then reads the value), after waiting (in the kernel) until all n_peers totals of
 * prev_epoch (0 = none) have arrived in own_mailbox, which guarantees no
 * slot is overwritten while a slower rank can still read it.  Stream-ordered
 * after the kernel that produced *total; a wait longer than ~10 s sets
 * *timeout_flag (device int, nullable) instead of hanging. */
int ps_publish_total(const void *total, void *const *peer_mailboxes, int n_peers, int rank, uint32_t epoch,
                     uint32_t prev_epoch, const void *own_mailbox, int *timeout_flag, void *stream);

/* ps_scan whose seed additionally includes the totals found in the n_wait
 * 16-byte slots at `mailbox` (pass own_mailbox + (e & 1) * n_peers slots: the
 * ranks before this one) tagged with mail_epoch.  The wait happens inside the scan kernel (the warp that folds
 * the seed polls; loads and reductions of the first regions proceed), so no
 * host synchronisation or collective launch sits between the passes.  A wait
 * longer than ~10 s sets *timeout_flag (device int, nullable) and continues
 * with zeros instead of hanging. */
int ps_scan_mailbox(const void *in, void *out, int64_t n, int dtype_in, int dtype_out, int exclusive,
                    uint64_t seed_bits, const void *mailbox, int n_wait, uint32_t mail_epoch, int *timeout_flag,
                    void *total_out, void *scratch, size_t scratch_bytes, uint32_t epoch, void *stream);

/* Bytes of scratch for ps_select over n elements. */
size_t ps_select_scratch_bytes(int64_t n);

/* Stream compaction / stable partition driven by a flag array -- the consumer
 * of exclusive offsets the paper motivates the prefix sum with (PAPER.md:34:
 * "determine the new offsets of data items during a partitioning step ... from
 * a previously constructed bitmap"; the offsets are ps_scan(flags, exclusive=1),
 * cf. _scan_kernel core.py:86-92 + exclusive_from_inclusive core.py:141-151).
 *   values       n elements of dtype_values (any 4- or 8-byte PS_DTYPE_*; bits copied)
 *   flags        n elements of dtype_flags (PS_DTYPE_UINT8 or any 4/8-byte dtype);
 *                an element is selected when its flag has any nonzero bit
 *   partition    0: out[0..k) = selected values in order (k = selected count)
 *                1: additionally out[k..n) = rejected values in order (stable partition)
 *   out          device, >= k (partition: n) elements; must not overlap values/flags
 *   count_out    device int64 (nullable) <- k
 * Compaction of >= 4 Mi elements with 4/8-byte flags and 16-byte aligned inputs runs in ONE pass
 * (select_stream.cuh: flags + values loaded once into shared-memory regions,
 * portion counts exchanged through epoch-tagged descriptors as in ps_scan);
 * partition mode and small inputs take three launches (per-8192-element tile
 * counts, exclusive scan of the counts, scatter through shared memory), which
 * read the flags twice.  epoch as for ps_scan ("select_kernel" tuning knob:
 * 0 auto, 1 three launches, 2 single pass). */
int ps_select(const void *values, const void *flags, int64_t n, int dtype_values, int dtype_flags, int partition,
              void *out, void *count_out, void *scratch, size_t scratch_bytes, uint32_t epoch, void *stream);

/* Device workspace for ps_scan_batched_host with chunk_rows rows of cols. */
size_t ps_scan_batched_host_workspace_bytes(int64_t chunk_rows, int64_t cols, int dtype_in, int dtype_out);

/* End-to-end batched scan of contiguous HOST rows (rows x cols, pinned for
 * full speed): chunks of chunk_rows rows go H2D -> ps_scan_batched -> D2H over
 * three CUDA streams, so both PCIe directions and the scan overlap.  Rows are
 * independent (no carry between chunks).  Blocks until out_host is written.
 * Epochs epoch .. epoch + ceil(rows / chunk_rows) - 1 are used.  The per-row
 * form of the reference's horizontal_scan(out=) (simd.py:134-148) on host data. */
int ps_scan_batched_host(const void *in_host, void *out_host, int64_t rows, int64_t cols, int dtype_in,
                         int dtype_out, int exclusive, void *workspace, size_t workspace_bytes, int64_t chunk_rows,
                         uint32_t epoch, void *stream);

/* Tuning knobs (process-wide; for benchmarks and tests):
 *   "scan_kernel"      0 = auto (3 for large inputs, 1 below rounds_min_bytes),
 *                      1 = single-pass decoupled look-back,
 *                      2 = cache-partitioned rounds (persistent, L2 regions),
 *                      3 = shared-memory-resident streaming regions (persistent)
 *   "round_bytes"      input + output bytes per L2 region of the rounds kernel (0 = default)
 *   "round_lead"       regions the rounds kernel's reducer warps run ahead
 *   "round_ramp"       ramp regions (halving sizes) at each end of the rounds kernel
 *   "round_prefetch"   1 = bulk L2 prefetch of each reducer portion (rounds kernel)
 *   "rows_kernel"      batched scans: 0 = auto, 1 = look-back tiles, 2 = one CTA per row
 *   "rounds_min_bytes" auto mode uses the shared-memory-region (stream) kernel from
 *                      this input size (smaller inputs: the look-back kernel)
 *   "select_kernel"    ps_select: 0 = auto, 1 = three launches, 2 = single pass (compaction)
 *   "stream_inflight"  stream scan and single-pass select kernels: at most this many
 *                      regions' loads outstanding per SM
 *                      (default 2; 0 = as many as the buffer ring holds)
 *   "stream_copy_in"   1-D inputs whose input and output sit at different 32-byte phases:
 *                      1 = stream kernel with the tile grid aligned to the output (bulk copies
 *                      where the input's 16-byte phase fits, element-wise cp.async by the
 *                      reducer warps otherwise), 0 = look-back tiles (default 1)
 *   "rows_dynamic"     rows kernel: 1 = rows handed out from a grid-wide ticket kept in
 *                      the scratch's control words (faster SMs take more rows),
 *                      0 = CTA c takes rows c, c+G, ... (default 1)
 *   "rows_multi"       rows kernel: 1 = rows of at most half a 64 KiB buffer share
 *                      buffers (several rows per TMA item), 0 = one row per buffer
 *   "tiles_row_lead"   batched rows on the look-back tiles kernel (row lengths not a
 *                      multiple of 16 bytes): 1 = each row's tile grid starts on its own
 *                      32-byte boundary (vector accesses) and short contiguous rows
 *                      without seeds run as one uniform-segment scan; 0 = shared lead
 *   "reduce_blocks"    ps_reduce: 1 = blocks of >= 256 KiB from a ticket (faster SMs
 *                      take more; block partials folded in block order), 0 = grid-stride
 *   "add_chunked"      ps_add_offset: 1 = one CTA per 64 KiB (hardware-balanced),
 *                      0 = a grid of 8 CTAs per SM with grid-stride shares
 *   "stall_seed" / "stall_prob" / "stall_ns"
 *                      stress tests only: every role hand-off of the look-back,
 *                      rounds and rows kernels sleeps with probability
 *                      stall_prob/1024 for a hashed time in [0, stall_ns)
 *                      (stall_ns 0 = off; the reference's delay_hook, engine.py:91)
 *   "seg_kernel"       ps_scan_segmented: 0 = auto (shared-memory regions from
 *                      rounds_min_bytes of input, look-back tiles below), 1 = look-back
 *                      tiles, 2 = shared-memory regions
 *   "float_exact"      stream kernel, float32 -> float32: 0 = in-chunk scans in float32
 *                      with the float64 carry applied as a float pair (FP32 pipe only,
 *                      <= 1e-6 relative to float32(cumsum(float64))), 1 = float64 per
 *                      element (bit-exact whenever the float64 sums are exact) (default 0)
 * Knobs are per calling host thread: setting one never changes what another
 * thread's calls launch.
 * Returns PS_ERR_ARG for an unknown key or value. */
int ps_set_tuning(const char *key, int64_t value);
int64_t ps_get_tuning(const char *key); /* -1 for an unknown key */

/* Human-readable text for a return code. */
const char *ps_error_string(int code);

/* ABI version (major*100 + minor). */
int ps_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PREFIXSCAN_B200_H */
