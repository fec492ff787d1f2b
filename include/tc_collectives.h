/*
 * tc_collectives.h -- C ABI of the B200 (sm_100a) tensor-core segmented
 * reduction and scan library (arXiv 1811.09736, re-designed for Blackwell).
 *
 * The reference (`halftile`, /root/reference/pkg) is a pure-Python package
 * with no FFI.  Each entry point below replaces the body of one reference
 * operator; the Python shim in paper_1811_09736_b200/ keeps the reference
 * signatures and validation and calls these through ctypes:
 *
 *   tc_seg_reduce  <- halftile.reduce.segmented_reduce  (reduce.py:379-446)
 *                     and the warp/block primitives it dispatches to:
 *                     reduce_16 (:92), reduce_256 (:109),
 *                     reduce_256n_efficient (:123), reduce_256n_inefficient
 *                     (:144), reduce_16n_strided (:171),
 *                     reduce_16n_coalesced (:201), block_reduce_256n (:278)
 *   tc_full_reduce <- halftile.reduce.grid_reduce       (reduce.py:332-373)
 *   tc_seg_scan    <- halftile.scan.segmented_scan      (scan.py:316-388)
 *                     and scan_16 (:58), scan_256/_256n (:94-119),
 *                     scan_16n (:122), block_scan_256n (:178)
 *   tc_full_scan   <- halftile.scan.grid_scan           (scan.py:249-310)
 *
 * Conventions
 *   - All data pointers are DEVICE pointers owned by the caller; the library
 *     never retains or frees them.  Calls are stream-ordered (no host sync)
 *     and reentrant across host threads on different streams, each with its
 *     own workspace.
 *   - Input is IEEE binary16, contiguous, 16-byte aligned, 0 < n < 2^37.
 *   - Segment semantics follow halftile.segmented.pad_segmented
 *     (segmented.py:57-89): segment k covers elements [k*seg, (k+1)*seg),
 *     the last segment may be ragged (shorter); a reduce returns
 *     ceil(n/seg) sums, a scan returns n prefix sums.
 *   - Arithmetic: products on the tensor core (tcgen05.mma kind::f16, fp32
 *     accumulation in TMEM), in-tile row / warp combines in fp32, cross-tile
 *     and cross-CTA carries in fp64 (CHUNK unit aggregates as double-float
 *     pairs), one rounding to the output dtype.  Every output is a sum of
 *     its OWN segment's elements only: |out - exact| <= 1 ulp_out(exact) +
 *     16 * 2^-24 * sum|x| (the segment, or the segment's prefix for a scan;
 *     tests/test_parity_signed_gpu.py).  Irregular segments: the same with
 *     sum|x| taken from the start of the 64-element row holding the
 *     segment's first element.  Exact-integer data is bit-exact.
 *   - Non-finite inputs: NaN / Inf * 0 in the MMA poisons the element's
 *     64-element row (the reference's engine.py:344 poisons a 16-wide tile
 *     row): outputs of segments running through it may be NaN (DESIGN.md
 *     section 5).
 *   - Argument errors are detected on the host before any launch and leave
 *     `out` untouched.  Status codes map 1:1 onto the reference exceptions:
 *     TC_BAD_LENGTH -> halftile.errors.BadLengthError, TC_BAD_CONFIG ->
 *     BadConfigError (errors.py:29-38).
 *   - `ws` is a caller-owned device workspace of at least
 *     tc_workspace_bytes(op, n, seg) bytes.  It MUST be zero-filled once at
 *     allocation; the kernels leave it in a reusable state.  One workspace
 *     must not be used by two in-flight calls at the same time.
 */
#ifndef TC_COLLECTIVES_H
#define TC_COLLECTIVES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define TC_OK 0
#define TC_BAD_LENGTH 1        /* -> BadLengthError (errors.py:29) */
#define TC_BAD_CONFIG 2        /* -> BadConfigError (errors.py:33) */
#define TC_BAD_ALIGNMENT 3     /* pointer not 16-byte aligned      */
#define TC_WORKSPACE_TOO_SMALL 4
#define TC_CUDA_ERROR 5        /* -> RuntimeError + tc_last_error() */
#define TC_NO_DEVICE 6         /* no sm_100 device / driver entry point */

/* output dtypes (engine.acc_dtype, engine.py:244-246: half | single) */
#define TC_F16 0
#define TC_F32 1
#define TC_F64 2               /* reduce only: fp64 partial for NCCL combine */
#define TC_BF16 3              /* input only (the *_ex entry points): bfloat16 */

/* op ids for tc_workspace_bytes */
#define TC_OP_REDUCE 0
#define TC_OP_SCAN 1
#define TC_OP_BN_STATS 2       /* tc_workspace_bytes(TC_OP_BN_STATS, N*C*HW, HW) */

/* Bytes of device workspace an op over n elements with segment size seg
 * needs (seg >= n means one segment: the grid/full variants). */
size_t tc_workspace_bytes(int op, int64_t n, int64_t seg);

/* Segmented sum: out[k] = sum(x[k*seg : min((k+1)*seg, n)]) for
 * k < ceil(n/seg), stored as out_dtype (TC_F16 | TC_F32 | TC_F64).
 * Replaces segmented_reduce (reduce.py:379). */
int tc_seg_reduce(const void* x, int64_t n, int64_t seg, void* out,
                  int out_dtype, void* ws, size_t ws_bytes, void* stream);

/* Same with an explicit input dtype: TC_F16 (binary16, as above) or TC_BF16
 * (bfloat16: same tcgen05 kind::f16 MMA with BF16 A/B operands, fp32
 * accumulation).  Extension beyond the reference (fp16 only), SURVEY.md
 * section 8(f)3. */
int tc_seg_reduce_ex(const void* x, int in_dtype, int64_t n, int64_t seg, void* out,
                     int out_dtype, void* ws, size_t ws_bytes, void* stream);

/* Full sum of n elements into out[0] (one output).  Replaces grid_reduce
 * (reduce.py:332).  Equivalent to tc_seg_reduce with seg = n. */
int tc_full_reduce(const void* x, int64_t n, void* out, int out_dtype,
                   void* ws, size_t ws_bytes, void* stream);

/* Segmented inclusive (exclusive != 0: exclusive) prefix sum, n outputs in
 * out_dtype (TC_F16 | TC_F32).  Replaces segmented_scan (scan.py:316); the
 * exclusive form equals the reference's shift-right-and-inject-zero
 * (scan.py:332-341).
 *   carry_in  (nullable, DEVICE, 1 double): the first segment continues a
 *             segment begun before x[0] whose running sum is *carry_in
 *             (cross-GPU carry of a sharded full scan).
 *   total_out (nullable, DEVICE, 1 double): receives the inclusive running
 *             sum of the last (open) segment, i.e. carry_in + sum(x) when
 *             seg >= n. */
int tc_seg_scan(const void* x, int64_t n, int64_t seg, void* out,
                int out_dtype, int exclusive, const double* carry_in,
                double* total_out, void* ws, size_t ws_bytes, void* stream);

/* Same with an explicit input dtype (TC_F16 | TC_BF16), see tc_seg_reduce_ex. */
int tc_seg_scan_ex(const void* x, int in_dtype, int64_t n, int64_t seg, void* out, int out_dtype,
                   int exclusive, const double* carry_in, double* total_out, void* ws,
                   size_t ws_bytes, void* stream);

/* Full (one-segment) scan.  Replaces grid_scan (scan.py:249). */
int tc_full_scan(const void* x, int64_t n, void* out, int out_dtype,
                 int exclusive, const double* carry_in, double* total_out,
                 void* ws, size_t ws_bytes, void* stream);

/* Irregular segments (extension; the paper elides
 * them, "irregular segmented reduction is implemented in terms
 * of regular segmented reduction").  Segment k covers
 * x[offsets[k], offsets[k+1]) for k < nseg; `offsets` is a DEVICE array of
 * nseg + 1 non-decreasing int64 with offsets[0] = 0 and offsets[nseg] = n
 * (empty segments allowed; the Python shim validates it, the kernels only
 * stay memory-safe on malformed offsets).  in_dtype TC_F16 | TC_BF16.
 * Same tile product as the regular path (the in-row prefix X.U on the tensor
 * core), with each row's segment starts taken from `offsets`.
 *
 * tc_irreg_reduce: out[k] = sum of segment k (0 for an empty one), out_dtype
 *   TC_F16 | TC_F32 | TC_F64.  One launch. */
int tc_irreg_reduce(const void* x, int in_dtype, int64_t n, const int64_t* offsets, int64_t nseg,
                    void* out, int out_dtype, void* ws, size_t ws_bytes, void* stream);

/* tc_irreg_scan: inclusive (exclusive != 0: exclusive) prefix sums restarted
 * at every segment start, n outputs (TC_F16 | TC_F32).  Two launches: the
 * carry each CTA range hands on (reads only the range tails behind the last
 * segment start), then the tile scan. */
int tc_irreg_scan(const void* x, int in_dtype, int64_t n, const int64_t* offsets, int64_t nseg,
                  void* out, int out_dtype, int exclusive, void* ws, size_t ws_bytes,
                  void* stream);

/* Batch-norm statistics (the TCU-reduction consumer the paper sketches,
 * PAPER.md:2185-2217) of an NCHW-contiguous tensor
 * x[N][C][HW] (in_dtype TC_F16 | TC_BF16): per channel c, mean[c] and the
 * biased variance var[c] over the N*HW elements, out_dtype TC_F32 | TC_F64
 * (DEVICE arrays of C).  One read of x: per (n, c) segment the shifted-data
 * moments sum(x - K_c), sum((x - K_c)^2), K_c = x[0][c][0], then a fixed-
 * order fp64 combine per channel (CUDA cores: the squares need the elements,
 * which a constant-B MMA cannot give).  ws >= tc_workspace_bytes(
 * TC_OP_BN_STATS, N*C*HW, HW); the scratch is cleared again after use.
 * launch.  One launch (the channel's last block combines in split order;
 * HW < 48: a per-segment kernel + a combine kernel), stream-ordered. */
int tc_bn_stats(const void* x, int in_dtype, int64_t N, int64_t C, int64_t HW, void* mean,
                void* var, int out_dtype, void* ws, size_t ws_bytes, void* stream);

/* Diagnostics: which kernel a tc_seg_reduce / tc_seg_scan call with these
 * arguments runs.  *mode: 0 LOCAL, 1 ROWS, 2 TILES, 3 GENERAL, 4 CHUNK,
 * 5 IRREG, 6 GSCR, 7 ROWSEG (whole segments per TMA row), 8 SPLIT (scan:
 * granules of 8 with the one granule a segment start splits re-summed).  *row_len: the
 * elements of one MMA row -- 64, or k * seg for ROWSEG (rows of k whole
 * segments).  A non-finite input poisons the outputs computed from its MMA
 * row accumulation: the 64-element row, the whole ROWSEG row for a reduce,
 * the 64-column chunk of the ROWSEG row for a scan. */
int tc_plan_info(int op, int64_t n, int64_t seg, int out_dtype, int has_carry, int has_total,
                 int* mode, int64_t* row_len);

/* Host <-> device copies of PAGEABLE host memory (the drop-in's numpy
 * arrays), staged through a pinned ring by a pool of host threads
 * (non-temporal stores) overlapped with the copy engine.
 * tc_h2d_pageable: stream-ordered on `stream`; returns once `src_host` may
 * be reused (every byte is in pinned memory or already on the device).
 * tc_d2h_pageable: ordered after earlier work on `stream`; returns when
 * `dst_host` holds the data.  One transfer at a time per process (calls
 * serialize).  Replaces the numpy <-> device conversion the reference does
 * not need (its arrays never leave the host: reduce.py:69-73). */
int tc_h2d_pageable(void* dst_dev, const void* src_host, size_t bytes, void* stream);
int tc_d2h_pageable(void* dst_host, const void* src_dev, size_t bytes, void* stream);

/* Human-readable name of a status code. */
const char* tc_status_string(int status);

/* Detail message of the last failing call on this host thread ("" if none). */
const char* tc_last_error(void);

/* Number of kernel launches issued by this host thread since the last call
 * to tc_reset_launch_count (used by bench.py's gpu_launches claim). */
uint64_t tc_launch_count(void);
void tc_reset_launch_count(void);

/* ABI version: (major << 16) | minor.  1.1 added the *_ex entry points,
 * 1.2 the tc_irreg_* entry points, 1.3 tc_bn_stats, 1.4 tc_plan_info,
 * 1.5 tc_h2d_pageable / tc_d2h_pageable. */
int tc_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TC_COLLECTIVES_H */
