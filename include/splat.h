/*
 * splat.h -- C ABI of the B200-native SPLAT sparse-MHSA hot path
 *            (arXiv 2407.16847, "SPLAT: A framework for optimised GPU code-
 *            generation for SParse reguLar ATtention").
 *
 * The library computes, per (batch b, head h), the sparse multi-head
 * self-attention of PAPER.md Eq. 1:
 *
 *     O = [ softmax( M (x) scale * Q K^T ) ] V
 *          `------- R-SDDMM -------'   (Sec. 7)
 *         `----------- R-SpMM ------------'  (Sec. 8)
 *
 * where M is a *regular* (affine-compressible, Def. 1) mask given
 * by a pattern descriptor, and the softmax of row i runs over the non-zeros
 * of row i only.  The mask is never materialised: it is stored in ACSR form
 * (affine-compressed sparse row, Sec. 5): per row a short list of
 * affine runs (start, step, count) -- the paper's (a, b, nnzs) triplet with
 * a = 1/step, b = -start/step, nnzs = count -- and a row_ptr array giving
 * each row's offset in the row-compressed row-major value arrays (Fig. 5(b)).
 * Rows of the Longformer / BigBird / Sparse-Transformer patterns are unions
 * of up to 3 runs, so this ABI generalises ACSR to <= SPLAT_MAX_SEGS runs
 * per row (reading R-3); the paper's format is the 1-run case.
 *
 * The paper's workflow (Listing 4) is "analyse + code-generate
 * once per mask, launch many times".  Here: splat_acsr_build() once per
 * pattern (metadata + tile plan, device resident), then any number of
 * asynchronous compute calls.
 *
 * Conventions for every compute call
 *   - Tensors are caller-owned DEVICE buffers on the handle's device,
 *     contiguous, shape [B, H, N, d] with d innermost (Q, K, V, O) or
 *     [B, H, nnz] (S, P: row-compressed row-major ACSR order, element x of
 *     row i at offset row_ptr[i] + x; within a row, columns ascend).  Base
 *     pointers must be 16-byte aligned.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     asynchronous on it and never synchronise or copy to host.  Exceptions:
 *     the strided-row decomposition allocates its lse scratch (4*B*H*N bytes,
 *     handle-owned) on the first call with a larger B*H, and
 *     splat_sparse_mhsa_host creates its pipeline streams on first use.
 *   - The return status covers argument validation and the launch
 *     (cudaGetLastError -> SPLAT_ERR_CUDA); a kernel fault surfaces at the
 *     caller's next synchronisation.
 *   - On any error, splat_last_error() returns a thread-local message.
 *   - There is no CPU fallback: a compute call on a handle without a device
 *     (device < 0) fails with SPLAT_ERR_INVALID_ARG.
 *   - The handle's metadata and plan are immutable after build, but a handle
 *     also owns mutable device state used by the compute calls (the fused
 *     d = 64 kernel's work counter, the strided-row lse scratch): compute
 *     calls on ONE handle must be ordered (one stream, or event-ordered);
 *     use one handle per concurrent stream.  Different handles are
 *     independent.
 */
#ifndef SPLAT_H_
#define SPLAT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPLAT_MAX_SEGS 4

typedef enum {
    SPLAT_OK = 0,
    SPLAT_ERR_INVALID_ARG = 1,   /* bad descriptor parameter / pointer / handle */
    SPLAT_ERR_NOT_REGULAR = 2,   /* reserved: explicit-mask ingest */
    SPLAT_ERR_SHAPE = 3,         /* tensor shape disagrees with the handle */
    SPLAT_ERR_UNSUPPORTED = 4,   /* valid request outside the implemented set */
    SPLAT_ERR_CUDA = 5,          /* CUDA runtime / launch error */
    SPLAT_ERR_OOM = 6            /* device allocation failed (build only) */
} splat_status;

typedef enum { SPLAT_BF16 = 0, SPLAT_FP32 = 1 } splat_dtype;

/* Pattern kinds.  pred(i, j) is "query row i attends key column j".
 *   WINDOW(lo, hi)        i-lo <= j <= i+hi            paper "Windowed" (Fig. 2);
 *                                                        causal sliding window of W keys = WINDOW(W-1, 0)
 *   BLOCKED(block)        floor(i/w) == floor(j/w)     paper "Blocked" (Fig. 2)
 *   STRIDED(stride)       j = i (mod X)                paper "Strided" (Fig. 2; App. B)
 *   DILATED(stride, radius) |i-j| <= rho*delta and j = i (mod delta)   (dilated window, delta = stride, rho = radius)
 *   GLOBAL_LOCAL(lo, hi, n_global)  i < g or j < g or i-lo <= j <= i+hi   (Longformer, cited P:139)
 *   BIGBIRD(block, radius)  with qb = i/bs, kb = j/bs, nb = ceil(N/bs):
 *                         qb in {0, nb-1} or kb in {0, nb-1} or |qb-kb| <= radius  (blocked family, P:139;
 *                         no random blocks)
 *   STRIDED_LOCAL(stride, causal=1)  j <= i and (i-j < l or (i-j) mod l == 0)   (Sparse Transformer strided)
 */
typedef enum {
    SPLAT_WINDOW = 0, SPLAT_BLOCKED = 1, SPLAT_STRIDED = 2, SPLAT_DILATED = 3,
    SPLAT_GLOBAL_LOCAL = 4, SPLAT_BIGBIRD = 5, SPLAT_STRIDED_LOCAL = 6
} splat_kind;

/* Pattern descriptor.  All fields int32; unused fields must be 0.
 * Valid ranges (else SPLAT_ERR_INVALID_ARG, mirroring SPEC S:45 "parameters
 * positive and <= seq_len"): 1 <= seq_len <= 2^24; 0 <= lo, hi <= seq_len;
 * 1 <= block <= seq_len; 1 <= stride <= seq_len; 0 <= radius <= seq_len;
 * 0 <= n_global <= seq_len.
 * SPLAT_ERR_UNSUPPORTED: GLOBAL_LOCAL with n_global == 1 and BIGBIRD with
 * block == 1 (the canonical greedy run decomposition pairs an isolated
 * column with the next one there, R-11), STRIDED_LOCAL with
 * causal == 0. */
typedef struct {
    int32_t kind;       /* splat_kind */
    int32_t seq_len;    /* N */
    int32_t lo, hi;     /* WINDOW, GLOBAL_LOCAL */
    int32_t block;      /* BLOCKED, BIGBIRD */
    int32_t n_global;   /* GLOBAL_LOCAL */
    int32_t stride;     /* STRIDED X, DILATED delta, STRIDED_LOCAL l */
    int32_t radius;     /* DILATED rho, BIGBIRD sliding radius (blocks) */
    int32_t causal;     /* STRIDED_LOCAL: must be 1 */
    int32_t reserved[7];
} splat_pattern;

typedef struct splat_acsr_s *splat_acsr;     /* opaque handle */

/* ---------------------------------------------------------------------------
 * splat_acsr_build -- ACSR metadata build + tile plan.
 *
 * Paper: analysis passes checkRegularity + generateACSRMetadata (Listing 4
 * P:682-683; construction Sec. 5.1) and the tiling / span /
 * alignment metadata (Sec. 7.2, Sec. 8.2, spmmMetaOpt
 * P:639).  Each row's runs are the canonical greedy decomposition of the
 * row's column set (2x2 solve of the first two columns, extended
 * while consecutive columns satisfy P:219, restarted at the first failing
 * column), computed in closed form from the descriptor by one GPU thread
 * per row, followed by a device scan for row_ptr.  The tile planner then
 * lists, per 128-row query tile, the 128-column key tiles that any of its
 * rows touches (span specialisation), flagged FULL (every row
 * covers the whole tile: no masking) or PARTIAL.
 *
 *   p       descriptor (host pointer, read only during the call)
 *   device  CUDA device ordinal; or -1 for a host-only INSPECTION handle
 *           (metadata + plan computed on the host by the same closed form;
 *           usable with splat_acsr_info / _copy_meta / _plan_*, rejected by
 *           every compute call)
 *   stream  cudaStream_t used for the build kernels (NULL = default)
 *   out     receives the handle (caller owns it; free with _destroy)
 * Synchronous: returns after metadata and plan are resident.
 * Errors: INVALID_ARG, UNSUPPORTED (see splat_pattern), OOM, CUDA.
 * ------------------------------------------------------------------------- */
splat_status splat_acsr_build(const splat_pattern *p, int device, void *stream, splat_acsr *out);

/* Sizes of a built handle (any pointer may be NULL).
 *   n        sequence length N
 *   nnz      non-zeros per (b, h) = row_ptr[N]
 *   max_segs largest number of runs in any row (<= SPLAT_MAX_SEGS)
 *   density  nnz / N^2 (the paper's densityAnalysis) */
splat_status splat_acsr_info(splat_acsr a, int32_t *n, int64_t *nnz, int32_t *max_segs,
                             double *density);

/* Copy the ACSR metadata to caller-owned HOST buffers (synchronous):
 *   seg      int32 [N][SPLAT_MAX_SEGS][3]: (start, step, count) of each run,
 *            runs in ascending column order, unused runs all zero
 *   nseg     uint8 [N]: number of runs in the row
 *   row_ptr  int64 [N+1]: exclusive prefix sum of the per-row counts
 * Any pointer may be NULL to skip it. */
splat_status splat_acsr_copy_meta(splat_acsr a, int32_t *seg, uint8_t *nseg, int64_t *row_ptr);

/* Tile-plan geometry: query-tile rows bm, key-tile columns bn, number of
 * query tiles (ceil(N/bm)) and of (query tile, key tile) entries. */
splat_status splat_plan_info(splat_acsr a, int32_t *bm, int32_t *bn, int32_t *n_qtiles,
                             int32_t *n_entries);

/* Copy the tile plan to caller-owned HOST buffers (synchronous):
 *   qt_ptr   int32 [n_qtiles+1]: entries of query tile t are [qt_ptr[t], qt_ptr[t+1])
 *   kv       int32 [n_entries]: key-tile index in bits 0..23, bit 24 set = PARTIAL
 *            (some row of the query tile misses some column of the key tile);
 *            key tiles of a query tile ascend
 *   order    int32 [n_qtiles]: query tiles, most key tiles first (LPT order
 *            used by the persistent kernels; ties by tile index) */
splat_status splat_plan_copy(splat_acsr a, int32_t *qt_ptr, int32_t *kv, int32_t *order);

/* Work of the d = 64 fused (split-group) kernel: its query tiles are two 64-row segments; with
 * row_classes = 1 the planner regrouped the segments by row class (rows touching nearly every key
 * block share tiles) because that needs fewer (tile, key window) entries; n_split_entries
 * is the number of entries per (b, h) that kernel walks. */
splat_status splat_plan_split_info(splat_acsr a, int32_t *row_classes, int32_t *n_split_entries);

/* Inspection of the split kernel's plan (host copies, synchronous): splat_plan_sizes(a, 0) units
 * per (b, h), (a, 1) entries (natural ones first, then the row-class ones), (a, 2) masks;
 * splat_plan_split_copy copies units int32 [n][4] (tile -- or segments a | b << 16 when
 * row_classes -- , j0, j1, 0), kv int32 [entries] (window start / 64 | PARTIAL bit 24; a row-class
 * entry with bit 25 set is a composite window of the two 64-column key blocks a = bits 0-11 (window
 * columns 0-63) and b = bits 12-23 (columns 64-127)), mask_id int32 [entries] (-1 = FULL) and masks
 * uint32 [n_masks][128 rows][4] (column bits of the window). */
int64_t splat_plan_sizes(splat_acsr a, int32_t which);
splat_status splat_plan_split_copy(splat_acsr a, int32_t *units, int32_t *kv, int32_t *mask_id, uint32_t *masks);

/* Split-K unit list of the same kernel, taken by a launch when its longest
 * whole tile would outlast a tile group's average share of the work (few heads per GPU): every tile
 * with more than 8 entries is cut into parts with contiguous entry ranges whose partial softmax
 * results the last part merges.  splat_plan_sizes(a, 3) = its units per (b, h) (0: no long tile);
 * units int32 [n][4] = (tile as above, j0, j1, part | parts << 8 | split-tile index << 16; 0 for a
 * whole tile), same entry numbering as splat_plan_split_copy. */
splat_status splat_plan_ksplit_copy(splat_acsr a, int32_t *units);

/* Free a handle and its device memory.  NULL is a no-op. */
splat_status splat_acsr_destroy(splat_acsr a);

/* ---------------------------------------------------------------------------
 * splat_rsddmm -- R-SDDMM (PAPER Sec. 7, Listing 1
 * P:412-431; Eq. 1):
 *     S[b,h, row_ptr[i]+x] = scale * < Q[b,h,i,:], K[b,h,c_x(i),:] >
 * for every row i and its x-th column c_x(i) (ascending).
 *   Q, K   device [B,H,N,d], dtype dt (SPLAT_BF16: bf16; SPLAT_FP32: fp32)
 *   S      device float32 [B,H,nnz] (written)
 *   d      head dim: 64 or 128 for SPLAT_BF16 (tensor-core path);
 *          1..256 for SPLAT_FP32 (SIMT fp32 path, no TF32)
 * Accumulation in fp32.
 * ------------------------------------------------------------------------- */
splat_status splat_rsddmm(splat_acsr a, const void *Q, const void *K, splat_dtype dt,
                          int32_t B, int32_t H, int32_t d, float scale, float *S, void *stream);

/* ---------------------------------------------------------------------------
 * splat_sparse_softmax -- row softmax over the ACSR values (SURVEY §8(a)
 * row a4; "computing the softmax for each input row", Listing 4
 * P:687/P:707; the paper calls cuDNN here):
 *     P[b,h,row_ptr[i]+x] = exp(S_x - m_i) / sum_y exp(S_y - m_i),
 *     m_i = max_y S[b,h,row_ptr[i]+y].
 * The scale is already applied by splat_rsddmm.  Empty rows: no-op.
 *   S      device float32 [B,H,nnz] (read)
 *   P      device [B,H,nnz] of p_dt (bf16 or fp32) (written); may not alias S
 * fp32 arithmetic.
 * ------------------------------------------------------------------------- */
splat_status splat_sparse_softmax(splat_acsr a, const float *S, void *P, splat_dtype p_dt,
                                  int32_t B, int32_t H, void *stream);

/* ---------------------------------------------------------------------------
 * splat_rspmm -- R-SpMM (PAPER Sec. 8, Listing 2
 * P:553-568):
 *     O[b,h,i,:] = sum_x P[b,h,row_ptr[i]+x] * V[b,h,c_x(i),:]
 *   P      device [B,H,nnz] of dtype dt
 *   V, O   device [B,H,N,d] of dtype dt (O written; empty rows -> 0)
 *   d      as for splat_rsddmm
 * fp32 accumulation; O rounded to dt (round to nearest even).
 * ------------------------------------------------------------------------- */
splat_status splat_rspmm(splat_acsr a, const void *P, const void *V, splat_dtype dt,
                         int32_t B, int32_t H, int32_t d, void *O, void *stream);

/* ---------------------------------------------------------------------------
 * splat_sparse_mhsa -- fused sparse MHSA (Eq. 1
 * P:134-137; the paper runs Listing 4's rsddmm -> softmax -> rspmm with HBM
 * buffers; this call fuses them so S and P never reach HBM):
 *     O[b,h] = softmax( M (x) scale * Q[b,h] K[b,h]^T ) V[b,h]
 *   Q, K, V, O   device [B,H,N,d] of dtype dt (O written; empty rows -> 0)
 *   d            as for splat_rsddmm
 *   scale        score scale, positive and finite (configs use 1/sqrt(d);
 *                1.0 reproduces Eq. 1); else SPLAT_ERR_INVALID_ARG
 * SPLAT_BF16 runs the sm_100a tensor-core kernel (TMA + tcgen05 + TMEM,
 * online softmax, fp32 accumulation); SPLAT_FP32 runs the SIMT fp32 kernel.
 * Strided masks are run on residue-major views of Q/K/V/O (rows grouped by
 * i mod stride, the paper's row classes P:367-374): STRIDED_LOCAL (d = 128)
 * as two passes merged by log-sum-exp, plain STRIDED (N = stride * nk, nk a
 * power of two) as one block-diagonal pass; the result is the same Eq. 1 O
 * in natural row order (§9c).
 * ------------------------------------------------------------------------- */
splat_status splat_sparse_mhsa(splat_acsr a, const void *Q, const void *K, const void *V,
                               splat_dtype dt, int32_t B, int32_t H, int32_t d, float scale,
                               void *O, void *stream);

/* ---------------------------------------------------------------------------
 * splat_sparse_mhsa_host -- the same fused call from HOST buffers (the
 * end-to-end path a user without device-resident tensors takes):
 * cudaMemcpyAsync of Qh, Kh, Vh into the caller-owned device staging
 * buffers dQ, dK, dV, splat_sparse_mhsa into dO, cudaMemcpyAsync of dO into
 * Oh.  The (b, h) slices are pipelined in chunks over three handle-owned
 * streams (host->device copy of chunk c+1 and device->host copy of chunk c-1
 * overlap the kernel on chunk c; (b, h) slices are independent, Eq. 1 per
 * head); `stream` waits for all of it, so the call is asynchronous
 * with respect to the host exactly as before (synchronise `stream` before
 * reading Oh).  Host buffers should be page-locked for the copies to be
 * asynchronous.  Shapes, dtypes and errors as splat_sparse_mhsa.
 * ------------------------------------------------------------------------- */
splat_status splat_sparse_mhsa_host(splat_acsr a, const void *Qh, const void *Kh, const void *Vh,
                                    splat_dtype dt, int32_t B, int32_t H, int32_t d, float scale,
                                    void *Oh, void *dQ, void *dK, void *dV, void *dO, void *stream);

/* ---------------------------------------------------------------------------
 * Thread-block tiling analysis of the R-SDDMM point set (
 * paper Sec. 7.2-7.3, App. A-C).  Host-only: no device,
 * no stream, synchronous, thread-safe (no shared state).
 *
 * P = {(x, y) : query row y attends key column x} of the descriptor's mask.
 * A thread block of m x n threads with anchor (x, y) and stretch s computes
 * Comp = {(x + c s, y + r s) : r < m, c < n} -- m thread ROWS (y extent), n
 * thread COLUMNS (x extent), reading T-1 -- and covers Comp ∩ P
 * (Def. 2).  Every arrangement here uses one stretch for all of
 * its blocks.
 *
 *   splat_poset_tile   poset tiling (Def. 5, Alg. 1):
 *                      each iteration anchors one block at every minimal
 *                      uncovered point (the set ⊤), until P is covered.
 *                      stretch > 0 forces s; stretch == 0 selects it
 *                      (Sec. 7.3.1): 1 for polygonal masks (every
 *                      row contiguous, App. A), the cheapest divisor of the
 *                      row stride X for strided masks (App. B), else the
 *                      cheapest s in [1, min(N, 64)]; ties -> fewer blocks.
 *   splat_naive_tile   App. C Def. 8: m-row patches from row
 *                      0, each tiled left to right with unit-stretch blocks
 *                      from its leftmost to its rightmost non-zero column.
 *   splat_tiling_cost_eval  the cost report of a caller-given arrangement.
 *
 *   anchors  host int32 [cap][2] = (x, y) per block in placement order (Alg. 1:
 *            iteration, then ascending y); the first min(cap, lambda) are
 *            written; may be NULL when cap == 0 (cost->lambda gives the size).
 *   cost     required: lambda, |P|, phi_TD = |(∪ Comp) \ P| (Comp points
 *            outside the N x N mask count), phi_R = lambda m n - |P| - phi_TD,
 *            phi_RU = |P| / (lambda m n), phi_CMR = mean of 1/Str = 1/s
 *            (Def. 3), cost = lambda / phi_CMR (Def. 4).
 * Errors: INVALID_ARG (null pointers, m or n outside [1, 4096], stretch
 * outside [0 (poset) or 1 (eval), N], negative anchors, or -- eval only -- an
 * arrangement whose covers miss a point of P, named in splat_last_error),
 * UNSUPPORTED (seq_len > 8192: the analysis keeps P as an N x N bitset).
 * ------------------------------------------------------------------------- */
typedef struct {
    int64_t lambda;     /* number of thread blocks */
    int64_t points;     /* |P| */
    int64_t phi_td;     /* collective thread divergence */
    int64_t phi_r;      /* redundant compute */
    double phi_ru;      /* reuse */
    double phi_cmr;     /* coalesced memory requests */
    double cost;        /* lambda / phi_cmr */
    int32_t stretch, m, n, reserved;
} splat_tiling_cost;

splat_status splat_poset_tile(const splat_pattern *p, int32_t m, int32_t n, int32_t stretch,
                              int32_t *anchors, int64_t cap, splat_tiling_cost *cost);
splat_status splat_naive_tile(const splat_pattern *p, int32_t m, int32_t n, int32_t *anchors,
                              int64_t cap, splat_tiling_cost *cost);
splat_status splat_tiling_cost_eval(const splat_pattern *p, int32_t m, int32_t n, int32_t stretch,
                                    const int32_t *anchors, int64_t n_blocks, splat_tiling_cost *cost);

/* ---------------------------------------------------------------------------
 * splat_acsr_from_mask -- ACSR build from an EXPLICIT bit mask (SURVEY §8(f)
 * NEXT #2): the paper's analysis pass as written, checkRegularity(Mask) +
 * generateACSRMetadata(Mask) (Listing 4, Sec. 5.1).
 *
 * Each row's non-zero columns are split into canonical greedy runs (reading
 * R-4: 2x2 solve on the first two unconsumed columns, extended while
 * the next column passes P:219, restarted at the first failing column) by a
 * GPU kernel, one warp per row; then row_ptr is scanned and the tile plan is
 * built exactly as for splat_acsr_build.  The handle works with every compute
 * call (no strided-row decomposition: there is no descriptor).
 *
 *   mask      n rows of ceil(n/32) uint32 words, row-major, column j of row i
 *             at bit (j % 32) of word i * ceil(n/32) + j / 32 (LSB first);
 *             bits >= n in a row's last word are ignored.  A DEVICE pointer
 *             on `device` (read only during the call), or a HOST pointer when
 *             device == -1 (inspection handle, computed on the host).
 *   n         1 <= n <= 131072 (the mask is n^2/8 bytes)
 *   max_runs  1..SPLAT_MAX_SEGS: 1 is Def. 1's regularity; 4
 *             admits the multi-run rows of reading R-3
 *   out       receives the handle (caller owns it; free with _destroy)
 *   bad_row, bad_col  (may be NULL) -1, or on NOT_REGULAR the first offending
 *             point in row-major order: the first row needing more than
 *             max_runs runs and the column that would start run max_runs+1
 *             (for max_runs = 1 the first column breaking the
 *             row's affine fit, e.g. column 5 of {0, 2, 4, 5}).
 * Synchronous.  Errors: INVALID_ARG, NOT_REGULAR (no handle), OOM, CUDA.
 * ------------------------------------------------------------------------- */
splat_status splat_acsr_from_mask(const uint32_t *mask, int32_t n, int32_t max_runs, int device, void *stream,
                                  splat_acsr *out, int32_t *bad_row, int32_t *bad_col);

/* ---------------------------------------------------------------------------
 * Data-layout reordering (PAPER "Data-layout reordering"
 * P:722, density analysis Listing 4 line 5 P:716, Fig. 15).  R-SDDMM
 * and the softmax produce S / P row-compressed & row-major (ACSR order of M);
 * the paper transposes P to column-compressed & column-major before its SIMT
 * R-SpMM when the mask density reaches alpha = 0.10, so that a column's
 * consecutive rows are read from consecutive addresses.
 *
 * splat_acsr_transpose: handle `at` of M^T (row j of M^T = the rows i with j
 *   in cols(i), ascending; greedy runs, reading R-4), built from a's runs
 *   through the mask-ingest builder on the same device (host handle if a is
 *   one).  Synchronous; allocates at build time only.  Errors: INVALID_ARG,
 *   UNSUPPORTED (N > 131072), NOT_REGULAR (a column of M needs more than
 *   SPLAT_MAX_SEGS runs), OOM, CUDA.  Free `at` with splat_acsr_destroy.
 * splat_transpose_values: Y[b,h, row_ptr_T[j] + rank of i in row j of M^T]
 *   = X[b,h, row_ptr[i] + rank of j in row i] for every non-zero (i, j):
 *   X, Y device [B,H,nnz] of dtype dt (bf16 or fp32), caller-owned; async on
 *   stream.  `at` must be splat_acsr_transpose(a).
 * splat_rspmm_cc: R-SpMM from column-compressed P (PT as written by
 *   splat_transpose_values): O[b,h,i,:] = sum_j PT[b,h, row_ptr_T[j] +
 *   rank_T(j, i)] V[b,h,j,:], SIMT with fp32 accumulation (the paper's
 *   precision), 1 <= d <= 256, V and O [B,H,N,d] of dtype dt.
 * splat_layout_choice: 1 (column-compressed) when nnz / N^2 >= alpha, else 0
 *   (row-compressed) -- the paper's density classification; 0 for NULL.
 * ------------------------------------------------------------------------- */
splat_status splat_acsr_transpose(splat_acsr a, void *stream, splat_acsr *at);
splat_status splat_transpose_values(splat_acsr a, splat_acsr at, const void *X, void *Y, splat_dtype dt,
                                    int32_t B, int32_t H, void *stream);
splat_status splat_rspmm_cc(splat_acsr a, splat_acsr at, const void *PT, const void *V, splat_dtype dt,
                            int32_t B, int32_t H, int32_t d, void *O, void *stream);
int32_t splat_layout_choice(splat_acsr a, double alpha);

/* Algorithmic FLOPs of one fused call: 4 * nnz * d * B * H (QK^T and PV at
 * 2*nnz*d each; the softmax is not counted; SURVEY reading A-14). */
double splat_flops(splat_acsr a, int32_t B, int32_t H, int32_t d);

/* Number of kernel launches the last successful compute call on this thread
 * issued (instrumentation for the bench's gpu_launches count). */
int32_t splat_last_launch_count(void);

/* Number of device allocations the library has made in this process (all of
 * them at handle build time: compute calls never allocate, SURVEY §8(b)
 * "Ownership"; the tests check the count does not move across compute calls). */
int64_t splat_device_alloc_count(void);

/* Thread-local message describing the last error on this thread ("" if none). */
const char *splat_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SPLAT_H_ */
