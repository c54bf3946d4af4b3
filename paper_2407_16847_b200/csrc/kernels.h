// kernels.h -- launchers of the device kernels (internal).
#pragma once

#include <cuda_runtime.h>

#include "splat_internal.h"

namespace splat {

// Device view of a handle: what every kernel needs.
struct DevAcsr {
    const int4 *seg;        // [N][4]: (start, step, count, offset-in-row)
    const uint8_t *nseg;    // [N]
    const int64_t *row_ptr; // [N+1]
    int n;
    long long nnz;
    // tile plan
    const int32_t *qt_ptr;  // [n_qt+1]
    const int32_t *kv;      // [n_entries]
    const int32_t *order;   // [n_qt]
    int n_qt;
    // query-tile pairs (fused kernel)
    const int32_t *pair_ent;    // kv | kUseA | kUseB | kPartA | kPartB
    const int4 *pair_info;      // [n_pairs][2]: (pair, e0, e1, jA0), (jA1, jB1, 0, 0) in pair_order order
    const uint4 *masks;         // [n_masks][128]: row column masks
    const uint4 *mask_rec;      // [n_masks][128][2]: R-SpMM row records (16 x u16 per row)
    const uint8_t *mask_cnt;    // [n_masks][128]: live columns per row
    const int32_t *kv_mask;     // [n_entries]: mask id per (query tile, key tile) entry, -1 = FULL
    const uint32_t *qt_bits;    // [n_entries]: chunk live (bit 4 quad + w) / full (bit 16 + 4 quad + w)
    int n_pairs, n_buckets;
    int bucket_start[kMaxBuckets + 1];
    // single query tiles (split-group fused kernel)
    const int4 *t_info;         // [n_qt]: (tile, j0, j1, 0), bucketed longest first
    int t_n_buckets;
    int row_classes;            // t_info tiles are packed 64-row segment pairs (a | b << 16)
    int t_bucket_start[kMaxBuckets + 1];
    unsigned long long *sched;  // [2]: dynamic work counter + done counter of the split kernel
    int t_n;                    // split-kernel units per (b, h) (t_info rows)
    int t_max_len, t_entries;   // longest whole-tile unit, plan entries per (b, h) of the split kernel
    // the split-K unit list (long tiles in parts): swapped in by the launch for few heads per GPU
    const int4 *t_info_ks;
    int t_n_ks, t_n_buckets_ks;
    int t_bucket_start_ks[kMaxBuckets + 1];
    // split-K partial results of the launch slot (plan.cpp: n_ksplit long tiles per head, up to
    // ks_pmax parts each): per (head, split tile, part, row) the normalised partial O (bf16, 64 per
    // row) and its lse2; per (head, split tile) the arrival counter (zero between launches)
    void *ks_o;
    float *ks_lse;
    unsigned *ks_cnt;
    int n_ksplit, ks_pmax;
    // the descriptor of a descriptor-built handle (has_pat = 1): kernels may evaluate a row's runs
    // in closed form (row_segments) instead of loading them; 0 for mask-ingest handles
    splat_pattern pat;
    int has_pat;
};

cudaError_t launch_acsr_build(const splat_pattern &p, int4 *seg, uint8_t *nseg, int64_t *row_ptr,
                              cudaStream_t st);
cudaError_t launch_acsr_scan(int64_t *row_ptr, int n, cudaStream_t st);
// unfused R-SDDMM (sddmm) / R-SpMM of plain STRIDED(l) on the permuted BLOCKED(nk) handle; S / P stay in
// the natural ACSR order of `nat`
cudaError_t launch_unfused_permuted(bool sddmm, const DevAcsr &perm, const DevAcsr &nat, int l, int nk, int R,
                                    const void *X, const void *Y, int BH, int d, float scale, void *out,
                                    cudaStream_t st, int *n_launch);
// fused bf16 MHSA of plain STRIDED(l) on residue-major views: `perm` is the BLOCKED(nk) handle of the
// permuted mask (N = l nk; nk | 128 with R = 128 / nk, or 128 | nk with R = 1); d = 64 or 128
cudaError_t launch_mhsa_tc_permuted(const DevAcsr &perm, int l, int nk, int R, const void *Q, const void *K,
                                    const void *V, int BH, int d, float scale, void *O, cudaStream_t st,
                                    int *n_launch);
// explicit bit mask (row stride ceil(n/32) words, LSB first) -> greedy runs; *bad = min over
// irregular rows of (row << 32 | first column of run max_runs + 1), all ones if none
cudaError_t launch_acsr_from_mask(const uint32_t *mask, int n, int max_runs, int4 *seg, uint8_t *nseg,
                                  int64_t *row_ptr, unsigned long long *bad, cudaStream_t st);

// data-layout reordering (layout.cu): Y (M^T's ACSR order) from X (M's); R-SpMM from column-compressed P
cudaError_t launch_transpose_values(const DevAcsr &A, const DevAcsr &AT, const void *X, void *Y, bool bf16, int BH,
                                    cudaStream_t st);
cudaError_t launch_rspmm_cc(const DevAcsr &A, const DevAcsr &AT, const void *PT, const void *V, bool bf16, int BH,
                            int d, void *O, cudaStream_t st, int align_x = 0);

// SIMT kernels (fp32 path; any d <= 256)
cudaError_t launch_rsddmm_simt(const DevAcsr &A, const void *Q, const void *K, bool bf16, int BH, int d,
                               float scale, float *S, cudaStream_t st);
cudaError_t launch_softmax(const DevAcsr &A, const float *S, void *P, bool p_bf16, int BH,
                           cudaStream_t st);
cudaError_t launch_rspmm_simt(const DevAcsr &A, const void *P, const void *V, bool bf16, int BH, int d,
                              void *O, cudaStream_t st);
cudaError_t launch_mhsa_simt(const DevAcsr &A, const void *Q, const void *K, const void *V, bool bf16,
                             int BH, int d, float scale, void *O, cudaStream_t st);

// sm_100a tensor-core kernels (bf16, d in {64, 128}); return cudaErrorNotSupported
// when the configuration is outside what they implement.
// d = 64 streaming fused kernel (tc_fused64.cu); A.sched = the call's launch-slot work counter
cudaError_t launch_mhsa64(const DevAcsr &A, const void *Q, const void *K, const void *V, int BH, float scale,
                          void *O, cudaStream_t st);
cudaError_t launch_mhsa_tc(const DevAcsr &A, const void *Q, const void *K, const void *V, int BH, int d,
                           float scale, void *O, cudaStream_t st, int *n_launch);
// Residue decomposition of STRIDED_LOCAL (splat_acsr_s::sub_band): pass 1 over the strided
// component in residue-major order, pass 2 over the causal band merging both partial softmaxes.
cudaError_t launch_mhsa_tc_residue(const DevAcsr &band, const DevAcsr &str, int l, int nk, int R, float *lse,
                                   const void *Q, const void *K, const void *V, int BH, int d, float scale, void *O,
                                   cudaStream_t st, int *n_launch);
// The same decomposition in ONE launch: `mix` is the merged plan (strided-pass pairs [0, u1), band-pass
// pairs [u1, u1 + u2)); units run head-interleaved and a band unit's merging epilogue waits on the
// head's counter in `dep` ([kLseHeads + 1], zero between launches; reset by the last CTA).
cudaError_t launch_mhsa_tc_residue1(const DevAcsr &mix, int u1, int u2, int l, int nk, int R, float *lse, unsigned *dep,
                                    const void *Q, const void *K, const void *V, int BH, int d, float scale, void *O,
                                    cudaStream_t st, int *n_launch);
// Unfused R-SDDMM (sddmm = true: X = Q, Y = K, out = S) or R-SpMM (X = P, Y = V, out = O) over the
// residue decomposition: pass 1 on the strided sub-pattern (residue-major views), pass 2 on the band.
cudaError_t launch_unfused_residue(bool sddmm, const DevAcsr &band, const DevAcsr &str, const DevAcsr &nat, int l,
                                   int nk, int R, const void *X, const void *Y, int BH, int d, float scale, void *out,
                                   cudaStream_t st, int *n_launch);
cudaError_t launch_rsddmm_tc(const DevAcsr &A, const void *Q, const void *K, int BH, int d, float scale, float *S,
                             cudaStream_t st);
cudaError_t launch_rspmm_tc(const DevAcsr &A, const void *P, const void *V, int BH, int d, void *O,
                            cudaStream_t st);

}  // namespace splat
