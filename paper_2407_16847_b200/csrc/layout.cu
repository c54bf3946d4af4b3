// layout.cu -- data-layout reordering of the ACSR values for R-SpMM (
// PAPER "Data-layout reordering" P:722 and Fig. 15).
//
// The paper's density analysis (Listing 4 line 5) classifies a mask as dense when its
// density reaches alpha and then transposes the ACSR values from the row-compressed & row-major
// layout R-SDDMM writes to a column-compressed & column-major one before its SIMT R-SpMM, whose
// threads then read consecutive rows of a column from consecutive addresses.  Here:
//
//   transpose_values_kernel : Y in the ACSR order of M^T (column-compressed: column j's rows
//       ascending at row_ptr_T[j] + rank) from X in M's order.  One warp per row i of M, lanes over
//       its non-zeros; the destination index (rank of i among the rows of column j, from M^T's
//       affine runs, reading A-7) is computed once and reused for every (b, h).
//   rspmm_cc_kernel : O[i, :] = sum_j PT[row_ptr_T[j] + rank_T(j, i)] V[j, :] (SIMT, fp32
//       arithmetic, the paper's precision P:166).  A CTA owns 32 query rows (lane = row) of one
//       (b, h) and ceil(d / 32) warps (warp w: output columns 32 w .. 32 w + 31); it walks the key
//       columns of the rows' span, reads the 32 rows' values of column j with one coalesced load
//       (consecutive rows of a step-1 run are consecutive in PT), and accumulates p V[j, :]
//       (V[j, 32 w + t] broadcast by shuffle).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace splat {
namespace {

__device__ __forceinline__ float ld_f(const float *p) { return *p; }
__device__ __forceinline__ float ld_f(const __nv_bfloat16 *p) { return __bfloat162float(*p); }
__device__ __forceinline__ void st_f(float *p, float v) { *p = v; }
__device__ __forceinline__ void st_f(__nv_bfloat16 *p, float v) { *p = __float2bfloat16_rn(v); }

// Column of the x-th non-zero of a row with runs g (start, step, count, offset-in-row).
__device__ __forceinline__ int col_at(const int4 *g, int ns, int x)
{
    int c = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s)
        if (s < ns && x >= g[s].w && x < g[s].w + g[s].z) c = g[s].x + g[s].y * (x - g[s].w);
    return c;
}

// Rank of column c among the non-zeros of a row with runs g, or -1 when c is not one of them
// (reading A-7: (c - start) % step == 0 and 0 <= (c - start) / step < count).
__device__ __forceinline__ int rank_of(const int4 *g, int ns, int c)
{
    int r = -1;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        if (s < ns) {
            const int dlt = c - g[s].x;
            if (dlt >= 0) {
                const int q = g[s].y == 1 ? dlt : dlt / g[s].y;
                if (q * g[s].y == dlt && q < g[s].z) r = g[s].w + q;
            }
        }
    }
    return r;
}

template <typename T>
__global__ void __launch_bounds__(256)
transpose_values_kernel(DevAcsr A, DevAcsr AT, const T *__restrict__ X, T *__restrict__ Y, int BH)
{
    const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (i >= A.n) return;
    int4 g[4];
    const int ns = A.nseg[i];
#pragma unroll
    for (int s = 0; s < 4; ++s) g[s] = A.seg[(size_t)i * 4 + s];
    const long long rb = A.row_ptr[i];
    const int len = (int)(A.row_ptr[i + 1] - rb);
    for (int x = lane; x < len; x += 32) {
        const int j = col_at(g, ns, x);
        int4 h[4];
        const int nt = AT.nseg[j];
#pragma unroll
        for (int s = 0; s < 4; ++s) h[s] = AT.seg[(size_t)j * 4 + s];
        const long long dst = AT.row_ptr[j] + rank_of(h, nt, i);   // i is a row of column j: rank >= 0
        const long long src = rb + x;
        for (int bh = 0; bh < BH; ++bh) Y[(size_t)bh * AT.nnz + dst] = X[(size_t)bh * A.nnz + src];
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
rspmm_cc_kernel(DevAcsr A, DevAcsr AT, const T *__restrict__ PT, const T *__restrict__ V, int d, T *__restrict__ O,
                int align_x)
{
    const int n_rt = (A.n + 31) / 32;
    const int bh = blockIdx.x / n_rt, i0 = (blockIdx.x % n_rt) * 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // align_x > 1 (diagnostics build, the Fig. 14 ablation): lanes take rows along the stride
    // lattice of STRIDED(align_x) -- row r' of the residue-major order is (r' mod nk) X + r' div nk
    // -- so every lane of a warp is a row of the same column residue (the paper's
    // linear-transformation alignment); 0: natural consecutive rows
    int i = i0 + lane;
    if (align_x > 1 && i < A.n) {
        const int nk = A.n / align_x;
        i = (i % nk) * align_x + i / nk;
    }
    // span of the 32 rows' columns
    int jlo = 0x7fffffff, jhi = -1;
    if (i < A.n) {
        const int ns = A.nseg[i];
        for (int s = 0; s < ns; ++s) {
            const int4 g = A.seg[(size_t)i * 4 + s];
            if (g.z > 0) {
                jlo = min(jlo, g.x);
                jhi = max(jhi, g.x + g.y * (g.z - 1));
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        jlo = min(jlo, __shfl_xor_sync(0xffffffffu, jlo, o));
        jhi = max(jhi, __shfl_xor_sync(0xffffffffu, jhi, o));
    }
    const T *Vb = V + (size_t)bh * A.n * d;
    const T *Pb = PT + (size_t)bh * AT.nnz;
    const int t0 = 32 * w;
    float acc[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) acc[t] = 0.f;
    for (int j = jlo; j <= jhi; ++j) {
        int4 h[4];
        const int nt = AT.nseg[j];
#pragma unroll
        for (int s = 0; s < 4; ++s) h[s] = AT.seg[(size_t)j * 4 + s];
        const int rk = i < A.n ? rank_of(h, nt, i) : -1;
        if (!__any_sync(0xffffffffu, rk >= 0)) continue;
        const float p = rk >= 0 ? ld_f(Pb + AT.row_ptr[j] + rk) : 0.f;
        const float vj = t0 + lane < d ? ld_f(Vb + (size_t)j * d + t0 + lane) : 0.f;
#pragma unroll
        for (int t = 0; t < 32; ++t) acc[t] = fmaf(p, __shfl_sync(0xffffffffu, vj, t), acc[t]);
    }
    if (i < A.n) {
        T *o = O + ((size_t)bh * A.n + i) * d + t0;
#pragma unroll
        for (int t = 0; t < 32; ++t)
            if (t0 + t < d) st_f(o + t, acc[t]);
    }
}

}  // namespace

cudaError_t launch_transpose_values(const DevAcsr &A, const DevAcsr &AT, const void *X, void *Y, bool bf16, int BH,
                                    cudaStream_t st)
{
    const dim3 grid((unsigned)((A.n + 7) / 8));
    if (bf16)
        transpose_values_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(A, AT, (const __nv_bfloat16 *)X, (__nv_bfloat16 *)Y, BH);
    else
        transpose_values_kernel<float><<<grid, 256, 0, st>>>(A, AT, (const float *)X, (float *)Y, BH);
    return cudaGetLastError();
}

cudaError_t launch_rspmm_cc(const DevAcsr &A, const DevAcsr &AT, const void *PT, const void *V, bool bf16, int BH,
                            int d, void *O, cudaStream_t st, int align_x)
{
    const int n_rt = (A.n + 31) / 32;
    const dim3 grid((unsigned)(BH * n_rt));
    const int threads = 32 * ((d + 31) / 32);
    if (bf16)
        rspmm_cc_kernel<__nv_bfloat16><<<grid, threads, 0, st>>>(A, AT, (const __nv_bfloat16 *)PT,
                                                                 (const __nv_bfloat16 *)V, d, (__nv_bfloat16 *)O, align_x);
    else
        rspmm_cc_kernel<float><<<grid, threads, 0, st>>>(A, AT, (const float *)PT, (const float *)V, d, (float *)O, align_x);
    return cudaGetLastError();
}

}  // namespace splat
