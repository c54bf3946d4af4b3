// simt.cu -- SIMT kernels: the fp32 path of every primitive (PAPER precision,
// FP32 FFMA; no TF32 so the 1e-5 bound holds) and the sparse row
// softmax for both dtypes.  One warp per (b, h, row).
//
//   R-SDDMM: S[row_ptr[i]+x] = scale * <q_i, k_{c_x(i)}>
//   softmax: per-row max, exp, sum, normalise
//   R-SpMM: o_i = sum_x P[row_ptr[i]+x] v_{c_x(i)}
//   fused    (Eq. 1): the three above with an online softmax, S/P in registers
//
// Column of the x-th non-zero of row i: the run s with off_s <= x < off_s +
// count_s gives c = start_s + step_s * (x - off_s)  (the paper's
// (sparse_i - b)/a).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace splat {
namespace {

constexpr int kWarps = 8;   // rows per CTA

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

struct RowId {
    int bh, i;
};

__device__ __forceinline__ RowId row_of_warp(int n)
{
    const int nrb = (n + kWarps - 1) / kWarps;
    const int rb = blockIdx.x;
    return {rb / nrb, (rb % nrb) * kWarps + (int)(threadIdx.x >> 5)};
}

__device__ __forceinline__ int col_of(const int4 *g, int ns, int x)
{
    int c = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s)
        if (s < ns && x >= g[s].w && x < g[s].w + g[s].z) c = g[s].x + g[s].y * (x - g[s].w);
    return c;
}

template <typename T>
__global__ void __launch_bounds__(kWarps * 32)
rsddmm_simt_kernel(DevAcsr A, const T *__restrict__ Q, const T *__restrict__ K, int d, float scale,
                   float *__restrict__ S)
{
    extern __shared__ float qs[];
    const RowId r = row_of_warp(A.n);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (r.i >= A.n) return;
    float *qw = qs + w * d;
    const T *q = Q + ((size_t)r.bh * A.n + r.i) * d;
    for (int t = lane; t < d; t += 32) qw[t] = to_f(q[t]);
    __syncwarp();
    const T *Kb = K + (size_t)r.bh * A.n * d;
    float *Sb = S + (size_t)r.bh * A.nnz + A.row_ptr[r.i];
    const int ns = A.nseg[r.i];
    for (int s = 0; s < ns; ++s) {
        const int4 g = A.seg[(size_t)r.i * 4 + s];
        for (int x = lane; x < g.z; x += 32) {
            const T *kr = Kb + (size_t)(g.x + g.y * x) * d;
            float acc = 0.f;
            for (int t = 0; t < d; ++t) acc = fmaf(qw[t], to_f(kr[t]), acc);
            Sb[g.w + x] = scale * acc;
        }
    }
}

template <typename TP>
__global__ void __launch_bounds__(kWarps * 32)
softmax_kernel(DevAcsr A, const float *__restrict__ S, TP *__restrict__ P)
{
    const RowId r = row_of_warp(A.n);
    const int lane = threadIdx.x & 31;
    if (r.i >= A.n) return;
    const long long b = A.row_ptr[r.i], len = A.row_ptr[r.i + 1] - b;
    if (len <= 0) return;
    const float *s = S + (size_t)r.bh * A.nnz + b;
    TP *p = P + (size_t)r.bh * A.nnz + b;
    float m = -INFINITY, l = 0.f;
    for (long long x = lane; x < len; x += 32) {
        const float v = s[x];
        const float mn = fmaxf(m, v);
        l = l * expf(m - mn) + expf(v - mn);
        m = mn;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o), l2 = __shfl_xor_sync(0xffffffffu, l, o);
        const float mn = fmaxf(m, m2);
        l = (m == -INFINITY ? 0.f : l * expf(m - mn)) + (m2 == -INFINITY ? 0.f : l2 * expf(m2 - mn));
        m = mn;
    }
    const float inv = 1.f / l;
    for (long long x = lane; x < len; x += 32) p[x] = from_f<TP>(expf(s[x] - m) * inv);
}

template <typename T>
__global__ void __launch_bounds__(kWarps * 32)
rspmm_simt_kernel(DevAcsr A, const T *__restrict__ P, const T *__restrict__ V, int d, T *__restrict__ O)
{
    const RowId r = row_of_warp(A.n);
    const int lane = threadIdx.x & 31;
    if (r.i >= A.n) return;
    float acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.f;
    const T *Pb = P + (size_t)r.bh * A.nnz + A.row_ptr[r.i];
    const T *Vb = V + (size_t)r.bh * A.n * d;
    const int ns = A.nseg[r.i];
    for (int s = 0; s < ns; ++s) {
        const int4 g = A.seg[(size_t)r.i * 4 + s];
        for (int x0 = 0; x0 < g.z; x0 += 32) {
            const int x = x0 + lane;
            const float pl = x < g.z ? to_f(Pb[g.w + x]) : 0.f;
            const int cnt = min(32, g.z - x0);
            for (int j = 0; j < cnt; ++j) {
                const float pj = __shfl_sync(0xffffffffu, pl, j);
                const T *vr = Vb + (size_t)(g.x + g.y * (x0 + j)) * d;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int t = lane + 32 * u;
                    if (t < d) acc[u] = fmaf(pj, to_f(vr[t]), acc[u]);
                }
            }
        }
    }
    T *o = O + ((size_t)r.bh * A.n + r.i) * d;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int t = lane + 32 * u;
        if (t < d) o[t] = from_f<T>(acc[u]);
    }
}

template <typename T>
__global__ void __launch_bounds__(kWarps * 32)
mhsa_simt_kernel(DevAcsr A, const T *__restrict__ Q, const T *__restrict__ K, const T *__restrict__ V,
                 int d, float scale, T *__restrict__ O)
{
    extern __shared__ float qs[];
    const RowId r = row_of_warp(A.n);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (r.i >= A.n) return;
    float *qw = qs + w * d;
    const T *q = Q + ((size_t)r.bh * A.n + r.i) * d;
    for (int t = lane; t < d; t += 32) qw[t] = to_f(q[t]);
    __syncwarp();
    int4 g[4];
    const int ns = A.nseg[r.i];
#pragma unroll
    for (int s = 0; s < 4; ++s) g[s] = A.seg[(size_t)r.i * 4 + s];
    const int len = (int)(A.row_ptr[r.i + 1] - A.row_ptr[r.i]);
    const T *Kb = K + (size_t)r.bh * A.n * d;
    const T *Vb = V + (size_t)r.bh * A.n * d;
    float m = -INFINITY, l = 0.f, acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.f;
    for (int e0 = 0; e0 < len; e0 += 32) {
        const int e = e0 + lane;
        const bool valid = e < len;
        const int col = valid ? col_of(g, ns, e) : 0;
        float s = -INFINITY;
        if (valid) {
            const T *kr = Kb + (size_t)col * d;
            float a = 0.f;
            for (int t = 0; t < d; ++t) a = fmaf(qw[t], to_f(kr[t]), a);
            s = scale * a;
        }
        float cm = s;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
        const float mn = fmaxf(m, cm);
        const float alpha = expf(m - mn);   // m = -inf on the first chunk -> 0
        const float p = valid ? expf(s - mn) : 0.f;
        float ps = p;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
        l = l * alpha + ps;
        m = mn;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] *= alpha;
        const int cnt = min(32, len - e0);
        for (int j = 0; j < cnt; ++j) {
            const float pj = __shfl_sync(0xffffffffu, p, j);
            const int cj = __shfl_sync(0xffffffffu, col, j);
            const T *vr = Vb + (size_t)cj * d;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = lane + 32 * u;
                if (t < d) acc[u] = fmaf(pj, to_f(vr[t]), acc[u]);
            }
        }
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    T *o = O + ((size_t)r.bh * A.n + r.i) * d;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int t = lane + 32 * u;
        if (t < d) o[t] = from_f<T>(acc[u] * inv);
    }
}

inline dim3 grid_rows(const DevAcsr &A, int BH)
{
    return dim3((unsigned)(BH * ((A.n + kWarps - 1) / kWarps)));
}

}  // namespace

cudaError_t launch_rsddmm_simt(const DevAcsr &A, const void *Q, const void *K, bool bf16, int BH, int d,
                               float scale, float *S, cudaStream_t st)
{
    const size_t sm = (size_t)kWarps * d * sizeof(float);
    if (bf16)
        rsddmm_simt_kernel<__nv_bfloat16><<<grid_rows(A, BH), kWarps * 32, sm, st>>>(
            A, (const __nv_bfloat16 *)Q, (const __nv_bfloat16 *)K, d, scale, S);
    else
        rsddmm_simt_kernel<float><<<grid_rows(A, BH), kWarps * 32, sm, st>>>(A, (const float *)Q,
                                                                              (const float *)K, d, scale, S);
    return cudaGetLastError();
}

cudaError_t launch_softmax(const DevAcsr &A, const float *S, void *P, bool p_bf16, int BH, cudaStream_t st)
{
    if (p_bf16)
        softmax_kernel<__nv_bfloat16><<<grid_rows(A, BH), kWarps * 32, 0, st>>>(A, S, (__nv_bfloat16 *)P);
    else
        softmax_kernel<float><<<grid_rows(A, BH), kWarps * 32, 0, st>>>(A, S, (float *)P);
    return cudaGetLastError();
}

cudaError_t launch_rspmm_simt(const DevAcsr &A, const void *P, const void *V, bool bf16, int BH, int d,
                              void *O, cudaStream_t st)
{
    if (bf16)
        rspmm_simt_kernel<__nv_bfloat16><<<grid_rows(A, BH), kWarps * 32, 0, st>>>(
            A, (const __nv_bfloat16 *)P, (const __nv_bfloat16 *)V, d, (__nv_bfloat16 *)O);
    else
        rspmm_simt_kernel<float><<<grid_rows(A, BH), kWarps * 32, 0, st>>>(A, (const float *)P,
                                                                            (const float *)V, d, (float *)O);
    return cudaGetLastError();
}

cudaError_t launch_mhsa_simt(const DevAcsr &A, const void *Q, const void *K, const void *V, bool bf16,
                             int BH, int d, float scale, void *O, cudaStream_t st)
{
    const size_t sm = (size_t)kWarps * d * sizeof(float);
    if (bf16)
        mhsa_simt_kernel<__nv_bfloat16><<<grid_rows(A, BH), kWarps * 32, sm, st>>>(
            A, (const __nv_bfloat16 *)Q, (const __nv_bfloat16 *)K, (const __nv_bfloat16 *)V, d, scale,
            (__nv_bfloat16 *)O);
    else
        mhsa_simt_kernel<float><<<grid_rows(A, BH), kWarps * 32, sm, st>>>(
            A, (const float *)Q, (const float *)K, (const float *)V, d, scale, (float *)O);
    return cudaGetLastError();
}

}  // namespace splat
