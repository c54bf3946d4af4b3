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

template <int W = kWarps>
__device__ __forceinline__ RowId row_of_warp(int n)
{
    const int nrb = (n + W - 1) / W;
    const int rb = blockIdx.x;
    return {rb / nrb, (rb % nrb) * W + (int)(threadIdx.x >> 5)};
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

// 4 consecutive P values from 4 probabilities: one 8-byte (bf16) or 16-byte (fp32) store
__device__ __forceinline__ void store4(__nv_bfloat16 *p, float a, float b, float c, float d)
{
    uint2 w;
    w.x = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a)) | ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b)) << 16);
    w.y = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(c)) | ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(d)) << 16);
    *reinterpret_cast<uint2 *>(p) = w;
}
__device__ __forceinline__ void store4(float *p, float a, float b, float c, float d)
{
    *reinterpret_cast<float4 *>(p) = make_float4(a, b, c, d);
}

__device__ __forceinline__ float ex2f(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Short rows (mean row length <= 256): the same three passes with LPR = 8 (mean <= 64) or 16 lanes
// per row and 32 / LPR rows per warp, so that a warp has several rows' loads in flight (a warp per row leaves the launch latency-bound: at
// N = 1024 and 0.4 % density it takes ~14 waves of ~4 dependent memory trips each).  No early
// exit: every lane reaches the shuffles; lanes of rows past the end just have no work.
template <typename TP, int LPR>
__global__ void __launch_bounds__(kWarps * 32)
softmax_short_kernel(DevAcsr A, const float *__restrict__ S, TP *__restrict__ P, int BH)
{
    constexpr float L2E = 1.4426950408889634f;
    const int lane = threadIdx.x & 31, sl = lane & (LPR - 1);
    const long long g = ((long long)blockIdx.x * kWarps + (threadIdx.x >> 5)) * (32 / LPR) + lane / LPR;
    const bool ok = g < (long long)BH * A.n;
    const int bh = ok ? (int)(g / A.n) : 0, i = ok ? (int)(g % A.n) : 0;
    const long long b = A.row_ptr[i];
    const int len = ok ? (int)(A.row_ptr[i + 1] - b) : 0;
    const long long e0 = (long long)bh * A.nnz + b;
    const float *s = S + e0;
    TP *p = P + e0;
    float m = -INFINITY, l = 0.f;
    // rows of at most 16 LPR elements (every row of the group, a warp-uniform test): held in
    // registers, S read once (streaming), one exponential per element
    constexpr int CAP = 16;
    const bool fits = __all_sync(0xffffffffu, len <= CAP * LPR);
    if (fits) {
        float v[CAP];
#pragma unroll
        for (int k = 0; k < CAP; ++k) {
            const int x = sl + LPR * k;
            v[k] = x < len ? __ldcs(s + x) : -INFINITY;
        }
#pragma unroll
        for (int k = 0; k < CAP; ++k) m = fmaxf(m, v[k]);
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const float mL = m * L2E;
#pragma unroll
        for (int k = 0; k < CAP; ++k) {
            v[k] = sl + LPR * k < len ? ex2f(fmaf(v[k], L2E, -mL)) : 0.f;
            l += v[k];
        }
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        const float inv = 1.f / l;
#pragma unroll
        for (int k = 0; k < CAP; ++k) {
            const int x = sl + LPR * k;
            if (x < len) p[x] = from_f<TP>(v[k] * inv);
        }
        return;
    }
    for (int x = sl; x < len; x += LPR) m = fmaxf(m, s[x]);
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float mL = m * L2E;
    for (int x = sl; x < len; x += LPR) l += ex2f(fmaf(s[x], L2E, -mL));
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    const float inv = 1.f / l;
    for (int x = sl; x < len; x += LPR) p[x] = from_f<TP>(ex2f(fmaf(s[x], L2E, -mL)) * inv);
}

// Three streaming passes over one ACSR row (max, sum of exp, write) by one warp; rows over 2048
// elements fold max and sum into one online pass.
template <typename TP>
__device__ __forceinline__ void softmax_row_passes(const float *__restrict__ s, TP *__restrict__ p, int len, int head,
                                                   int nv, int tail0, int lane)
{
    constexpr float L2E = 1.4426950408889634f;
    const float4 *s4 = reinterpret_cast<const float4 *>(s + head);
    float m = -INFINITY, l = 0.f;
    if (len > 2048) {
        // long rows (their re-reads would miss L2): one online pass for max and sum
        // (the sum is rescaled when the running max grows), then the write pass
        auto add = [&](float vmax, float s0) {   // s0 = sum of 2^((v - vmax) log2 e) of the group
            const float mn = fmaxf(m, vmax);
            l = l * ex2f((m - mn) * L2E) + s0 * ex2f((vmax - mn) * L2E);
            m = mn;
        };
        if (lane < head) add(s[lane], 1.f);
#pragma unroll 4
        for (int q = lane; q < nv; q += 32) {
            const float4 v = s4[q];
            const float vm = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)), vmL = vm * L2E;
            add(vm, (ex2f(fmaf(v.x, L2E, -vmL)) + ex2f(fmaf(v.y, L2E, -vmL))) +
                        (ex2f(fmaf(v.z, L2E, -vmL)) + ex2f(fmaf(v.w, L2E, -vmL))));
        }
        for (int x = tail0 + lane; x < len; x += 32) add(s[x], 1.f);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, o), l2 = __shfl_xor_sync(0xffffffffu, l, o);
            const float mn = fmaxf(m, m2);
            l = (m == -INFINITY ? 0.f : l * ex2f((m - mn) * L2E)) + (m2 == -INFINITY ? 0.f : l2 * ex2f((m2 - mn) * L2E));
            m = mn;
        }
    } else {
        if (lane < head) m = s[lane];
#pragma unroll 4
        for (int q = lane; q < nv; q += 32) {
            const float4 v = s4[q];
            m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        }
        for (int x = tail0 + lane; x < len; x += 32) m = fmaxf(m, s[x]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const float mL0 = m * L2E;
        if (lane < head) l = ex2f(fmaf(s[lane], L2E, -mL0));
#pragma unroll 4
        for (int q = lane; q < nv; q += 32) {
            const float4 v = s4[q];
            l += (ex2f(fmaf(v.x, L2E, -mL0)) + ex2f(fmaf(v.y, L2E, -mL0))) + (ex2f(fmaf(v.z, L2E, -mL0)) + ex2f(fmaf(v.w, L2E, -mL0)));
        }
        for (int x = tail0 + lane; x < len; x += 32) l += ex2f(fmaf(s[x], L2E, -mL0));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    }
    const float mL = m * L2E;
    const float inv = 1.f / l;
    if (lane < head) p[lane] = from_f<TP>(ex2f(fmaf(s[lane], L2E, -mL)) * inv);
    TP *p4 = p + head;
#pragma unroll 4
    for (int q = lane; q < nv; q += 32) {
        const float4 v = s4[q];
        store4(p4 + 4 * q, ex2f(fmaf(v.x, L2E, -mL)) * inv, ex2f(fmaf(v.y, L2E, -mL)) * inv,
               ex2f(fmaf(v.z, L2E, -mL)) * inv, ex2f(fmaf(v.w, L2E, -mL)) * inv);
    }
    for (int x = tail0 + lane; x < len; x += 32) p[x] = from_f<TP>(ex2f(fmaf(s[x], L2E, -mL)) * inv);
}

// Row softmax over the ACSR row (the softmax of each input row of the ACSR, which
// stores only the non-zeros; reading R-1).  Warp per row, three streaming passes over the row --
// max, sum of exp, write -- with 16-byte loads of S on the aligned body of the row (the second and
// third reads hit L2); exp(x - m) = 2^((x - m) log2 e) on MUFU.EX2.
//
// RC > 0: rows of at most 128 RC elements are held in registers (RC float4 per lane, all loads
// issued at once, streaming / evict-first: S is read exactly once) and take one exponential per
// element; longer rows take the three passes.
template <typename TP, int RC>
__global__ void __launch_bounds__(kWarps * 32)
softmax_kernel(DevAcsr A, const float *__restrict__ S, TP *__restrict__ P)
{
    const RowId r = row_of_warp(A.n);
    const int lane = threadIdx.x & 31;
    if (r.i >= A.n) return;
    const long long b = A.row_ptr[r.i];
    const int len = (int)(A.row_ptr[r.i + 1] - b);
    if (len <= 0) return;
    const long long e0 = (long long)r.bh * A.nnz + b;       // element index of the row start
    const float *s = S + e0;
    TP *p = P + e0;
    const int head = min(len, (int)((4 - (e0 & 3)) & 3));  // elements before the first 16-byte boundary
    const int nv = (len - head) >> 2;                        // aligned float4 groups
    const int tail0 = head + 4 * nv;
    const float4 *s4 = reinterpret_cast<const float4 *>(s + head);
    constexpr float L2E = 1.4426950408889634f;
    float m = -INFINITY, l = 0.f;
    if (RC > 0 && len <= 128 * RC) {
        constexpr int R = RC > 0 ? RC : 1;
        float4 v[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int q = lane + 32 * k;
            v[k] = q < nv ? __ldcs(s4 + q) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        }
        // head (< 4 elements before the first 16-byte boundary) and tail (< 4 after the last)
        const int xt = tail0 + lane;
        float hv = lane < head ? __ldcs(s + lane) : -INFINITY;
        float tv = xt < len ? __ldcs(s + xt) : -INFINITY;
        m = fmaxf(hv, tv);
        const int kmax = (nv + 31) >> 5;                   // float4 groups holding row data (warp-uniform)
#pragma unroll
        for (int k = 0; k < R; ++k)
            if (k < kmax) m = fmaxf(m, fmaxf(fmaxf(v[k].x, v[k].y), fmaxf(v[k].z, v[k].w)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const float mL = m * L2E;
        // masked-out slots hold -inf: 2^(-inf) = 0 adds nothing
        hv = ex2f(fmaf(hv, L2E, -mL));
        tv = ex2f(fmaf(tv, L2E, -mL));
        l = hv + tv;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            if (k < kmax) {                                 // no exponentials of the padding groups
                v[k].x = ex2f(fmaf(v[k].x, L2E, -mL));
                v[k].y = ex2f(fmaf(v[k].y, L2E, -mL));
                v[k].z = ex2f(fmaf(v[k].z, L2E, -mL));
                v[k].w = ex2f(fmaf(v[k].w, L2E, -mL));
                l += (v[k].x + v[k].y) + (v[k].z + v[k].w);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        const float inv = 1.f / l;
        if (lane < head) p[lane] = from_f<TP>(hv * inv);
        if (xt < len) p[xt] = from_f<TP>(tv * inv);
        TP *p4 = p + head;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int q = lane + 32 * k;
            if (q < nv) store4(p4 + 4 * q, v[k].x * inv, v[k].y * inv, v[k].z * inv, v[k].w * inv);
        }
        return;
    }
    softmax_row_passes(s, p, len, head, nv, tail0, lane);
}

// <q, k> for one key row: 16-byte loads and four independent FMA chains when d % 4 == 0 and the
// row is 16-byte aligned (fp32), else the plain loop (the order of the partial sums differs from
// a single chain by rounding only; the fp32 tolerance is 1e-5 max-abs, SURVEY C-5)
__device__ __forceinline__ float dot_row(const float *qw, const float *kr, int d)
{
    if ((d & 3) == 0 && ((reinterpret_cast<uintptr_t>(kr) & 15) == 0)) {
        const float4 *k4 = reinterpret_cast<const float4 *>(kr);
        const float4 *q4 = reinterpret_cast<const float4 *>(qw);
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 16
        for (int t = 0; t < d / 4; ++t) {
            const float4 k = __ldg(k4 + t), q = q4[t];
            a0 = fmaf(q.x, k.x, a0);
            a1 = fmaf(q.y, k.y, a1);
            a2 = fmaf(q.z, k.z, a2);
            a3 = fmaf(q.w, k.w, a3);
        }
        return (a0 + a1) + (a2 + a3);
    }
    float a = 0.f;
    for (int t = 0; t < d; ++t) a = fmaf(qw[t], kr[t], a);
    return a;
}
__device__ __forceinline__ float dot_row(const float *qw, const __nv_bfloat16 *kr, int d)
{
    float a0 = 0.f, a1 = 0.f;
    int t = 0;
    for (; t + 1 < d; t += 2) {
        a0 = fmaf(qw[t], to_f(kr[t]), a0);
        a1 = fmaf(qw[t + 1], to_f(kr[t + 1]), a1);
    }
    if (t < d) a0 = fmaf(qw[t], to_f(kr[t]), a0);
    return a0 + a1;
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

// Fused fp32 / SIMT path: one warp per (b, h, row), W warps (rows) per CTA.  Per 32-key chunk: lane x
// computes <q, k_x> (q staged in shared memory), warp-shuffle max / sum (online softmax), then
// O += p V over the chunk with the V rows of 4 keys loaded before their FMAs (4 loads in flight
// per lane instead of one dependent load per key).
template <typename T, int W>
__global__ void __launch_bounds__(W * 32)
mhsa_simt_kernel(DevAcsr A, const T *__restrict__ Q, const T *__restrict__ K, const T *__restrict__ V,
                 int d, float scale, T *__restrict__ O)
{
    extern __shared__ float qs[];
    const RowId r = row_of_warp<W>(A.n);
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
    const int nu = (d + 31) >> 5;          // output columns per lane: lane + 32 u, u < nu <= 8
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
            s = scale * dot_row(qw, kr, d);
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
        for (int j0 = 0; j0 < cnt; j0 += 4) {
            float pj[4], vv[4][8];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int j = min(j0 + jj, 31);
                pj[jj] = __shfl_sync(0xffffffffu, p, j);
                const int cj = __shfl_sync(0xffffffffu, col, j);
                if (j0 + jj >= cnt) pj[jj] = 0.f;            // p of an invalid lane is 0 already
                const T *vr = Vb + (size_t)cj * d;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int t = lane + 32 * u;
                    vv[jj][u] = (u < nu && t < d) ? to_f(vr[t]) : 0.f;
                }
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[u] = fmaf(pj[jj], vv[jj][u], acc[u]);
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

// Small problems (fewer than 8 rows per SM, e.g. the tiny config's 256 rows): one CTA of 128
// threads per (b, h, row), so the row's memory trips are few and wide instead of one warp walking
// its keys.  Per chunk of 128 keys: thread j computes s_j = scale <q, k_{c_j}> (q in shared
// memory, the K row read with all loads in flight), block max / sum (online softmax over chunks);
// then thread t accumulates O[t] (and O[t + 128]) over the chunk's keys, V rows coalesced across
// threads.  fp32 arithmetic throughout (the paper's FP32).
constexpr int kRowThreads = 128;

template <typename T>
__device__ __forceinline__ float dot_full(const float *q, const T *__restrict__ k, int d);

// fp32 rows: 16-byte loads when d % 4 == 0 (rows are then 16-byte aligned)
template <>
__device__ __forceinline__ float dot_full<float>(const float *q, const float *__restrict__ k, int d)
{
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    if ((d & 3) == 0) {
        const float4 *k4 = reinterpret_cast<const float4 *>(k);
#pragma unroll 8
        for (int t = 0; t < d / 4; ++t) {
            const float4 kv = __ldg(k4 + t);
            a0 = fmaf(q[4 * t], kv.x, a0);
            a1 = fmaf(q[4 * t + 1], kv.y, a1);
            a2 = fmaf(q[4 * t + 2], kv.z, a2);
            a3 = fmaf(q[4 * t + 3], kv.w, a3);
        }
        return (a0 + a1) + (a2 + a3);
    }
    for (int t = 0; t < d; ++t) a0 = fmaf(q[t], k[t], a0);
    return a0;
}

template <typename T>
__device__ __forceinline__ float dot_full(const float *q, const T *__restrict__ k, int d)
{
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int t = 0;
    for (; t + 4 <= d; t += 4) {
        a0 = fmaf(q[t], to_f(k[t]), a0);
        a1 = fmaf(q[t + 1], to_f(k[t + 1]), a1);
        a2 = fmaf(q[t + 2], to_f(k[t + 2]), a2);
        a3 = fmaf(q[t + 3], to_f(k[t + 3]), a3);
    }
    for (; t < d; ++t) a0 = fmaf(q[t], to_f(k[t]), a0);
    return (a0 + a1) + (a2 + a3);
}

template <typename T>
__global__ void __launch_bounds__(kRowThreads)
mhsa_simt_row_kernel(DevAcsr A, const T *__restrict__ Q, const T *__restrict__ K, const T *__restrict__ V, int d,
                     float scale, T *__restrict__ O)
{
    __shared__ float qsh[256];
    __shared__ float psh[kRowThreads];
    __shared__ int csh[kRowThreads];
    __shared__ float rmax[kRowThreads / 32], rsum[kRowThreads / 32];
    const int bh = blockIdx.x / A.n, i = blockIdx.x % A.n;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const T *q = Q + ((size_t)bh * A.n + i) * d;
    for (int t = tid; t < d; t += kRowThreads) qsh[t] = to_f(q[t]);
    int4 g[4];
    int ns, len;
    if (A.has_pat) {
        // the row's runs in closed form from the descriptor (the affine indices of P:216-219):
        // no dependent metadata load before the K rows are fetched
        Seg sg[4];
        ns = row_segments(A.pat, i, sg);
        len = 0;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            g[s] = s < ns ? make_int4(sg[s].start, sg[s].step, sg[s].count, len) : make_int4(0, 1, 0, len);
            if (s < ns) len += sg[s].count;
        }
    } else {
        ns = A.nseg[i];
#pragma unroll
        for (int s = 0; s < 4; ++s) g[s] = A.seg[(size_t)i * 4 + s];
        len = (int)(A.row_ptr[i + 1] - A.row_ptr[i]);
    }
    const T *Kb = K + (size_t)bh * A.n * d;
    const T *Vb = V + (size_t)bh * A.n * d;
    __syncthreads();
    float m = -INFINITY, l = 0.f, acc0 = 0.f, acc1 = 0.f;
    for (int e0 = 0; e0 < len; e0 += kRowThreads) {
        const int e = e0 + tid;
        const bool valid = e < len;
        const int col = valid ? col_of(g, ns, e) : 0;
        if (valid) {
            // the key's V row into L2 now: the accumulation below then reads it from L2, not HBM
            const char *vrow = reinterpret_cast<const char *>(Vb + (size_t)col * d);
            for (int b = 0; b < d * (int)sizeof(T); b += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(vrow + b));
        }
        const float s = valid ? scale * dot_full(qsh, Kb + (size_t)col * d, d) : -INFINITY;
        float cm = s;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
        if (lane == 0) rmax[w] = cm;
        __syncthreads();
        cm = fmaxf(fmaxf(rmax[0], rmax[1]), fmaxf(rmax[2], rmax[3]));
        const float mn = fmaxf(m, cm);
        const float alpha = expf(m - mn);   // m = -inf on the first chunk -> 0
        const float p = valid ? expf(s - mn) : 0.f;
        psh[tid] = p;
        csh[tid] = col;
        float ps = p;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
        if (lane == 0) rsum[w] = ps;
        __syncthreads();
        l = l * alpha + ((rsum[0] + rsum[1]) + (rsum[2] + rsum[3]));
        m = mn;
        acc0 *= alpha;
        acc1 *= alpha;
        const int cnt = min(kRowThreads, len - e0);
        if (d <= kRowThreads / 2) {
            // two key groups (even / odd keys) over the same output column: twice the loads in flight
            const int t = tid & (kRowThreads / 2 - 1), grp = tid / (kRowThreads / 2);
            if (t < d) {
#pragma unroll 16
                for (int j = grp; j < cnt; j += 2) acc0 = fmaf(psh[j], to_f(Vb[(size_t)csh[j] * d + t]), acc0);
            }
        } else if (tid < d) {
            const bool two = tid + kRowThreads < d;
#pragma unroll 8
            for (int j = 0; j < cnt; ++j) {
                const T *vr = Vb + (size_t)csh[j] * d;
                acc0 = fmaf(psh[j], to_f(vr[tid]), acc0);
                if (two) acc1 = fmaf(psh[j], to_f(vr[tid + kRowThreads]), acc1);
            }
        }
        __syncthreads();     // psh / csh / rmax / rsum are rewritten by the next chunk
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    T *o = O + ((size_t)bh * A.n + i) * d;
    if (d <= kRowThreads / 2) {
        // the odd-key group's partial sums join the even group's (fixed order: deterministic)
        if (tid >= kRowThreads / 2) psh[tid - kRowThreads / 2] = acc0;
        __syncthreads();
        if (tid < d) o[tid] = from_f<T>((acc0 + psh[tid]) * inv);
        return;
    }
    if (tid < d) o[tid] = from_f<T>(acc0 * inv);
    if (tid + kRowThreads < d) o[tid + kRowThreads] = from_f<T>(acc1 * inv);
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
    if (A.nnz <= 256ll * A.n) {
        const bool r8 = A.nnz <= 64ll * A.n;
        const long long rows = (long long)BH * A.n, per_cta = kWarps * (r8 ? 4 : 2);
        const unsigned grid = (unsigned)((rows + per_cta - 1) / per_cta);
        if (p_bf16 && r8)
            softmax_short_kernel<__nv_bfloat16, 8><<<grid, kWarps * 32, 0, st>>>(A, S, (__nv_bfloat16 *)P, BH);
        else if (p_bf16)
            softmax_short_kernel<__nv_bfloat16, 16><<<grid, kWarps * 32, 0, st>>>(A, S, (__nv_bfloat16 *)P, BH);
        else if (r8)
            softmax_short_kernel<float, 8><<<grid, kWarps * 32, 0, st>>>(A, S, (float *)P, BH);
        else
            softmax_short_kernel<float, 16><<<grid, kWarps * 32, 0, st>>>(A, S, (float *)P, BH);
        return cudaGetLastError();
    }
    // register capacity by the mean row length: Longformer / BigBird rows (~440-560) fit 8 float4
    // per lane, a 4096-key window 32; the rare longer rows (global rows) take the three passes
    const int knob = diag_env("SPLAT_SOFTMAX_RC");      // diagnostics build: 1 = three passes only
    const int rc = knob == 1 ? 0 : A.nnz <= 640ll * A.n ? 8 : A.nnz <= 4096ll * A.n ? 32 : 0;
    const dim3 grid = grid_rows(A, BH);
#define SPLAT_SOFTMAX_LAUNCH(RC)                                                                         \
    do {                                                                                               \
        if (p_bf16) softmax_kernel<__nv_bfloat16, RC><<<grid, kWarps * 32, 0, st>>>(A, S, (__nv_bfloat16 *)P); \
        else softmax_kernel<float, RC><<<grid, kWarps * 32, 0, st>>>(A, S, (float *)P);                \
    } while (0)
    if (rc == 8) SPLAT_SOFTMAX_LAUNCH(8);
    else if (rc == 32) SPLAT_SOFTMAX_LAUNCH(32);
    else SPLAT_SOFTMAX_LAUNCH(0);
#undef SPLAT_SOFTMAX_LAUNCH
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
    // few rows (fewer than 8 per SM): one CTA per row so every SM gets work and each row's memory
    // trips are few and wide
    if ((long long)BH * A.n <= 148ll * 8 && d <= 256) {
        const dim3 grid((unsigned)(BH * A.n));
        if (bf16)
            mhsa_simt_row_kernel<__nv_bfloat16><<<grid, kRowThreads, 0, st>>>(A, (const __nv_bfloat16 *)Q,
                (const __nv_bfloat16 *)K, (const __nv_bfloat16 *)V, d, scale, (__nv_bfloat16 *)O);
        else
            mhsa_simt_row_kernel<float><<<grid, kRowThreads, 0, st>>>(A, (const float *)Q, (const float *)K,
                                                                      (const float *)V, d, scale, (float *)O);
        return cudaGetLastError();
    }
    const size_t sm = (size_t)kWarps * d * sizeof(float);
    const dim3 grid((unsigned)(BH * ((A.n + kWarps - 1) / kWarps)));
    if (bf16)
        mhsa_simt_kernel<__nv_bfloat16, kWarps><<<grid, kWarps * 32, sm, st>>>(A, (const __nv_bfloat16 *)Q,
            (const __nv_bfloat16 *)K, (const __nv_bfloat16 *)V, d, scale, (__nv_bfloat16 *)O);
    else
        mhsa_simt_kernel<float, kWarps><<<grid, kWarps * 32, sm, st>>>(A, (const float *)Q, (const float *)K,
                                                                       (const float *)V, d, scale, (float *)O);
    return cudaGetLastError();
}

}  // namespace splat
