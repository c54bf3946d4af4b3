// tc_unfused.cu -- R-SDDMM and R-SpMM on sm_100a tensor cores, bf16.
//
// The paper's primitives (Listing 1 P:412-431 and the R-SpMM listing P:553-568) run one SIMT
// thread per output point.  Here the dense 128x128 sub-tiles of the contractions named by the
// tile plan (span specialisation) go through tcgen05:
//
//   R-SDDMM : S_tile = Q_t K_j^T (TMA -> 128B-swizzled SMEM -> tcgen05.mma -> TMEM, double
//             buffered) and 4 epilogue warps scatter scale * S of the tile's non-zeros to their
//             ACSR positions (thread = row; position = row_ptr[i] + rank of the column in its
//             row, the rank of the first column of the tile from the row's runs, the rest by
//             popcount of the pattern's row mask).
//   R-SpMM  : the 4 gather warps expand the row's ACSR values of key tile j into a dense bf16
//             P tile in TMEM (zeros off the mask), then O += P V_j as a TS-MMA (A from TMEM,
//             V an MN-major SMEM operand), O accumulated in TMEM over the tile's key tiles and
//             written once as bf16.
//
// Work units: (b*H+h, 128-row query tile), head-major, tiles in LPT order; persistent CTAs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sm100.cuh"

namespace splat {
namespace {

using namespace sm100;

constexpr int kThreadsU = 192;           // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue / gather
constexpr int kSub = 128 * 128;          // [128 rows x 64 bf16] swizzle-128B sub-tile (16 KB)

template <int D>
struct CfgU {
    static constexpr int kChunks = D / 64;
    static constexpr int kTileBytes = kChunks * kSub;
    static constexpr int QS = 2;
    static constexpr int KS = D == 64 ? 4 : 3;
    static constexpr int OFF_Q = 0;                       // SDDMM only
    static constexpr int OFF_K = OFF_Q + QS * kTileBytes;  // K ring (SDDMM) / V ring (SpMM)
    static constexpr int OFF_BAR = OFF_K + KS * kTileBytes;
    static constexpr int NBAR = 2 * QS + 2 * KS + 6;
    static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
};

struct ParamsU {
    DevAcsr A;
    int BH;
    float scale;
    float *S;                    // SDDMM output
    const __nv_bfloat16 *P;      // SpMM input (ACSR order)
    __nv_bfloat16 *O;            // SpMM output
};

__device__ __forceinline__ void unit_tile(const DevAcsr &A, int u, int &bh, int &t)
{
    bh = u / A.n_qt;
    t = A.order[u % A.n_qt];
}

// number of columns of the row's runs that lie left of column c0
__device__ __forceinline__ int run_rank(const int4 &g, int c0)
{
    if (g.z <= 0 || c0 <= g.x) return 0;
    const int n = (c0 - g.x + g.y - 1) / g.y;
    return n < g.z ? n : g.z;
}

struct RowRuns {
    int4 g[4];   // the row's <= 4 affine runs (start, step, count, offset); count 0 when absent
};

__device__ __forceinline__ int rank_before(const RowRuns &R, int c0)
{
    return run_rank(R.g[0], c0) + run_rank(R.g[1], c0) + run_rank(R.g[2], c0) + run_rank(R.g[3], c0);
}

__device__ __forceinline__ void row_info(const DevAcsr &A, int row, long long &base, RowRuns &R)
{
#pragma unroll
    for (int q = 0; q < 4; ++q) R.g[q] = make_int4(0, 1, 0, 0);
    base = 0;
    if (row < A.n) {
        base = A.row_ptr[row];
        const int ns = A.nseg[row];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < ns) R.g[q] = A.seg[(size_t)row * 4 + q];
    }
}

// ============================================================================ R-SDDMM
template <int D>
__global__ void __launch_bounds__(kThreadsU, 1)
rsddmm_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK, const ParamsU prm)
{
    using C = CfgU<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *q_full = bars, *q_empty = bars + C::QS;
    uint64_t *k_full = q_empty + C::QS, *k_empty = k_full + C::KS;
    uint64_t *s_full = k_empty + C::KS, *s_empty = s_full + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + C::NBAR);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const DevAcsr &A = prm.A;
    const int n_units = A.n_qt * prm.BH;

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::QS; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
        for (int i = 0; i < C::KS; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4); }
        fence_mbar_init();
        tma_prefetch(&tmQ); tma_prefetch(&tmK);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        int qi = 0, qc = 0, ki = 0, kc = 0;
        uint32_t qph = 0, kph = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int bh, t;
            unit_tile(A, u, bh, t);
            if (qc >= C::QS) mbar_wait(&q_empty[qi], qph ^ 1);
            if (lane == 0) {
                mbar_expect_tx(&q_full[qi], C::kTileBytes);
#pragma unroll
                for (int c = 0; c < C::kChunks; ++c)
                    tma_load_3d(smem + C::OFF_Q + qi * C::kTileBytes + c * kSub, &tmQ, &q_full[qi], 64 * c, t * 128, bh);
            }
            ++qc;
            if (++qi == C::QS) { qi = 0; qph ^= 1; }
            for (int e = A.qt_ptr[t]; e < A.qt_ptr[t + 1]; ++e) {
                const int kv = A.kv[e] & kKvMask;
                if (kc >= C::KS) mbar_wait(&k_empty[ki], kph ^ 1);
                if (lane == 0) {
                    mbar_expect_tx(&k_full[ki], C::kTileBytes);
#pragma unroll
                    for (int c = 0; c < C::kChunks; ++c)
                        tma_load_3d(smem + C::OFF_K + ki * C::kTileBytes + c * kSub, &tmK, &k_full[ki], 64 * c,
                                    kv * 128, bh);
                }
                ++kc;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idS = idesc_bf16(128, 128, false);
        const uint32_t sQ = smem_u32(smem + C::OFF_Q), sK = smem_u32(smem + C::OFF_K);
        int qi = 0, ki = 0, sb = 0;
        uint32_t qph = 0, kph = 0, scnt[2] = {0, 0};
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int bh, t;
            unit_tile(A, u, bh, t);
            mbar_wait(&q_full[qi], qph);
            const uint32_t qb = sQ + qi * C::kTileBytes;
            for (int e = A.qt_ptr[t]; e < A.qt_ptr[t + 1]; ++e) {
                mbar_wait(&k_full[ki], kph);
                if (scnt[sb] > 0) mbar_wait(&s_empty[sb], (scnt[sb] - 1) & 1);
                tc_fence_after();
                const uint32_t kb = sK + ki * C::kTileBytes;
                if (lane == 0) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = (kk >> 2) * kSub + (kk & 3) * 32;
                        mma_bf16_ss(tmem + sb * 128, sdesc_sw128(qb + off, 16, 1024), sdesc_sw128(kb + off, 16, 1024),
                                    idS, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(&s_full[sb]);
                    mma_commit(&k_empty[ki]);
                }
                ++scnt[sb];
                sb ^= 1;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
            }
            if (lane == 0) mma_commit(&q_empty[qi]);
            if (++qi == C::QS) { qi = 0; qph ^= 1; }
        }
    } else {
        // epilogue: thread = row of the query tile (TMEM lane)
        const int quad = warp & 3, r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        int sb = 0;
        uint32_t scnt[2] = {0, 0};
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int bh, t;
            unit_tile(A, u, bh, t);
            const int row = t * 128 + r;
            long long base;
            RowRuns R;
            row_info(A, row, base, R);
            float *srow = prm.S + (size_t)bh * A.nnz + base;
            for (int e = A.qt_ptr[t]; e < A.qt_ptr[t + 1]; ++e) {
                const int ent = A.kv[e];
                const int c0 = (ent & kKvMask) * 128;
                uint32_t mk[4] = {~0u, ~0u, ~0u, ~0u};
                if (ent & kPartialBit) {
                    const uint4 m4 = A.masks[(size_t)A.kv_mask[e] * 128 + r];
                    mk[0] = m4.x; mk[1] = m4.y; mk[2] = m4.z; mk[3] = m4.w;
                }
                if (row >= A.n) mk[0] = mk[1] = mk[2] = mk[3] = 0u;
                const int rk = rank_before(R, c0);
                float v[128];
                mbar_wait(&s_full[sb], scnt[sb] & 1);
                tc_fence_after();
#pragma unroll
                for (int w = 0; w < 4; ++w) tmem_ld32(tmem + lane_off + sb * 128 + 32 * w, v + 32 * w);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[sb]);
                ++scnt[sb];
                sb ^= 1;
                float *out = srow + rk;
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const uint32_t m = mk[w];
                    if (m == 0xffffffffu) {
#pragma unroll
                        for (int x = 0; x < 32; ++x) out[x] = prm.scale * v[32 * w + x];
                        out += 32;
                    } else if (m) {
                        int k = 0;
#pragma unroll
                        for (int x = 0; x < 32; ++x)
                            if ((m >> x) & 1u) out[k++] = prm.scale * v[32 * w + x];
                        out += k;
                    }
                }
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

// ============================================================================ R-SpMM
template <int D>
__global__ void __launch_bounds__(kThreadsU, 1)
rspmm_tc_kernel(const __grid_constant__ CUtensorMap tmV, const ParamsU prm)
{
    using C = CfgU<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *v_full = bars, *v_empty = bars + C::KS;
    uint64_t *p_full = v_empty + C::KS, *p_empty = p_full + 2;
    uint64_t *o_full = p_empty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + C::NBAR);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const DevAcsr &A = prm.A;
    const int n_units = A.n_qt * prm.BH;

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::KS; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&p_full[i], 4); mbar_init(&p_empty[i], 1); }
        mbar_init(o_full, 1);
        fence_mbar_init();
        tma_prefetch(&tmV);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;     // P buffers at columns [0,64), [64,128); O at [128, 128+D)

    if (warp == 0) {
        int ki = 0, kc = 0;
        uint32_t kph = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int bh, t;
            unit_tile(A, u, bh, t);
            for (int e = A.qt_ptr[t]; e < A.qt_ptr[t + 1]; ++e) {
                const int kv = A.kv[e] & kKvMask;
                if (kc >= C::KS) mbar_wait(&v_empty[ki], kph ^ 1);
                if (lane == 0) {
                    mbar_expect_tx(&v_full[ki], C::kTileBytes);
#pragma unroll
                    for (int c = 0; c < C::kChunks; ++c)
                        tma_load_3d(smem + C::OFF_K + ki * C::kTileBytes + c * kSub, &tmV, &v_full[ki], 64 * c,
                                    kv * 128, bh);
                }
                ++kc;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idO = idesc_bf16(128, D, true);
        const uint32_t sV = smem_u32(smem + C::OFF_K);
        int ki = 0, pb = 0;
        uint32_t kph = 0, pcnt[2] = {0, 0};
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int bh, t;
            unit_tile(A, u, bh, t);
            bool first = true;
            for (int e = A.qt_ptr[t]; e < A.qt_ptr[t + 1]; ++e) {
                mbar_wait(&v_full[ki], kph);
                mbar_wait(&p_full[pb], pcnt[pb] & 1);
                ++pcnt[pb];
                tc_fence_after();
                const uint32_t vb = sV + ki * C::kTileBytes;
                if (lane == 0) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16_ts(tmem + 128, tmem + pb * 64 + kk * 8, sdesc_sw128(vb + kk * 2048, kSub, 1024), idO,
                                    (first && kk == 0) ? 0u : 1u);
                    mma_commit(&v_empty[ki]);
                    mma_commit(&p_empty[pb]);
                }
                first = false;
                pb ^= 1;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
            }
            if (lane == 0) mma_commit(o_full);
        }
    } else {
        // gather + epilogue: thread = row of the query tile (TMEM lane)
        const int quad = warp & 3, r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        int pb = 0;
        uint32_t puse[2] = {0, 0}, ocnt = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int bh, t;
            unit_tile(A, u, bh, t);
            const int row = t * 128 + r;
            long long base;
            RowRuns R;
            row_info(A, row, base, R);
            const unsigned short *prow =
                reinterpret_cast<const unsigned short *>(prm.P) + (size_t)bh * A.nnz + base;
            for (int e = A.qt_ptr[t]; e < A.qt_ptr[t + 1]; ++e) {
                const int ent = A.kv[e];
                const int c0 = (ent & kKvMask) * 128;
                uint32_t mk[4] = {~0u, ~0u, ~0u, ~0u};
                if (ent & kPartialBit) {
                    const uint4 m4 = A.masks[(size_t)A.kv_mask[e] * 128 + r];
                    mk[0] = m4.x; mk[1] = m4.y; mk[2] = m4.z; mk[3] = m4.w;
                }
                if (row >= A.n) mk[0] = mk[1] = mk[2] = mk[3] = 0u;
                const unsigned short *src = prow + rank_before(R, c0);
                uint32_t pw[64];
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const uint32_t m = mk[w];
                    uint32_t h[32];
                    if (m == 0xffffffffu) {
#pragma unroll
                        for (int x = 0; x < 32; ++x) h[x] = __ldg(src + x);
                        src += 32;
                    } else {
                        int k = 0;
#pragma unroll
                        for (int x = 0; x < 32; ++x) {
                            h[x] = 0u;
                            if ((m >> x) & 1u) h[x] = __ldg(src + k++);
                        }
                        src += k;
                    }
#pragma unroll
                    for (int x = 0; x < 16; ++x) pw[16 * w + x] = h[2 * x] | (h[2 * x + 1] << 16);
                }
                // this P buffer is free once the PV that read it two tiles ago has completed
                if (puse[pb] > 0) mbar_wait(&p_empty[pb], (puse[pb] - 1) & 1);
                tc_fence_after();
                tmem_st32(tmem + lane_off + pb * 64, reinterpret_cast<const float *>(pw));
                tmem_st32(tmem + lane_off + pb * 64 + 32, reinterpret_cast<const float *>(pw + 32));
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[pb]);
                ++puse[pb];
                pb ^= 1;
            }
            // epilogue: O (the plain sum P V) -> bf16 -> HBM
            mbar_wait(o_full, ocnt & 1);
            ++ocnt;
            tc_fence_after();
            const bool empty = A.qt_ptr[t] == A.qt_ptr[t + 1];   // no key tile: O = 0
            __nv_bfloat16 *orow = prm.O + ((size_t)bh * A.n + row) * D;
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                float o[32];
                tmem_ld32(tmem + lane_off + 128 + c * 32, o);
                tmem_wait_ld();
                if (empty) {
#pragma unroll
                    for (int x = 0; x < 32; ++x) o[x] = 0.f;
                }
                if (row < A.n) {
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        uint4 w4;
                        w4.x = pack_bf16(o[8 * v + 0], o[8 * v + 1]);
                        w4.y = pack_bf16(o[8 * v + 2], o[8 * v + 3]);
                        w4.z = pack_bf16(o[8 * v + 4], o[8 * v + 5]);
                        w4.w = pack_bf16(o[8 * v + 6], o[8 * v + 7]);
                        *reinterpret_cast<uint4 *>(orow + c * 32 + 8 * v) = w4;
                    }
                }
            }
            tc_fence_before();
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

template <int D>
cudaError_t launch_sddmm_d(const DevAcsr &A, const void *Q, const void *K, int BH, float scale, float *S,
                           cudaStream_t st)
{
    CUtensorMap mq, mk;
    if (!make_map(&mq, Q, BH, A.n, D) || !make_map(&mk, K, BH, A.n, D)) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(rsddmm_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgU<D>::SMEM);
    if (e != cudaSuccess) return e;
    ParamsU p{};
    p.A = A;
    p.BH = BH;
    p.scale = scale;
    p.S = S;
    int dev = 0;
    cudaGetDevice(&dev);
    const long long units = (long long)A.n_qt * BH;
    const int grid = (int)(units < num_sms(dev) ? units : num_sms(dev));
    rsddmm_tc_kernel<D><<<grid, kThreadsU, CfgU<D>::SMEM, st>>>(mq, mk, p);
    return cudaGetLastError();
}

template <int D>
cudaError_t launch_spmm_d(const DevAcsr &A, const void *P, const void *V, int BH, void *O, cudaStream_t st)
{
    CUtensorMap mv;
    if (!make_map(&mv, V, BH, A.n, D)) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(rspmm_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgU<D>::SMEM);
    if (e != cudaSuccess) return e;
    ParamsU p{};
    p.A = A;
    p.BH = BH;
    p.P = reinterpret_cast<const __nv_bfloat16 *>(P);
    p.O = reinterpret_cast<__nv_bfloat16 *>(O);
    int dev = 0;
    cudaGetDevice(&dev);
    const long long units = (long long)A.n_qt * BH;
    const int grid = (int)(units < num_sms(dev) ? units : num_sms(dev));
    rspmm_tc_kernel<D><<<grid, kThreadsU, CfgU<D>::SMEM, st>>>(mv, p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_rsddmm_tc(const DevAcsr &A, const void *Q, const void *K, int BH, int d, float scale, float *S,
                             cudaStream_t st)
{
    if (d == 64) return launch_sddmm_d<64>(A, Q, K, BH, scale, S, st);
    if (d == 128) return launch_sddmm_d<128>(A, Q, K, BH, scale, S, st);
    return cudaErrorNotSupported;
}

cudaError_t launch_rspmm_tc(const DevAcsr &A, const void *P, const void *V, int BH, int d, void *O, cudaStream_t st)
{
    if (d == 64) return launch_spmm_d<64>(A, P, V, BH, O, st);
    if (d == 128) return launch_spmm_d<128>(A, P, V, BH, O, st);
    return cudaErrorNotSupported;
}

}  // namespace splat
