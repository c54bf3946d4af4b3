// tc_fused.cu -- fused sparse MHSA on sm_100a tensor cores.
//
// Computes O = softmax(M (x) scale*Q K^T) V per (b, h) (PAPER Eq. 1)
// without writing S or P to HBM.  The paper launches R-SDDMM, softmax and
// R-SpMM as separate kernels with HBM buffers in between (Listing 4,
// P:700-711); here one persistent kernel walks the tile plan:
//
//   work unit  = (b*H+h, 128-row query tile t), LPT order, CTAs round-robin
//   per unit   : for each 128-column key tile j listed for t (span):
//     TMA warp  : K_j, V_j  -> 128B-swizzled SMEM rings (3-D tensor maps,
//                 out-of-range rows zero-filled)
//     MMA warp  : S_j = Q K_j^T  (tcgen05.mma kind::f16, M=128 N=128, fp32
//                 accumulator in TMEM, double-buffered), then O += P_j V_j
//                 (M=128 N=d, V as an MN-major operand)
//     4 softmax warps (one query row per thread, TMEM lane = row):
//                 tcgen05.ld S_j -> fast-index mask on PARTIAL tiles (A-7:
//                 column c of run (start, step, count) iff (c-start) % step
//                 == 0 and 0 <= (c-start)/step < count) -> online max / sum
//                 with exp2 (log2 e folded into the scale) -> P_j (bf16) into
//                 SMEM in the UMMA K-major layout; O in TMEM is rescaled
//                 only when the running max grows by more than 2^8.
//   epilogue   : O / l -> bf16 -> HBM.
//
// TMEM: S buffers at columns [0,128) and [128,256), O at [256, 256+d).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <mutex>

#include "kernels.h"
#include "sm100.cuh"

namespace splat {
namespace {

using namespace sm100;

constexpr int kThreads = 192;          // warp 0 TMA, warp 1 MMA, warps 2..5 softmax
constexpr int kTileBytes64 = 128 * 128; // one [128 rows x 64 bf16] swizzle-128B sub-tile (16 KB)
constexpr float kRescaleThresh = 8.0f;  // log2 units

template <int D>
struct Cfg {
    static constexpr int kChunks = D / 64;                  // 64-column sub-tiles along d
    static constexpr int kTileBytes = kChunks * kTileBytes64; // one Q/K/V tile
    static constexpr int QS = D == 64 ? 2 : 1;
    static constexpr int KS = D == 64 ? 3 : 2;
    static constexpr int PS = 2;
    static constexpr int kPBytes = 2 * kTileBytes64;        // 128 x 128 bf16
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + QS * kTileBytes;
    static constexpr int OFF_V = OFF_K + KS * kTileBytes;
    static constexpr int OFF_P = OFF_V + KS * kTileBytes;
    static constexpr int OFF_BAR = OFF_P + PS * kPBytes;
    static constexpr int NBAR = 2 * QS + 4 * KS + 8;
    static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;   // + alignment slack
};

struct Params {
    DevAcsr A;
    int BH, N;
    float scale_log2;
    __nv_bfloat16 *O;
};

__device__ __forceinline__ void set_bits(uint32_t (&m)[4], int lo, int hi)
{
    // set bits [lo, hi] (0 <= lo <= hi < 128)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const int a = max(lo, 32 * w), b = min(hi, 32 * w + 31);
        if (a <= b) {
            const int n = b - a + 1;
            const uint32_t bits = n == 32 ? 0xffffffffu : ((1u << n) - 1u);
            m[w] |= bits << (a - 32 * w);
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
mhsa_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const Params prm)
{
    using C = Cfg<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *q_full = bars, *q_empty = bars + C::QS;
    uint64_t *k_full = q_empty + C::QS, *k_empty = k_full + C::KS;
    uint64_t *v_full = k_empty + C::KS, *v_empty = v_full + C::KS;
    uint64_t *s_full = v_empty + C::KS, *s_empty = s_full + 2;
    uint64_t *p_full = s_empty + 2, *p_empty = p_full + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + C::NBAR);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const DevAcsr &A = prm.A;
    const int n_units = A.n_qt * prm.BH;

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::QS; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
        for (int i = 0; i < C::KS; ++i) {
            mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4);
            mbar_init(&p_full[i], 4); mbar_init(&p_empty[i], 1);
        }
        fence_mbar_init();
        tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            int qi = 0, ki = 0, vi = 0;
            uint32_t qph = 0, kph = 0, vph = 0;
            int qcnt = 0, kcnt = 0, vcnt = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                const int t = A.order[u / prm.BH], bh = u % prm.BH;
                if (qcnt >= C::QS) mbar_wait(&q_empty[qi], qph ^ 1);
                mbar_expect_tx(&q_full[qi], C::kTileBytes);
#pragma unroll
                for (int c = 0; c < C::kChunks; ++c)
                    tma_load_3d(smem + C::OFF_Q + qi * C::kTileBytes + c * kTileBytes64, &tmQ, &q_full[qi], 64 * c,
                                t * 128, bh);
                ++qcnt;
                if (++qi == C::QS) { qi = 0; qph ^= 1; }
                const int e0 = A.qt_ptr[t], e1 = A.qt_ptr[t + 1];
                for (int e = e0; e < e1; ++e) {
                    const int kv = A.kv[e] & kKvMask;
                    if (kcnt >= C::KS) mbar_wait(&k_empty[ki], kph ^ 1);
                    mbar_expect_tx(&k_full[ki], C::kTileBytes);
#pragma unroll
                    for (int c = 0; c < C::kChunks; ++c)
                        tma_load_3d(smem + C::OFF_K + ki * C::kTileBytes + c * kTileBytes64, &tmK, &k_full[ki],
                                    64 * c, kv * 128, bh);
                    ++kcnt;
                    if (++ki == C::KS) { ki = 0; kph ^= 1; }
                    if (vcnt >= C::KS) mbar_wait(&v_empty[vi], vph ^ 1);
                    mbar_expect_tx(&v_full[vi], C::kTileBytes);
#pragma unroll
                    for (int c = 0; c < C::kChunks; ++c)
                        tma_load_3d(smem + C::OFF_V + vi * C::kTileBytes + c * kTileBytes64, &tmV, &v_full[vi],
                                    64 * c, kv * 128, bh);
                    ++vcnt;
                    if (++vi == C::KS) { vi = 0; vph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idS = idesc_bf16(128, 128, false);
            constexpr uint32_t idO = idesc_bf16(128, D, true);
            const uint32_t sQ = smem_u32(smem + C::OFF_Q), sK = smem_u32(smem + C::OFF_K);
            const uint32_t sV = smem_u32(smem + C::OFF_V), sP = smem_u32(smem + C::OFF_P);
            int qi = 0, ki = 0, vi = 0;
            uint32_t qph = 0, kph = 0, vph = 0;
            uint32_t s_use[2] = {0, 0}, p_use[2] = {0, 0};
            int sb = 0;   // next S buffer
            uint32_t pv_count = 0;   // PVs issued so far (global P-buffer alternation, as the softmax's)
            auto issue_pv = [&](bool first) {
                const int pb = pv_count & 1;
                ++pv_count;
                mbar_wait(&p_full[pb], p_use[pb] & 1);
                mbar_wait(&v_full[vi], vph);
                tc_fence_after();
                const uint32_t pbase = sP + pb * C::kPBytes, vbase = sV + vi * C::kTileBytes;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t a = sdesc_sw128(pbase + (kk >> 2) * kTileBytes64 + (kk & 3) * 32, 16, 1024);
                    const uint64_t b = sdesc_sw128(vbase + kk * 2048, kTileBytes64, 1024);
                    mma_bf16_ss(tmem + 256, a, b, idO, (first && kk == 0) ? 0u : 1u);
                }
                mma_commit(&v_empty[vi]);
                mma_commit(&p_empty[pb]);
                ++p_use[pb];
                if (++vi == C::KS) { vi = 0; vph ^= 1; }
            };
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                const int t = A.order[u / prm.BH];
                const int e0 = A.qt_ptr[t], n = A.qt_ptr[t + 1] - e0;
                mbar_wait(&q_full[qi], qph);
                const uint32_t qbase = sQ + qi * C::kTileBytes;
                for (int j = 0; j < n; ++j) {
                    mbar_wait(&k_full[ki], kph);
                    if (s_use[sb] > 0) mbar_wait(&s_empty[sb], (s_use[sb] - 1) & 1);
                    tc_fence_after();
                    const uint32_t kbase = sK + ki * C::kTileBytes;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = (kk >> 2) * kTileBytes64 + (kk & 3) * 32;
                        mma_bf16_ss(tmem + sb * 128, sdesc_sw128(qbase + off, 16, 1024),
                                    sdesc_sw128(kbase + off, 16, 1024), idS, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(&k_empty[ki]);
                    mma_commit(&s_full[sb]);
                    ++s_use[sb];
                    sb ^= 1;
                    if (++ki == C::KS) { ki = 0; kph ^= 1; }
                    if (j == n - 1) {
                        mma_commit(&q_empty[qi]);
                        if (++qi == C::QS) { qi = 0; qph ^= 1; }
                    }
                    if (j > 0) issue_pv(j - 1 == 0);
                }
                issue_pv(n == 1);
            }
        }
    } else {
        // ------------------------------------------------------------ softmax warps
        const int quad = warp & 3;              // TMEM lane quadrant this warp may access
        const int r = quad * 32 + lane;         // row within the query tile
        const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
        const uint32_t sP = smem_u32(smem + C::OFF_P);
        uint32_t s_use[2] = {0, 0}, p_use[2] = {0, 0};
        int sb = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const int t = A.order[u / prm.BH], bh = u % prm.BH;
            const int e0 = A.qt_ptr[t], n = A.qt_ptr[t + 1] - e0;
            const int row = t * 128 + r;
            int4 g[3];
            int ns = 0;
            if (row < A.n) {
                ns = A.nseg[row];
#pragma unroll
                for (int s = 0; s < 3; ++s) g[s] = A.seg[(size_t)row * 4 + s];
            }
            float m_run = -INFINITY, l_run = 0.f;
            for (int j = 0; j < n; ++j) {
                const int ent = A.kv[e0 + j];
                const int kv0 = (ent & kKvMask) * 128;
                const bool partial = (ent & kPartialBit) != 0;
                float s[128];
                mbar_wait(&s_full[sb], s_use[sb] & 1);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld32(lane_addr + sb * 128 + c * 32, s + 32 * c);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[sb]);
                ++s_use[sb];
                const int pb = sb;   // P buffer follows the S buffer parity (= j & 1 within the stream)
                sb ^= 1;
                if (partial) {
                    uint32_t mk[4] = {0, 0, 0, 0};
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        if (q < ns) {
                            const int start = g[q].x, step = g[q].y, cnt = g[q].z;
                            const int last = start + step * (cnt - 1);
                            const int lo = max(start, kv0), hi = min(last, kv0 + 127);
                            if (lo <= hi) {
                                if (step == 1) {
                                    set_bits(mk, lo - kv0, hi - kv0);
                                } else {
#pragma unroll
                                    for (int w = 0; w < 4; ++w) {
                                        const int a = max(lo, kv0 + 32 * w), b = min(hi, kv0 + 32 * w + 31);
                                        const int first = start + ((a - start + step - 1) / step) * step;
                                        uint32_t bits = 0;
                                        for (int c = first; c <= b; c += step) bits |= 1u << (c - kv0 - 32 * w);
                                        mk[w] |= bits;
                                    }
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int x = 0; x < 128; ++x)
                        if (!((mk[x >> 5] >> (x & 31)) & 1u)) s[x] = -INFINITY;
                }
                float mx = s[0];
#pragma unroll
                for (int x = 1; x < 128; ++x) mx = fmaxf(mx, s[x]);
                mx *= prm.scale_log2;
                float alpha = 1.f;
                bool resc = false;
                if (mx > m_run + kRescaleThresh) {
                    if (m_run != -INFINITY) {
                        alpha = ex2(m_run - mx);
                        resc = true;
                    }
                    m_run = mx;
                    l_run *= alpha;
                }
                const float mref = m_run == -INFINITY ? 0.f : m_run;
                float ls = 0.f;
                // P buffer must be free: PV of its previous use complete
                if (p_use[pb] > 0) mbar_wait(&p_empty[pb], (p_use[pb] - 1) & 1);
                const uint32_t prow = sP + pb * C::kPBytes + r * 128;
#pragma unroll
                for (int c16 = 0; c16 < 16; ++c16) {
                    uint32_t w[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const float p0 = ex2(fmaf(s[c16 * 8 + 2 * h], prm.scale_log2, -mref));
                        const float p1 = ex2(fmaf(s[c16 * 8 + 2 * h + 1], prm.scale_log2, -mref));
                        ls += p0 + p1;
                        w[h] = pack_bf16(p0, p1);
                    }
                    const uint32_t addr = prow + (c16 >> 3) * kTileBytes64 + (((c16 & 7) ^ (r & 7)) << 4);
                    st_shared_v4(addr, w[0], w[1], w[2], w[3]);
                }
                l_run += ls;
                fence_proxy_async_smem();
                // rescale O (TMEM) when some row of this warp moved its max by > 2^8
                if (__any_sync(0xffffffffu, resc) && j > 0) {
                    const int pprev = pb ^ 1;   // PV_{j-1} used the other P buffer
                    mbar_wait(&p_empty[pprev], (p_use[pprev] - 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        float o[32];
                        tmem_ld32(lane_addr + 256 + c * 32, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int x = 0; x < 32; ++x) o[x] *= alpha;
                        tmem_st32(lane_addr + 256 + c * 32, o);
                    }
                    tmem_wait_st();
                }
                ++p_use[pb];
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[pb]);
            }
            // epilogue: wait for the last PV, O / l -> bf16 -> HBM
            {
                const int pl = (sb ^ 1);     // buffer of the last P
                mbar_wait(&p_empty[pl], (p_use[pl] - 1) & 1);
                tc_fence_after();
                const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
                __nv_bfloat16 *orow = prm.O + ((size_t)bh * prm.N + row) * D;
#pragma unroll
                for (int c = 0; c < D / 32; ++c) {
                    float o[32];
                    tmem_ld32(lane_addr + 256 + c * 32, o);
                    tmem_wait_ld();
                    if (row < prm.N) {
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            uint4 w;
                            w.x = pack_bf16(o[8 * v + 0] * inv, o[8 * v + 1] * inv);
                            w.y = pack_bf16(o[8 * v + 2] * inv, o[8 * v + 3] * inv);
                            w.z = pack_bf16(o[8 * v + 4] * inv, o[8 * v + 5] * inv);
                            w.w = pack_bf16(o[8 * v + 6] * inv, o[8 * v + 7] * inv);
                            *reinterpret_cast<uint4 *>(orow + c * 32 + 8 * v) = w;
                        }
                    }
                }
                tc_fence_before();
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode()
{
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

bool make_map(CUtensorMap *m, const void *base, int BH, int N, int d)
{
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)N, (cuuint64_t)BH};
    cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)N * d * 2};
    cuuint32_t box[3] = {64, 128, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms(int dev)
{
    static int cache[64] = {0};
    if (dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
    return cache[dev];
}

template <int D>
cudaError_t launch_d(const DevAcsr &A, const void *Q, const void *K, const void *V, int BH, float scale, void *O,
                     cudaStream_t st)
{
    CUtensorMap mq, mk, mv;
    if (!make_map(&mq, Q, BH, A.n, D) || !make_map(&mk, K, BH, A.n, D) || !make_map(&mv, V, BH, A.n, D))
        return cudaErrorInvalidValue;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(mhsa_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<D>::SMEM);
        if (e != cudaSuccess) return e;
        attr_set[dev & 63] = true;
    }
    Params p;
    p.A = A;
    p.BH = BH;
    p.N = A.n;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.O = reinterpret_cast<__nv_bfloat16 *>(O);
    const long long units = (long long)A.n_qt * BH;
    const int grid = (int)(units < num_sms(dev) ? units : num_sms(dev));
    mhsa_tc_kernel<D><<<grid, kThreads, Cfg<D>::SMEM, st>>>(mq, mk, mv, p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mhsa_tc(const DevAcsr &A, const void *Q, const void *K, const void *V, int BH, int d,
                           float scale, void *O, cudaStream_t st, int *n_launch)
{
    *n_launch = 1;
    if (d == 64) return launch_d<64>(A, Q, K, V, BH, scale, O, st);
    if (d == 128) return launch_d<128>(A, Q, K, V, BH, scale, O, st);
    return cudaErrorNotSupported;
}

}  // namespace splat
