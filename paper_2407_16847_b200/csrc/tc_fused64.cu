// tc_fused64.cu -- fused sparse MHSA for d = 64 on sm_100a, half-row variant.
//
// O = softmax(M (x) scale*Q K^T) V per (b, h) (PAPER Eq. 1; the softmax runs over each
// row's non-zeros, reading R-1 of DESIGN.md); S and P never leave the SM.  A work unit is one
// 128-row query tile of one (b, h) against its plan entries (the key tiles touched by any of its
// rows: the span of P:573 at tile granularity), handed out dynamically from the call's work
// counter, longest units first.
//
// Two independent tile groups g per CTA (640 threads), each with
//   producer warp g      : Q of each unit (TMA); per entry K, V (TMA) and the entry's chunk bits
//                          plus, for a PARTIAL entry, its 128 row masks (2 KB bulk copy) into a ring;
//   MMA warp 2 + g       : S = Q K^T (SS, M = N = 128), O += P V (TS, P from TMEM);
//   8 softmax warps      : warps 4 + 8g + 4h + q, lane quadrant q, half h of the S row (columns
//                          [64 h, 64 h + 64)); thread = query row = TMEM lane.
// so every SM sub-partition runs four softmax warps (two groups x two halves) -- the latency of a
// tile's serial chain (S ready -> load -> max -> exchange -> exponentials -> P store -> hand-off)
// of one warp is covered by the other three.  The two halves of a row exchange their maxima
// through shared memory (named barriers per group and quadrant) and then take the same decision
// for the row's running reference (stale max: O and the sums are rescaled only when the max grows
// by more than 2^kBump), so the output is exactly the softmax of the row in exact arithmetic.
// exp2 (log2 e folded into the scale) runs on MUFU and, for part of every chunk, on the FMA pipe
// (degree-3 polynomial).  Each half sums its own exponentials; the two partial sums meet in the
// epilogue.
//
// TMEM (512 columns): S_g [128 g, 128 g + 128), O_g [256 + 64 g, +64), P_g [384 + 64 g, +64).
// Diagnostics build only (SPLAT_TC_PAIRED64=3): the product library does not contain this kernel.
#ifdef SPLAT_DIAG
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sm100.cuh"
#include "softmax_math.cuh"

namespace splat {
namespace {

using namespace sm100;
using namespace smx;

constexpr int kThreads64 = 640;
constexpr float kBump = 8.0f;        // stale max: rescale only when the row max grows by > 2^8

#ifndef SPLAT_NEMU64
#define SPLAT_NEMU64 8               // exponentials of each 32-column chunk emulated on the FMA pipe
#endif

struct H64 {
    static constexpr int QS = 2, KS = 2, VS = 2, MS = 3;
    static constexpr int TB = 128 * 128;                         // 16 KB: 128 rows x 64 bf16
    static constexpr int MB = 128 * 16;                          // 2 KB: 128 row masks of 128 bits
    static constexpr int OFF_Q = 0, OFF_K = QS * TB, OFF_V = OFF_K + KS * TB, OFF_M = OFF_V + VS * TB;
    static constexpr int OFF_XM = OFF_M + MS * MB;               // [2 bufs][2 halves][128] f32 row maxima
    static constexpr int OFF_XL = OFF_XM + 2 * 2 * 128 * 4;      // [2 halves][128] f32 partial sums
    static constexpr int GROUP = OFF_XL + 2 * 128 * 4;           // per tile group
    static constexpr int OFF_BAR = 2 * GROUP;
    // per group: q_full[QS] q_empty[QS] k_full[KS] k_empty[KS] v_full[VS] v_empty[VS] m_full[MS]
    //            m_empty[MS] s_full s_empty p_full pv_done epi
    static constexpr int NB = 2 * QS + 2 * KS + 2 * VS + 2 * MS + 5;
    static constexpr int OFF_EB = OFF_BAR + 2 * NB * 8;          // [2][MS] u32 chunk bits of the ring entry
    static constexpr int OFF_HDR = (OFF_EB + 2 * MS * 4 + 15) / 16 * 16;   // [2][QS] int4 (t, bh, j0, j1)
    static constexpr int OFF_TMEM = OFF_HDR + 2 * QS * 16;
    static constexpr int SMEM = OFF_TMEM + 16 + 1024;
    static_assert(SMEM <= 232448, "shared memory budget");
};

struct P64 {
    DevAcsr A;
    int BH, N;
    float scale_log2;
    __nv_bfloat16 *O;
    unsigned long long *sched;   // [work counter, done counter] of this call's launch slot
    int dbg;
};

struct Unit64 {
    int t, bh, j0, j1;
};

__device__ __forceinline__ Unit64 fetch_unit64(const DevAcsr &A, int BH, int v)
{
    int k = 0, bh = 0;
    for (int b = 0; b < A.t_n_buckets; ++b) {
        const int nb = A.t_bucket_start[b + 1] - A.t_bucket_start[b];
        const int ub = nb * BH;
        if (v < ub) {
            bh = v / nb;
            k = A.t_bucket_start[b] + v % nb;
            break;
        }
        v -= ub;
    }
    const int4 x = A.t_info[k];
    return Unit64{x.x, bh, x.y, x.z};
}

#define DBG64(m) (kDiag && (prm.dbg & (m)))

#if defined(SPLAT_FUSED_PROF) && !defined(SPLAT_DIAG)
#error "SPLAT_FUSED_PROF needs the diagnostics build (-DSPLAT_DIAG)"
#endif
#ifdef SPLAT_FUSED_PROF
// Profiling aid (diagnostics build): cycles per phase of every warp, accumulated in registers and
// summed over all CTAs at exit; read with splat_debug_prof64.  [warp][phase], phase 15 = total.
__device__ unsigned long long g_prof64[20][16];
#define PROF_DECL unsigned int pf_t = (unsigned int)clock(), pf_t0 = pf_t; unsigned int pf_acc[12] = {0,0,0,0,0,0,0,0,0,0,0,0};
#define PROF(k) do { const unsigned int t_ = (unsigned int)clock(); pf_acc[k] += t_ - pf_t; pf_t = t_; } while (0)
#define PROF_FLUSH() do { if (lane == 0) { for (int k_ = 0; k_ < 12; ++k_) atomicAdd(&g_prof64[warp][k_], (unsigned long long)pf_acc[k_]); \
                               atomicAdd(&g_prof64[warp][15], (unsigned long long)((unsigned int)clock() - pf_t0)); } } while (0)
#else
#define PROF_DECL
#define PROF(k) do { } while (0)
#define PROF_FLUSH() do { } while (0)
#endif

__global__ void __launch_bounds__(kThreads64, 1)
mhsa64_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, const P64 prm)
{
    using C = H64;
    extern __shared__ __align__(1024) uint8_t smem[];
    if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0u) __trap();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // group of this warp: producers 0 / 1, MMA 2 / 3, softmax 4-11 / 12-19
    const int g = warp >= 4 ? (warp - 4) >> 3 : (warp & 1);
    uint8_t *gs = smem + g * C::GROUP;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR) + g * C::NB;
    uint64_t *q_full = bars, *q_empty = q_full + C::QS;
    uint64_t *k_full = q_empty + C::QS, *k_empty = k_full + C::KS;
    uint64_t *v_full = k_empty + C::KS, *v_empty = v_full + C::VS;
    uint64_t *m_full = v_empty + C::VS, *m_empty = m_full + C::MS;
    uint64_t *s_full = m_empty + C::MS, *s_empty = s_full + 1, *p_full = s_empty + 1;
    uint64_t *pv_done = p_full + 1, *epi = pv_done + 1;
    uint32_t *ebits = reinterpret_cast<uint32_t *>(smem + C::OFF_EB) + g * C::MS;
    int4 *hdr = reinterpret_cast<int4 *>(smem + C::OFF_HDR) + g * C::QS;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::OFF_TMEM);
    const DevAcsr &A = prm.A;
    const int n_units = A.n_qt * prm.BH;

    if (threadIdx.x == 0) {
        for (int gg = 0; gg < 2; ++gg) {
            uint64_t *b = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR) + gg * C::NB;
            int o = 0;
            for (int i = 0; i < C::QS; ++i) mbar_init(&b[o++], 1);   // q_full  (producer)
            for (int i = 0; i < C::QS; ++i) mbar_init(&b[o++], 9);   // q_empty (unit's last QK^T commit + 8 softmax warps)
            for (int i = 0; i < 2 * C::KS + 2 * C::VS; ++i) mbar_init(&b[o++], 1);
            for (int i = 0; i < C::MS; ++i) mbar_init(&b[o++], 1);   // m_full  (producer)
            for (int i = 0; i < C::MS; ++i) mbar_init(&b[o++], 8);   // m_empty (8 softmax warps)
            mbar_init(&b[o++], 1);   // s_full  (MMA commit)
            mbar_init(&b[o++], 8);   // s_empty (8 softmax warps)
            mbar_init(&b[o++], 8);   // p_full  (8 softmax warps)
            mbar_init(&b[o++], 1);   // pv_done (MMA commit)
            mbar_init(&b[o++], 1);   // epi     (MMA commit)
        }
        fence_mbar_init();
        tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 2) {
        // ------------------------------------------------------------ producer of group g
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
        PROF_DECL
        int qi = 0, qc = 0, ki = 0, kc = 0, vi = 0, vc = 0, mi = 0, mc = 0;
        uint32_t qph = 0, kph = 0, vph = 0, mph = 0;
        bool pv = false;            // V of the previous entry still to load
        int pv_kv = 0, pv_bh = 0;
        auto load_v = [&]() {
            PROF(0);
            if (vc >= C::VS) mbar_wait(&v_empty[vi], vph ^ 1);
            PROF(3);
            if (lane == 0) {
                mbar_expect_tx(&v_full[vi], C::TB);
                tma_load_3d(gs + C::OFF_V + vi * C::TB, &tmV, &v_full[vi], 0, pv_kv * kKvUnit, pv_bh);
            }
            ++vc;
            if (++vi == C::VS) { vi = 0; vph ^= 1; }
            pv = false;
        };
        auto grab = [&]() {
            int v = 0;
            if (lane == 0) v = (int)atomicAdd(prm.sched, 1ull);
            v = __shfl_sync(0xffffffffu, v, 0);
            return v < n_units ? fetch_unit64(A, prm.BH, v) : Unit64{-1, 0, 0, 0};
        };
        Unit64 nx = grab();
        while (true) {
            const Unit64 un = nx;
            if (qc >= C::QS) mbar_wait(&q_empty[qi], qph ^ 1);
            if (un.t < 0) {
                if (lane == 0) {
                    hdr[qi] = make_int4(-1, 0, 0, 0);
                    mbar_arrive(&q_full[qi]);
                }
                break;
            }
            nx = grab();                      // next unit, fetched in the shadow of this one
            if (lane == 0) {
                hdr[qi] = make_int4(un.t, un.bh, un.j0, un.j1);
                mbar_expect_tx(&q_full[qi], C::TB);      // release: the header is visible to the waiters
                tma_load_3d(gs + C::OFF_Q + qi * C::TB, &tmQ, &q_full[qi], 0, un.t * 128, un.bh);
            }
            ++qc;
            if (++qi == C::QS) { qi = 0; qph ^= 1; }
            // entry metadata, read by lane 0 one entry ahead (the loads overlap the barrier waits)
            int kv = 0, mid = -1;
            uint32_t bits = 0u;
            if (lane == 0 && un.j0 < un.j1) {
                kv = A.kv[un.j0] & kKvMask;
                mid = A.kv_mask[un.j0];
                bits = A.qt_bits[un.j0];
            }
            for (int j = un.j0; j < un.j1; ++j) {
                int nkv = 0, nmid = -1;
                uint32_t nbits = 0u;
                if (lane == 0 && j + 1 < un.j1) {
                    nkv = A.kv[j + 1] & kKvMask;
                    nmid = A.kv_mask[j + 1];
                    nbits = A.qt_bits[j + 1];
                }
                // chunk bits, and the row masks where some warp has a masked chunk
                PROF(0);
                if (mc >= C::MS) mbar_wait(&m_empty[mi], mph ^ 1);
                PROF(1);
                if (lane == 0) {
                    ebits[mi] = bits;
                    const uint32_t need = bits & ~(bits >> 16) & 0xFFFFu;
                    if (need && mid >= 0) {
                        mbar_expect_tx(&m_full[mi], C::MB);
                        bulk_load(gs + C::OFF_M + mi * C::MB, A.masks + (size_t)mid * 128, C::MB, &m_full[mi]);
                    } else {
                        mbar_arrive(&m_full[mi]);
                    }
                }
                ++mc;
                if (++mi == C::MS) { mi = 0; mph ^= 1; }
                PROF(0);
                if (kc >= C::KS) mbar_wait(&k_empty[ki], kph ^ 1);
                PROF(2);
                if (lane == 0) {
                    mbar_expect_tx(&k_full[ki], C::TB);
                    tma_load_3d(gs + C::OFF_K + ki * C::TB, &tmK, &k_full[ki], 0, kv * kKvUnit, un.bh);
                }
                ++kc;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
                if (pv) load_v();
                pv = true;
                pv_kv = kv;
                pv_bh = un.bh;
                kv = nkv;
                mid = nmid;
                bits = nbits;
            }
        }
        if (pv) load_v();
        PROF(0);
        PROF_FLUSH();
    } else if (warp < 4) {
        // ------------------------------------------------------------ MMA issuer of group g
        // S(j) = Q K_j^T as soon as K_j is resident and the softmax has read S(j-1); then
        // O += P(j-1) V_(j-1).  Every operand warp-uniform, issue under elect.sync.
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
        PROF_DECL
        const int gu = __shfl_sync(0xffffffffu, g, 0);
        const uint32_t tmu = __shfl_sync(0xffffffffu, tmem, 0);
        uint8_t *gsu = smem + gu * C::GROUP;
        uint64_t *bu = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR) + gu * C::NB;
        uint64_t *uq_full = bu, *uq_empty = uq_full + C::QS, *uk_full = uq_empty + C::QS, *uk_empty = uk_full + C::KS;
        uint64_t *uv_full = uk_empty + C::KS, *uv_empty = uv_full + C::VS;
        uint64_t *us_full = uv_empty + C::VS + 2 * C::MS, *us_empty = us_full + 1, *up_full = us_empty + 1;
        uint64_t *upv_done = up_full + 1, *uepi = upv_done + 1;
        constexpr uint32_t idS = idesc_bf16(128, 128, false);
        constexpr uint32_t idO = idesc_bf16(128, 64, true);
        const uint32_t sQ = smem_u32(gsu + C::OFF_Q), sK = smem_u32(gsu + C::OFF_K), sV = smem_u32(gsu + C::OFF_V);
        const uint32_t s_tm = tmu + gu * 128, o_tm = tmu + 256 + gu * 64, p_tm = tmu + 384 + gu * 64;
        int qi = 0;
        uint32_t qph = 0, pcnt = 0, scnt = 0, gent = 0;
        bool pend = false, p_first = false, p_last = false;
        int pst = 0;
        uint32_t pph = 0;
        auto flush_pv = [&]() {
            PROF(0);
            mbar_wait(up_full, pcnt & 1);
            PROF(4);
            ++pcnt;
            mbar_wait(&uv_full[pst], pph);
            PROF(5);
            tc_fence_after();
            const uint32_t vbase = sV + pst * C::TB;
            if (elect_one()) {
                if (!DBG64(1)) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16_ts(o_tm, p_tm + kk * 8, sdesc_sw128(vbase + kk * 2048, C::TB, 1024), idO,
                                    (p_first && kk == 0) ? 0u : 1u);
                }
                mma_commit(&uv_empty[pst]);
                mma_commit(upv_done);
                if (p_last) mma_commit(uepi);
            }
            __syncwarp();
            pend = false;
        };
        int4 *uhdr = reinterpret_cast<int4 *>(smem + C::OFF_HDR) + gu * C::QS;
        while (true) {
            mbar_wait(&uq_full[qi], qph);
            const int4 h4 = uhdr[qi];
            const int ut = __shfl_sync(0xffffffffu, h4.x, 0);
            if (ut < 0) break;
            const int uj0 = __shfl_sync(0xffffffffu, h4.z, 0), uj1 = __shfl_sync(0xffffffffu, h4.w, 0);
            const uint32_t qb = sQ + qi * C::TB;
            if (uj0 == uj1) {      // no entries: the epilogue writes zeros
                if (pend) flush_pv();
                if (elect_one()) { mma_commit(uepi); mma_commit(&uq_empty[qi]); }
                __syncwarp();
            }
            for (int j = uj0; j < uj1; ++j) {
                const int st = gent % C::KS;
                const uint32_t ph = (gent / C::KS) & 1;
                const int vs = gent % C::VS;
                const uint32_t vph = (gent / C::VS) & 1;
                ++gent;
                PROF(0);
                mbar_wait(&uk_full[st], ph);
                PROF(1);
                if (scnt > 0) mbar_wait(us_empty, (scnt - 1) & 1);   // softmax has read the previous S
                PROF(2);
                ++scnt;
                tc_fence_after();
                const uint32_t kbase = sK + st * C::TB;
                if (elect_one()) {
                    if (!DBG64(1)) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_bf16_ss(s_tm, sdesc_sw128(qb + kk * 32, 16, 1024), sdesc_sw128(kbase + kk * 32, 16, 1024),
                                        idS, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(us_full);
                    mma_commit(&uk_empty[st]);
                    if (j == uj1 - 1) mma_commit(&uq_empty[qi]);     // the unit's last QK^T: Q slot free
                }
                __syncwarp();
                if (pend) flush_pv();
                pend = true;
                pst = vs;
                pph = vph;
                p_first = j == uj0;
                p_last = j == uj1 - 1;
            }
            if (++qi == C::QS) { qi = 0; qph ^= 1; }
        }
        if (pend) flush_pv();
        PROF(0);
        PROF_FLUSH();
    } else {
        // ------------------------------------------------------------ softmax half-rows of group g
        // register budget: 640 threads x 96 = 61440; warps 0-3 give 4 x 32 x (96 - 40) back, the 16
        // softmax warps take 16 x 32 x (104 - 96) of them
        asm volatile("setmaxnreg.inc.sync.aligned.u32 104;");
        const int quad = warp & 3;              // TMEM lane quadrant of this warp
        const int h = ((warp - 4) >> 2) & 1;    // half of the S row: columns [64 h, 64 h + 64)
        const int r = quad * 32 + lane;         // row within the query tile
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const uint32_t s_tm = tmem + lane_off + g * 128 + 64 * h;
        const uint32_t o_tm = tmem + lane_off + 256 + g * 64 + 32 * h;
        const uint32_t p_tm = tmem + lane_off + 384 + g * 64 + 32 * h;
        const float c2 = prm.scale_log2;
        const uint64_t cc = pack2(c2, c2);
        const uint4 *mring = reinterpret_cast<const uint4 *>(gs + C::OFF_M);
        float *xm = reinterpret_cast<float *>(gs + C::OFF_XM);      // [2][128]
        float *xl = reinterpret_cast<float *>(gs + C::OFF_XL);      // [2][128]
        const int bar_id = 1 + 4 * g + quad;    // named barrier of the two warps of this quadrant
        uint32_t s_cnt = 0, e_cnt = 0;
        int qs = 0, mi = 0;
        uint32_t qph = 0, mph = 0;
        PROF_DECL
        // the deferred epilogue of the previous unit: O / (l_h0 + l_h1) -> bf16 -> HBM
        bool pe_on = false;
        float pe_l = 0.f;
        int pe_t = 0, pe_bh = 0;
        auto epilogue = [&]() {
            PROF(11);
            xl[h * 128 + r] = pe_l;
            named_bar(bar_id, 64);
            const float l = pe_l + xl[(1 - h) * 128 + r];
            named_bar(bar_id, 64);               // both read before xl is rewritten
            mbar_wait(epi, e_cnt & 1);
            ++e_cnt;
            tc_fence_after();
            float o[32];
            tmem_ld32(o_tm, o);
            tmem_wait_ld();
            tc_fence_before();
            const float inv = l > 0.f ? 1.f / l : 0.f;
            const int row = pe_t * 128 + r;
            if (row < prm.N) {
                uint4 *dst = reinterpret_cast<uint4 *>(prm.O + ((size_t)pe_bh * prm.N + row) * 64 + 32 * h);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint4 w;
                    w.x = inv == 0.f ? 0u : pack_bf16(o[8 * c + 0] * inv, o[8 * c + 1] * inv);
                    w.y = inv == 0.f ? 0u : pack_bf16(o[8 * c + 2] * inv, o[8 * c + 3] * inv);
                    w.z = inv == 0.f ? 0u : pack_bf16(o[8 * c + 4] * inv, o[8 * c + 5] * inv);
                    w.w = inv == 0.f ? 0u : pack_bf16(o[8 * c + 6] * inv, o[8 * c + 7] * inv);
                    dst[c] = w;
                }
            }
            pe_on = false;
            PROF(6);
        };
        while (true) {
            mbar_wait(&q_full[qs], qph);            // the unit's header is published
            const int4 h4 = hdr[qs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&q_empty[qs]);   // header read: the slot may be refilled after the unit's QK^T
            if (++qs == C::QS) { qs = 0; qph ^= 1; }
            const int ut = __shfl_sync(0xffffffffu, h4.x, 0);
            if (ut < 0) break;
            const int ubh = h4.y;
            const int j0 = __shfl_sync(0xffffffffu, h4.z, 0), j1 = __shfl_sync(0xffffffffu, h4.w, 0);
            float m_ref = -INFINITY, l_run = 0.f;
            for (int j = j0; j < j1; ++j) {
                const bool first = j == j0;
                // ---- entry metadata: this half's chunk bits (uniform) and the row's mask words
                PROF(11);
                mbar_wait(&m_full[mi], mph);
                const uint32_t bits = __shfl_sync(0xffffffffu, ebits[mi], 0);
                const uint32_t live = (bits >> (4 * quad + 2 * h)) & 3u;
                const uint32_t need = live & ~(bits >> (16 + 4 * quad + 2 * h));
                uint2 mw = make_uint2(~0u, ~0u);
                if (need) {
                    const uint4 m4 = mring[mi * 128 + r];
                    mw = h ? make_uint2(m4.z, m4.w) : make_uint2(m4.x, m4.y);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&m_empty[mi]);
                if (++mi == C::MS) { mi = 0; mph ^= 1; }
                // ---- S half-row -> registers; S goes back to the MMA warp
                PROF(0);
                mbar_wait(s_full, s_cnt & 1);
                ++s_cnt;
                PROF(1);
                tc_fence_after();
                float sv[64];
                tmem_ld32(s_tm, sv);
                tmem_ld32(s_tm + 32, sv + 32);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(s_empty);
                PROF(2);
                // ---- mask, half max, exchange with the other half of the row
                float hm = -INFINITY;
                if (live & 1u) {
                    if (need & 1u) apply_mask(sv, mw.x);
                    hm = max32(sv);
                }
                if (live & 2u) {
                    if (need & 2u) apply_mask(sv + 32, mw.y);
                    hm = fmaxf(hm, max32(sv + 32));
                }
                PROF(3);
                xm[((s_cnt & 1) * 2 + h) * 128 + r] = hm;
                named_bar(bar_id, 64);
                const float mx = fmaxf(hm, xm[((s_cnt & 1) * 2 + 1 - h) * 128 + r]) * c2;
                PROF(4);
                float alpha = 1.f;
                bool resc = false;
                if (mx > m_ref + kBump) {
                    if (m_ref != -INFINITY) {
                        alpha = ex2(m_ref - mx);
                        resc = true;
                    }
                    m_ref = mx;
                    l_run *= alpha;
                }
                const float mref = m_ref == -INFINITY ? 0.f : m_ref;
                const uint64_t mm = pack2(-mref, -mref);
                // ---- exponentials of the live chunks
                uint64_t acc0 = pack2(0.f, 0.f), acc1 = acc0;
                uint32_t pw[32];
                if (live == 3u && !DBG64(2)) {
                    exp32<SPLAT_NEMU64>(sv, cc, mm, acc0, acc1, pw);
                    exp32<SPLAT_NEMU64>(sv + 32, cc, mm, acc0, acc1, pw + 16);
                } else if (live && !DBG64(2)) {
                    // one live chunk: compute it once, place the packed P by chunk
                    if (live & 2u) {
#pragma unroll
                        for (int x = 0; x < 32; ++x) sv[x] = sv[32 + x];
                    }
                    uint32_t pq[16];
                    exp32<SPLAT_NEMU64>(sv, cc, mm, acc0, acc1, pq);
#pragma unroll
                    for (int x = 0; x < 16; ++x) {
                        pw[x] = (live & 1u) ? pq[x] : 0u;
                        pw[16 + x] = (live & 1u) ? 0u : pq[x];
                    }
                } else {
#pragma unroll
                    for (int x = 0; x < 32; ++x) pw[x] = 0u;
                }
                PROF(5);
                // the previous unit's epilogue, in the shadow of this unit's first tile (this tile's P
                // -- and with it the unit's first PV, which overwrites O -- comes after it)
                if (first && pe_on) epilogue();
                // ---- the previous PV has read P (and O is final for it)
                if (s_cnt > 1) {
                    mbar_wait(pv_done, (s_cnt - 2) & 1);
                    tc_fence_after();
                }
                PROF(7);
                if (!first && __any_sync(0xffffffffu, resc)) {
                    float o[32];
                    tmem_ld32(o_tm, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int x = 0; x < 32; ++x) o[x] *= alpha;
                    tmem_st32(o_tm, o);
                }
                PROF(8);
                tmem_st32(p_tm, reinterpret_cast<const float *>(pw));
                {
                    float a, b, c, d;
                    unpack2(acc0, a, b);
                    unpack2(acc1, c, d);
                    l_run += (a + b) + (c + d);
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full);
                PROF(9);
            }
            if (pe_on) epilogue();       // empty unit: the previous unit's epilogue was not deferred into a tile
            pe_on = true;
            pe_l = j0 == j1 ? 0.f : l_run;
            pe_t = ut;
            pe_bh = ubh;
        }
        if (pe_on) epilogue();
        PROF(11);
        PROF_FLUSH();
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
    // the last CTA to finish resets the slot's work counter for the next launch (every grab of
    // every CTA happened before its increment of the done counter)
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(prm.sched + 1, 1ull) == (unsigned long long)gridDim.x - 1ull) {
            prm.sched[0] = 0ull;
            prm.sched[1] = 0ull;
            __threadfence();
        }
    }
}

}  // namespace

#ifdef SPLAT_FUSED_PROF
extern "C" int splat_debug_prof64(unsigned long long *out)
{
    cudaMemcpyFromSymbol(out, g_prof64, sizeof(g_prof64));
    static const unsigned long long z[20 * 16] = {};
    cudaMemcpyToSymbol(g_prof64, z, sizeof(z));
    return 0;
}
#endif

cudaError_t launch_mhsa64(const DevAcsr &A, const void *Q, const void *K, const void *V, int BH, float scale,
                          void *O, cudaStream_t st)
{
    if (A.n_ksplit > 0) return cudaErrorNotSupported;   // split-K units: the split kernel only
    CUtensorMap mq, mk, mv;
    if (!make_map(&mq, Q, BH, A.n, 64) || !make_map(&mk, K, BH, A.n, 64) || !make_map(&mv, V, BH, A.n, 64))
        return cudaErrorInvalidValue;
    if (!A.sched) return cudaErrorInvalidValue;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(mhsa64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, H64::SMEM);
        if (e != cudaSuccess) return e;
        attr_set[dev & 63] = true;
    }
    P64 p{};
    p.A = A;
    p.BH = BH;
    p.N = A.n;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.O = reinterpret_cast<__nv_bfloat16 *>(O);
    p.sched = A.sched;
    static const int dbg = diag_env("SPLAT_TC_DEBUG");
    p.dbg = dbg;
    const long long units = (long long)A.n_qt * BH;
    const long long ctas = (units + 1) / 2;
    const int grid = (int)(ctas < num_sms(dev) ? ctas : num_sms(dev));
    mhsa64_kernel<<<grid, kThreads64, H64::SMEM, st>>>(mq, mk, mv, p);
    return cudaGetLastError();
}

}  // namespace splat
#endif  // SPLAT_DIAG
