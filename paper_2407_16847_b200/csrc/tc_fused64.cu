// tc_fused64.cu -- fused sparse MHSA for d = 64 on sm_100a.
//
// O = softmax(M (x) scale*Q K^T) V per (b, h) (PAPER Eq. 1; softmax over each row's
// non-zeros, reading R-1 of DESIGN.md), S and P never leave the SM.  Work unit: one 128-row query
// tile of one (b, h) against its plan entries (key tiles touched by any of its rows -- the span of
// P:573 at tile granularity), handed out dynamically from a per-call work counter.
//
// Each CTA runs two independent tile groups g = 0, 1 (one query tile each):
//   warp 0 / 3  : producer of group g -- Q (TMA), per entry: K (TMA), the entry's chunk bits and,
//                 for a PARTIAL entry, its 128 row masks (2 KB bulk copy) into a mask ring, V one
//                 entry behind K.
//   warp 1 / 2  : MMA issuer of group g -- S = Q K^T (SS, N = 128), O += P V (TS, P from TMEM).
//   warps 4-7 / 8-11 : softmax of group g, thread = query row = TMEM lane.
//
// The softmax is a streaming pass over the S row: chunks 0-1 are loaded, chunks 2-3 are loaded
// while 0-1 are exponentiated, and exponentials use a per-row reference m_ref that only moves when
// a chunk's max exceeds it by more than kBump (log2 units): the max of each chunk is compared, not
// waited for, so no chunk waits for the whole row.  Moving the reference rescales what was already
// accumulated with that reference (the running sum, this tile's packed P, and O before the next
// PV) -- exact in exact arithmetic, so the output is the same softmax (Eq. 1).  exp2 with log2(e)
// folded into the scale runs on MUFU for most columns and on the FMA pipe (degree-3 polynomial)
// for the rest.  Every per-entry decision (live / masked 32-column chunks of the warp) comes from
// shared memory and is warp-uniform, so the chunk loop has no divergent branches.
//
// TMEM (512 columns): S_g [128 g, 128 g + 128), O_g [256 + 64 g, +64), P_g [384 + 64 g, +64).
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

constexpr int kThreads64 = 384;
constexpr float kBump = 8.0f;        // reference moves when a chunk max exceeds it by > 2^8

#ifndef SPLAT_NEMU64
#define SPLAT_NEMU64 8               // exponentials of each 32-column chunk emulated on the FMA pipe
#endif

struct F64 {
    static constexpr int QS = 2, KS = 2, MS = 4;
    static constexpr int TB = 128 * 128;                         // 16 KB: 128 rows x 64 bf16
    static constexpr int MB = 128 * 16;                          // 2 KB: 128 row masks of 128 bits
    static constexpr int OFF_Q = 0, OFF_K = QS * TB, OFF_V = OFF_K + KS * TB, OFF_M = OFF_V + KS * TB;
    static constexpr int GROUP = OFF_M + MS * MB;                // 104 KB per group
    static constexpr int OFF_BAR = 2 * GROUP;
    // per group: q_full[QS] q_empty[QS] k_full[KS] k_empty[KS] v_full[KS] v_empty[KS] m_full[MS] m_empty[MS]
    //            s_full s_empty p_full pv_done epi
    static constexpr int NB = 2 * QS + 4 * KS + 2 * MS + 5;
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

// exp2(s * c - m) of one 32-column chunk -> 16 packed bf16 pairs, row-sum partials in acc0 / acc1
__device__ __forceinline__ void exp_chunk(const float *v, uint64_t cc, uint64_t mm, uint64_t &acc0, uint64_t &acc1,
                                          uint32_t *pw)
{
    exp32<SPLAT_NEMU64>(v, cc, mm, acc0, acc1, pw);
}

// p *= a for 16 packed bf16 pairs (reference moved after they were computed)
__device__ __forceinline__ void rescale_pw(uint32_t *pw, float a)
{
#pragma unroll
    for (int x = 0; x < 16; ++x) {
        const float lo = __uint_as_float(pw[x] << 16), hi = __uint_as_float(pw[x] & 0xffff0000u);
        pw[x] = pack_bf16(lo * a, hi * a);
    }
}

#define DBG64(m) (kDiag && (prm.dbg & (m)))

__global__ void __launch_bounds__(kThreads64, 1)
mhsa64_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, const P64 prm)
{
    using C = F64;
    extern __shared__ __align__(1024) uint8_t smem[];
    if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0u) __trap();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = warp >= 4 ? (warp - 4) >> 2 : (warp == 0 || warp == 1 ? 0 : 1);
    uint8_t *gs = smem + g * C::GROUP;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR) + g * C::NB;
    uint64_t *q_full = bars, *q_empty = q_full + C::QS;
    uint64_t *k_full = q_empty + C::QS, *k_empty = k_full + C::KS;
    uint64_t *v_full = k_empty + C::KS, *v_empty = v_full + C::KS;
    uint64_t *m_full = v_empty + C::KS, *m_empty = m_full + C::MS;
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
            for (int i = 0; i < 2 * C::QS + 4 * C::KS; ++i) mbar_init(&b[o++], 1);
            for (int i = 0; i < C::MS; ++i) mbar_init(&b[o++], 1);   // m_full (producer)
            for (int i = 0; i < C::MS; ++i) mbar_init(&b[o++], 4);   // m_empty (4 softmax warps)
            mbar_init(&b[o++], 1);   // s_full  (MMA commit)
            mbar_init(&b[o++], 4);   // s_empty (4 softmax warps)
            mbar_init(&b[o++], 4);   // p_full  (4 softmax warps)
            mbar_init(&b[o++], 1);   // pv_done (MMA commit)
            mbar_init(&b[o++], 1);   // epi     (MMA commit)
        }
        fence_mbar_init();
        tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 || warp == 3) {
        // ------------------------------------------------------------ producer of group g
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        int qi = 0, qc = 0, ki = 0, kc = 0, vi = 0, vc = 0, mi = 0, mc = 0;
        uint32_t qph = 0, kph = 0, vph = 0, mph = 0;
        bool pv = false;            // V of the previous entry still to load
        int pv_kv = 0, pv_bh = 0;
        auto load_v = [&]() {
            if (vc >= C::KS) mbar_wait(&v_empty[vi], vph ^ 1);
            if (lane == 0) {
                mbar_expect_tx(&v_full[vi], C::TB);
                tma_load_3d(gs + C::OFF_V + vi * C::TB, &tmV, &v_full[vi], 0, pv_kv * 128, pv_bh);
            }
            ++vc;
            if (++vi == C::KS) { vi = 0; vph ^= 1; }
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
                // entry metadata: chunk bits, and the row masks where some warp has a masked chunk
                if (mc >= C::MS) mbar_wait(&m_empty[mi], mph ^ 1);
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
                if (kc >= C::KS) mbar_wait(&k_empty[ki], kph ^ 1);
                if (lane == 0) {
                    mbar_expect_tx(&k_full[ki], C::TB);
                    tma_load_3d(gs + C::OFF_K + ki * C::TB, &tmK, &k_full[ki], 0, kv * 128, un.bh);
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
    } else if (warp == 1 || warp == 2) {
        // ------------------------------------------------------------ MMA issuer of group g
        // every operand warp-uniform (shfl from lane 0), issue under elect.sync: the UMMA
        // descriptors stay in uniform registers and UTCHMMAs issue back to back
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        const int gu = __shfl_sync(0xffffffffu, g, 0);
        const uint32_t tmu = __shfl_sync(0xffffffffu, tmem, 0);
        uint8_t *gsu = smem + gu * C::GROUP;
        uint64_t *bu = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR) + gu * C::NB;
        uint64_t *uq_full = bu, *uq_empty = uq_full + C::QS, *uk_full = uq_empty + C::QS, *uk_empty = uk_full + C::KS;
        uint64_t *uv_full = uk_empty + C::KS, *uv_empty = uv_full + C::KS;
        uint64_t *us_full = uv_empty + C::KS + 2 * C::MS, *us_empty = us_full + 1, *up_full = us_empty + 1;
        uint64_t *upv_done = up_full + 1, *uepi = upv_done + 1;
        constexpr uint32_t idS = idesc_bf16(128, 128, false);
        constexpr uint32_t idO = idesc_bf16(128, 64, true);
        const uint32_t sQ = smem_u32(gsu + C::OFF_Q), sK = smem_u32(gsu + C::OFF_K), sV = smem_u32(gsu + C::OFF_V);
        const uint32_t s_tm = tmu + gu * 128, o_tm = tmu + 256 + gu * 64, p_tm = tmu + 384 + gu * 64;
        int qi = 0;
        uint32_t qph = 0, pcnt = 0, scnt = 0, gent = 0;
        bool pend = false, p_first = false, p_last = false;
        int pst = 0, pq = 0;
        uint32_t pph = 0;
        auto flush_pv = [&]() {
            mbar_wait(up_full, pcnt & 1);
            ++pcnt;
            mbar_wait(&uv_full[pst], pph);
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
                if (p_last) {
                    mma_commit(uepi);
                    mma_commit(&uq_empty[pq]);
                }
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
                ++gent;
                mbar_wait(&uk_full[st], ph);
                if (scnt > 0) mbar_wait(us_empty, (scnt - 1) & 1);   // softmax has read the previous S
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
                }
                __syncwarp();
                if (pend) flush_pv();
                pend = true;
                pst = st;
                pph = ph;
                p_first = j == uj0;
                p_last = j == uj1 - 1;
                pq = qi;
            }
            if (++qi == C::QS) { qi = 0; qph ^= 1; }
        }
        if (pend) flush_pv();
    } else {
        // ------------------------------------------------------------ softmax warps of group g
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
        const int quad = warp & 3;              // TMEM lane quadrant of this warp
        const int r = quad * 32 + lane;         // row within the query tile
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const uint32_t s_tm = tmem + lane_off + g * 128;
        const uint32_t o_tm = tmem + lane_off + 256 + g * 64;
        const uint32_t p_tm = tmem + lane_off + 384 + g * 64;
        const float c2 = prm.scale_log2;
        const uint64_t cc = pack2(c2, c2);
        const uint4 *mring = reinterpret_cast<const uint4 *>(gs + C::OFF_M);
        uint32_t s_cnt = 0, e_cnt = 0;
        // O / l -> bf16 -> the thread's output row (8 x 16-byte stores)
        auto epilogue = [&](float l, int t, int bh) {
            mbar_wait(epi, e_cnt & 1);
            ++e_cnt;
            tc_fence_after();
            const float inv = l > 0.f ? 1.f / l : 0.f;
            float o[64];
            tmem_ld32(o_tm, o);
            tmem_ld32(o_tm + 32, o + 32);
            tmem_wait_ld();
            tc_fence_before();
            const int row = t * 128 + r;
            if (row < prm.N) {
                uint4 *dst = reinterpret_cast<uint4 *>(prm.O + ((size_t)bh * prm.N + row) * 64);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    uint4 w;
                    w.x = pack_bf16(o[8 * c + 0] * inv, o[8 * c + 1] * inv);
                    w.y = pack_bf16(o[8 * c + 2] * inv, o[8 * c + 3] * inv);
                    w.z = pack_bf16(o[8 * c + 4] * inv, o[8 * c + 5] * inv);
                    w.w = pack_bf16(o[8 * c + 6] * inv, o[8 * c + 7] * inv);
                    dst[c] = w;
                }
            }
        };
        bool pe_on = false;          // deferred epilogue of the previous unit
        float pe_l = 0.f;
        int pe_t = 0, pe_bh = 0;
        int qs = 0, mi = 0;
        uint32_t qph = 0, mph = 0;
        while (true) {
            mbar_wait(&q_full[qs], qph);            // the unit's header is published
            const int4 h4 = hdr[qs];
            if (++qs == C::QS) { qs = 0; qph ^= 1; }
            const int ut = __shfl_sync(0xffffffffu, h4.x, 0);
            if (ut < 0) break;
            const int ubh = h4.y;
            const int j0 = __shfl_sync(0xffffffffu, h4.z, 0), j1 = __shfl_sync(0xffffffffu, h4.w, 0);
            if (j0 == j1) {
                if (pe_on) { epilogue(pe_l, pe_t, pe_bh); pe_on = false; }
                epilogue(0.f, ut, ubh);
                continue;
            }
            float m_ref = -INFINITY, l_run = 0.f;
            for (int j = j0; j < j1; ++j) {
                const bool first = j == j0;
                // ---- entry metadata: chunk bits (uniform) and this row's mask words
                mbar_wait(&m_full[mi], mph);
                const uint32_t bits = __shfl_sync(0xffffffffu, ebits[mi], 0);
                const uint32_t live = (bits >> (4 * quad)) & 0xFu;
                const uint32_t need = live & ~(bits >> (16 + 4 * quad));
                uint4 m4 = make_uint4(~0u, ~0u, ~0u, ~0u);
                if (need) m4 = mring[mi * 128 + r];
                __syncwarp();
                if (lane == 0) mbar_arrive(&m_empty[mi]);
                if (++mi == C::MS) { mi = 0; mph ^= 1; }
                const uint32_t mk[4] = {m4.x, m4.y, m4.z, m4.w};
                // ---- S row -> registers (live chunks only), then S goes back to the MMA warp
                mbar_wait(s_full, s_cnt & 1);
                ++s_cnt;
                tc_fence_after();
                float sv[128];
                tmem_ld32(s_tm, sv);
                tmem_ld32(s_tm + 32, sv + 32);
                tmem_ld32(s_tm + 64, sv + 64);
                tmem_ld32(s_tm + 96, sv + 96);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(s_empty);   // the next QK^T may overwrite S
                // ---- streaming exponentials, chunk by chunk against the running reference
                uint64_t acc0 = pack2(0.f, 0.f), acc1 = acc0;
                uint32_t pw[64];
                float a_tile = 1.f;          // product of this tile's reference moves (O rescale)
                float a_late = 1.f;          // ... of the moves after P[0, 32) was stored
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float *v = sv + 32 * c;
                    if (!(live & (1u << c))) {
#pragma unroll
                        for (int x = 0; x < 16; ++x) pw[16 * c + x] = 0u;
                    } else {
                        if (need & (1u << c)) apply_mask(v, mk[c]);
                        const float cm = max32(v) * c2;
                        const bool up = cm > m_ref + kBump;
                        if (__any_sync(0xffffffffu, up)) {
                            // move the reference: rescale what was computed against the old one
                            const float mn = up ? cm : m_ref;
                            const float a = up ? (m_ref == -INFINITY ? 0.f : ex2(m_ref - mn)) : 1.f;
                            m_ref = mn;
                            l_run *= a;
                            a_tile *= a;
                            acc0 = ffma2(acc0, pack2(a, a), pack2(0.f, 0.f));
                            acc1 = ffma2(acc1, pack2(a, a), pack2(0.f, 0.f));
                            if (c >= 2) {
                                a_late *= a;
#pragma unroll
                                for (int cp = 2; cp < c; ++cp) rescale_pw(pw + 16 * cp, a);
                            } else {
#pragma unroll
                                for (int cp = 0; cp < c; ++cp) rescale_pw(pw + 16 * cp, a);
                            }
                        }
                        const float mref = m_ref == -INFINITY ? 0.f : m_ref;
                        if (DBG64(2)) {
#pragma unroll
                            for (int x = 0; x < 16; ++x) pw[16 * c + x] = 0u;
                        } else {
                            exp_chunk(v, cc, pack2(-mref, -mref), acc0, acc1, pw + 16 * c);
                        }
                    }
                    if (c == 1) {
                        // first half of P: after the previous PV has read P (and O is final for it)
                        if (s_cnt > 1) {
                            mbar_wait(pv_done, (s_cnt - 2) & 1);
                            tc_fence_after();
                        }
                        tmem_st32(p_tm, reinterpret_cast<const float *>(pw));
                    }
                }
                if (__any_sync(0xffffffffu, a_late != 1.f)) {
                    // the reference moved after P[0, 32) was stored: rescale it in TMEM (rare)
                    tmem_wait_st();
                    float t32[32];
                    tmem_ld32(p_tm, t32);
                    tmem_wait_ld();
                    uint32_t *w = reinterpret_cast<uint32_t *>(t32);
                    rescale_pw(w, a_late);
                    rescale_pw(w + 16, a_late);
                    tmem_st32(p_tm, t32);
                }
                if (!first && __any_sync(0xffffffffu, a_tile != 1.f)) {
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        float o[32];
                        tmem_ld32(o_tm + c * 32, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int x = 0; x < 32; ++x) o[x] *= a_tile;
                        tmem_st32(o_tm + c * 32, o);
                    }
                }
                tmem_st32(p_tm + 32, reinterpret_cast<const float *>(pw + 32));
                {
                    float a, b, c, d;
                    unpack2(acc0, a, b);
                    unpack2(acc1, c, d);
                    l_run += (a + b) + (c + d);
                }
                if (first && pe_on) {        // the previous unit's epilogue (its last PV is long complete)
                    epilogue(pe_l, pe_t, pe_bh);
                    pe_on = false;
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full);
            }
            pe_on = true;
            pe_l = l_run;
            pe_t = ut;
            pe_bh = ubh;
        }
        if (pe_on) epilogue(pe_l, pe_t, pe_bh);
    }
    __syncthreads();
    if (warp == 1) {
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

cudaError_t launch_mhsa64(const DevAcsr &A, const void *Q, const void *K, const void *V, int BH, float scale,
                          void *O, cudaStream_t st)
{
    CUtensorMap mq, mk, mv;
    if (!make_map(&mq, Q, BH, A.n, 64) || !make_map(&mk, K, BH, A.n, 64) || !make_map(&mv, V, BH, A.n, 64))
        return cudaErrorInvalidValue;
    if (!A.sched) return cudaErrorInvalidValue;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(mhsa64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F64::SMEM);
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
    mhsa64_kernel<<<grid, kThreads64, F64::SMEM, st>>>(mq, mk, mv, p);
    return cudaGetLastError();
}

}  // namespace splat
