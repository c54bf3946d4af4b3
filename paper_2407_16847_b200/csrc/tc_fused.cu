// tc_fused.cu -- fused sparse MHSA on sm_100a tensor cores.
//
// Computes O = softmax(M (x) scale*Q K^T) V per (b, h) (PAPER Eq. 1)
// without writing S or P to HBM.  The paper launches R-SDDMM, softmax and
// R-SpMM as separate kernels with HBM buffers in between (Listing 4,
// P:700-711); here one persistent kernel walks the tile plan (plan.cpp).
//
//   work unit : (b*H+h, pair of adjacent 128-row query tiles A = 2p, B = 2p+1),
//               processed against the UNION of the two key-tile lists (span
//               specialisation, at tile granularity), so one K/V load
//               serves both tiles.  Units are walked in cost buckets, longest
//               first, head-major inside a bucket (K/V of a head stay in L2).
//   warp 0    : TMA producer -- Q_A, Q_B, then K_e, V_e of every union entry e
//               into 128B-swizzled SMEM rings (3-D tensor maps [BH, N, d],
//               out-of-range rows zero-filled).
//   warp 1    : tcgen05.mma issuer (one thread).  Per entry e and tile g that
//               uses it: O_g += P_g(prev) V_prev (A operand P from TMEM, V an
//               MN-major SMEM operand), then S_g = Q_g K_e^T (both K-major,
//               M=128 N=128 K=16 steps, fp32 accumulator in TMEM).
//   warps 4-7 / 8-11 : softmax of tile A / tile B (ping-pong: one group's
//               exponentials overlap the other group's MMAs).  Thread = query
//               row = TMEM lane.  tcgen05.ld S -> fast-index mask on PARTIAL
//               entries (reading A-7: column c of run (start, step, count) iff
//               (c-start) % step == 0 and 0 <= (c-start)/step < count),
//               fully-masked 32-column chunks skip the exponentials -> running
//               max (FMNMX3), exp2 with log2(e) folded into the scale (FFMA2 +
//               MUFU.EX2), row sum (FADD2) -> P as packed bf16 written back over
//               S in TMEM (tcgen05.st).  O is rescaled in TMEM only when the
//               running max grows by more than 2^8 (stale-max trick).
//   epilogue  : O / l -> bf16 -> HBM.
//
// TMEM (512 columns): S_A [0,128), S_B [128,256), O_A [256,256+d), O_B [256+d, 256+2d).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "kernels.h"
#include "sm100.cuh"
#include "softmax_math.cuh"

namespace splat {
namespace {

using namespace sm100;

constexpr int kThreads = 384;            // WG0: warp 0 TMA, warp 1 MMA; WG1: softmax A; WG2: softmax B
constexpr int kTileBytes64 = 128 * 128;  // [128 rows x 64 bf16] swizzle-128B sub-tile (16 KB)
constexpr float kRescaleThresh = 8.0f;   // log2 units

template <int D>
struct Cfg {
    static constexpr int kChunks = D / 64;
    static constexpr int kTileBytes = kChunks * kTileBytes64;
    static constexpr int QS = D == 64 ? 2 : 1;   // Q buffers per tile group
    static constexpr int KS = D == 64 ? 4 : 2;   // K and V ring depth
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + 2 * QS * kTileBytes;
    static constexpr int OFF_V = OFF_K + KS * kTileBytes;
    static constexpr int OFF_O = OFF_V + KS * kTileBytes;          // O staging: one 64-column sub-tile per group
    static constexpr int OFF_BAR = OFF_O + 2 * kTileBytes64;
    static constexpr int NBAR = 4 * QS + 4 * KS + 10;
    // SEP (d = 64): P gets its own TMEM columns (S 2x128 + O 2x64 + P 2x64 = 512), so S is released
    // as soon as the softmax has loaded it and the next S = Q K^T overlaps the exponentials.
    // d = 128 (S 2x128 + O 2x128 = 512): P overwrites S and the next S waits for the PV.
    static constexpr bool SEP = D == 64;
    static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
};

struct Params {
    DevAcsr A;
    int BH, N;
    float scale_log2;
    __nv_bfloat16 *O;
    int dbg;        // profiling aid only (SPLAT_TC_DEBUG): 1 = no MMAs issued, 2 = no softmax math
    // residue decomposition (splat_acsr_s::sub_band), paired kernel only:
    //   pass 1 (view = 1): tiles are residue-major (4-D maps, R residues x nk rows); the epilogue
    //                      stores O_s / l_s to the natural rows of O and lse2 = m + log2(l) to lse
    //   pass 2 (merge = 1): natural band tiles; the epilogue merges with O_s (read from O) and lse
    //   plain STRIDED (view = 1, lse = null): the only pass; the epilogue stores O / l directly
    int view, merge, rv_R, rv_nk, rv_l;
    int rv_sh;                   // log2(rv_nk) (a power of two: nk | 128 or 128 | nk)
    float *lse;
    unsigned long long *sched;   // split kernel: [work counter, done counter], zero between launches
    // one-launch residue decomposition (VM = 2): the plan is the strided pass's pairs [0, mix_u1)
    // followed by the band pass's [mix_u1, mix_u1 + mix_u2); units run head-interleaved with a lag of
    // mix_lag heads (fetch_unit_mixed); dep[bh] counts the strided-pass tiles of head bh whose O_s and
    // lse are in memory (dep_target = all of them), dep[kLseHeads] the CTAs done (the last resets all)
    int mix_u1, mix_u2, mix_lag, dep_target;
    unsigned *dep;
};

// Profiling knobs (SPLAT_TC_DEBUG) exist only in the diagnostics build (libsplat_diag.so); in the
// product build DBG() is a compile-time 0.
#define DBG(m) (kDiag && (prm.dbg & (m)))

#if defined(SPLAT_TRACE) && !defined(SPLAT_DIAG)
#error "SPLAT_TRACE needs the diagnostics build (-DSPLAT_DIAG)"
#endif
#if defined(SPLAT_FUSED_PROF) && !defined(SPLAT_DIAG)
#error "SPLAT_FUSED_PROF needs the diagnostics build (-DSPLAT_DIAG)"
#endif
#if (defined(SPLAT_X_NOMAX) || defined(SPLAT_X_NOSUM) || defined(SPLAT_X_DEPNOW)) && !defined(SPLAT_DIAG)
#error "ablation macros need the diagnostics build (-DSPLAT_DIAG)"
#endif
#ifdef SPLAT_DIAG
// Profiling aid (SPLAT_TC_DEBUG & 4): clock64 timestamps of pipeline events in CTA 0.
__device__ unsigned long long g_trace[6][2048];
__device__ int g_trace_n[6];
#endif
#ifdef SPLAT_TRACE
// per-role event counter lives in a register (tr_n, declared at the top of the kernel)
#define TRACE(R, TAG)                                                                                    \
    do {                                                                                                 \
        if (DBG(4) && blockIdx.x == 0) {                                                          \
            if (tr_n < 2048) g_trace[R][tr_n] = ((unsigned long long)(TAG) << 48) | (clock64() & 0xffffffffffffull); \
            ++tr_n;                                                                                      \
            g_trace_n[R] = tr_n;                                                                         \
        }                                                                                                \
    } while (0)
#else
#define TRACE(R, TAG) do { } while (0)
#endif

// Per-unit metadata, fetched one unit ahead so the dependent global loads never sit on the
// critical path of a role.
struct UnitInfo {
    int pair, bh, e0, e1;
    int j0[3];      // the two query tiles' own entry ranges: tile g owns [j0[g], j0[g+1])
    int pass;       // VM = 2: 1 = strided pass (residue-major views), 0 = band pass (natural, merge)
};

__device__ __forceinline__ UnitInfo fetch_unit(const DevAcsr &A, int BH, int u)
{
    // bucket arithmetic on kernel parameters, then a single (independent) load
    int k = 0, bh = 0;
    for (int b = 0; b < A.n_buckets; ++b) {
        const int nb = A.bucket_start[b + 1] - A.bucket_start[b];
        const int ub = nb * BH;
        if (u < ub) {
            bh = u / nb;
            k = A.bucket_start[b] + u % nb;
            break;
        }
        u -= ub;
    }
    const int4 info = A.pair_info[2 * k], info2 = A.pair_info[2 * k + 1];
    UnitInfo x;
    x.pair = info.x;
    x.bh = bh;
    x.e0 = info.y;
    x.e1 = info.z;
    x.j0[0] = info.w;
    x.j0[1] = info2.x;
    x.j0[2] = info2.y;
    x.pass = 0;
    return x;
}

// One-launch residue decomposition: unit u of the head-interleaved sequence.  Block s of the
// sequence holds the strided-pass pairs of head s (s < BH) followed by the band-pass pairs of head
// s - lag (s >= lag), so a band unit of head h is issued about lag heads' worth of units after the
// strided units it depends on (their O_s / lse are then normally complete and still in L2).
__device__ __forceinline__ UnitInfo fetch_unit_mixed(const DevAcsr &A, int BH, int U1, int U2, int lag, int u)
{
    const int lc = lag < BH ? lag : BH;
    int bh, k, pass;
    if (u < lc * U1) {
        bh = u / U1; k = u % U1; pass = 1;
    } else {
        const int v = u - lc * U1, blk = U1 + U2;
        if (v < (BH - lc) * blk) {
            const int s = lc + v / blk, w = v % blk;
            if (w < U1) { bh = s; k = w; pass = 1; }
            else { bh = s - lag; k = w - U1; pass = 0; }
        } else {
            const int v2 = v - (BH - lc) * blk;
            bh = BH - lc + v2 / U2; k = v2 % U2; pass = 0;
        }
    }
    const int kk = pass ? k : U1 + k;
    const int4 info = A.pair_info[2 * kk], info2 = A.pair_info[2 * kk + 1];
    UnitInfo x;
    x.pair = info.x;
    x.bh = bh;
    x.e0 = info.y;
    x.e1 = info.z;
    x.j0[0] = info.w;
    x.j0[1] = info2.x;
    x.j0[2] = info2.y;
    x.pass = pass;
    return x;
}

// A query tile's own plan entries (softmax warps): lane l caches mask id and chunk bits of
// entries j0 + l + 32k, k < 2 (beyond 64 entries: global loads).
struct TileRegs {
    int m[2];
    uint32_t b[2];
};

__device__ __forceinline__ void load_tile(const DevAcsr &A, int j0, int j1, int lane, TileRegs &tr)
{
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int j = j0 + lane + 32 * k;
        tr.m[k] = j < j1 ? A.kv_mask[j] : -1;
        tr.b[k] = j < j1 ? A.qt_bits[j] : 0u;
    }
}

__device__ __forceinline__ void tile_at(const DevAcsr &A, const TileRegs &tr, int j0, int j, int &mid, uint32_t &bits)
{
    const int i = j - j0;
    if (i < 64) {
        mid = __shfl_sync(0xffffffffu, i < 32 ? tr.m[0] : tr.m[1], i & 31);
        bits = __shfl_sync(0xffffffffu, i < 32 ? tr.b[0] : tr.b[1], i & 31);
    } else {
        mid = A.kv_mask[j];
        bits = A.qt_bits[j];
    }
}

// Column mask of row r for entry j (all ones where the warp's chunks need no masking).
__device__ __forceinline__ uint4 fetch_mask(const DevAcsr &A, const TileRegs &tr, int j0, int j, int quad, int r)
{
    int mid;
    uint32_t bits;
    tile_at(A, tr, j0, j, mid, bits);
    const uint32_t need = (bits >> (4 * quad)) & ~(bits >> (16 + 4 * quad)) & 0xFu;
    uint4 m = make_uint4(~0u, ~0u, ~0u, ~0u);
    if (need && mid >= 0) m = A.masks[(size_t)mid * 128 + r];
    return m;
}

// The unit's plan entries cached in the registers of a (uniformly executing) warp: lane l
// holds entries e0 + l + 32k, k < 4; ent_at() broadcasts with a shuffle (beyond 128 entries it
// falls back to a global load).
struct EntRegs {
    int r[4];
};

__device__ __forceinline__ void load_ents(const DevAcsr &A, const UnitInfo &un, int lane, EntRegs &er)
{
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int idx = un.e0 + lane + 32 * k;
        er.r[k] = idx < un.e1 ? A.pair_ent[idx] : 0;
    }
}

__device__ __forceinline__ int ent_at(const DevAcsr &A, const UnitInfo &un, const EntRegs &er, int e)
{
    const int i = e - un.e0;
    if (i < 128) {
        const int k = i >> 5;
        const int v = k == 0 ? er.r[0] : (k == 1 ? er.r[1] : (k == 2 ? er.r[2] : er.r[3]));
        return __shfl_sync(0xffffffffu, v, i & 31);
    }
    return A.pair_ent[e];
}

using namespace smx;

// VM (view mode): 0 = natural order; 1 = residue-major 4-D views (strided-row residue pass, permuted
// plain STRIDED); 2 = one-launch residue decomposition -- strided-pass units on the views tmQ..tmO,
// band-pass units on the natural maps tmQ2..tmO2 (unused otherwise).  Separate instantiations, so
// the natural-order kernel carries none of the view arithmetic.
template <int D, int VM>
__global__ void __launch_bounds__(kThreads, 1)
mhsa_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
               const __grid_constant__ CUtensorMap tmQ2, const __grid_constant__ CUtensorMap tmK2,
               const __grid_constant__ CUtensorMap tmV2, const __grid_constant__ CUtensorMap tmO2, const Params prm)
{
    constexpr bool VIEW = VM == 1;
#define SPLAT_FETCH(u_) (VM == 2 ? fetch_unit_mixed(A, prm.BH, prm.mix_u1, prm.mix_u2, prm.mix_lag, (u_)) \
                                 : fetch_unit(A, prm.BH, (u_)))
    using C = Cfg<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // No static shared memory precedes the dynamic buffer, so it starts 1024-byte aligned (checked;
    // the launch still reserves 1 KB of slack).  Using smem_raw itself -- not an integer align-up --
    // keeps the shared state space visible to the compiler (LDS/STS, constant offsets).
    uint8_t *smem = smem_raw;
    if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u) != 0u) __trap();
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *q_full = bars;                     // [2][QS]
    uint64_t *q_empty = q_full + 2 * C::QS;      // [2][QS]
    uint64_t *k_full = q_empty + 2 * C::QS, *k_empty = k_full + C::KS;
    uint64_t *v_full = k_empty + C::KS, *v_empty = v_full + C::KS;
    uint64_t *s_full = v_empty + C::KS;          // [2]  MMA -> softmax: S_g ready
    uint64_t *p_full = s_full + 2;               // [2]  softmax -> MMA: P_g written (O_g rescaled)
    uint64_t *epi = p_full + 2;                  // [2]  MMA -> softmax: last PV of the tile done
    uint64_t *s_empty = epi + 2;                 // [2]  softmax -> MMA: S_g loaded (SEP)
    uint64_t *pv_done = s_empty + 2;             // [2]  MMA -> softmax: PV_g complete (SEP)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + C::NBAR);
    constexpr bool SEP = C::SEP;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const DevAcsr &A = prm.A;
    const int n_units = A.n_pairs * prm.BH;
#ifdef SPLAT_TRACE
    int tr_n = 0;
#endif

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2 * C::QS; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
        for (int i = 0; i < C::KS; ++i) {
            mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 2);
            mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 2);
        }
        for (int g = 0; g < 2; ++g) {
            mbar_init(&s_full[g], 1); mbar_init(&p_full[g], 4); mbar_init(&epi[g], 1);
            mbar_init(&s_empty[g], 4); mbar_init(&pv_done[g], 1);
        }
        fence_mbar_init();
        tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); tma_prefetch(&tmO);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // Register budget (SEP): each SM sub-partition holds 16K registers and runs warps w, w+4, w+8;
    // warpgroup 0 (TMA, 2 MMA issuers, 1 idle) hands registers to the two softmax warpgroups,
    // which keep a whole 128-column S row in registers: 128*(168-56) == 256*(224-168).  The
    // setmaxnreg of each role sits inside the role's branch so ptxas can allocate per region.
    if (warp == 0 || warp == 3) {
        // ------------------------------------------------------------ TMA producers (warp-uniform loops)
        // warp 0: Q_A, Q_B of every unit and K_e of every union entry; warp 3: V_e.  K and V rings
        // advance independently: a K stage frees when both groups' S = Q K^T have completed, a V
        // stage only after both PVs, so K can run up to KS entries ahead of the softmax.
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        const bool kq = warp == 0;
        int qi[2] = {0, 0}, qc[2] = {0, 0};
        uint32_t qph[2] = {0, 0};
        int ki = 0, kc = 0;
        uint32_t kph = 0;
        uint64_t *full = kq ? k_full : v_full, *empty = kq ? k_empty : v_empty;
        const CUtensorMap *tm = kq ? &tmK : &tmV;
        uint8_t *ring = smem + (kq ? C::OFF_K : C::OFF_V);
        UnitInfo nx{};
        if (blockIdx.x < n_units) nx = SPLAT_FETCH(blockIdx.x);
        EntRegs ner;
        load_ents(A, nx, lane, ner);
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const UnitInfo un = nx;
            const EntRegs er = ner;
            if (u + (int)gridDim.x < n_units) nx = SPLAT_FETCH(u + gridDim.x);
            const int pair = un.pair, bh = un.bh;
            const bool uv = VM == 1 || (VM == 2 && un.pass);     // this unit runs on the residue-major views
            const CUtensorMap *tmu = VM == 2 && !uv ? (kq ? &tmK2 : &tmV2) : tm;
            if (kq) {
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    const int t = 2 * pair + g;
                    if (t >= A.n_qt) continue;
                    const int slot = g * C::QS + qi[g];
                    if (qc[g] >= C::QS) mbar_wait(&q_empty[slot], qph[g] ^ 1);
                    if (lane == 0) {
                        mbar_expect_tx(&q_full[slot], C::kTileBytes);
#pragma unroll
                        for (int c = 0; c < C::kChunks; ++c)
                            if (uv)
                                tma_load_4d(smem + C::OFF_Q + slot * C::kTileBytes + c * kTileBytes64, &tmQ,
                                            &q_full[slot], 64 * c, (t << 7) & (prm.rv_nk - 1), (t << 7) >> prm.rv_sh, bh);
                            else
                                tma_load_3d(smem + C::OFF_Q + slot * C::kTileBytes + c * kTileBytes64,
                                            VM == 2 ? &tmQ2 : &tmQ, &q_full[slot], 64 * c, t * 128, bh);
                    }
                    ++qc[g];
                    if (++qi[g] == C::QS) { qi[g] = 0; qph[g] ^= 1; }
                }
            }
            const int e0 = un.e0, e1 = un.e1;
            for (int e = e0; e < e1; ++e) {
                const int kv = ent_at(A, un, er, e) & kKvMask;
                if (e == e0 + 1) load_ents(A, nx, lane, ner);     // next unit's entries, in the shadow
                TRACE(kq ? 0 : 5, 30);
                if (kc >= C::KS) mbar_wait(&empty[ki], kph ^ 1);
                TRACE(kq ? 0 : 5, 31);
                if (lane == 0) {
                    mbar_expect_tx(&full[ki], C::kTileBytes);
#pragma unroll
                    for (int c = 0; c < C::kChunks; ++c)
                        if (uv)
                            tma_load_4d(ring + ki * C::kTileBytes + c * kTileBytes64, tmu, &full[ki], 64 * c,
                                        (kv << 6) & (prm.rv_nk - 1), (kv << 6) >> prm.rv_sh, bh);
                        else
                            tma_load_3d(ring + ki * C::kTileBytes + c * kTileBytes64, tmu, &full[ki], 64 * c, kv * kKvUnit, bh);
                }
                ++kc;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
            }
            if (e1 - e0 <= 1) load_ents(A, nx, lane, ner);
        }
    } else if (warp == 1 || warp == 2) {
        // ------------------------------------------------------------ MMA issuers (warp-uniform)
        // Warp 1 serves tile group A, warp 2 tile group B, so the two groups never wait for each
        // other's turnaround.  Per group the sequence is S(e) = Q K_e^T, [P(e) ready]
        // O += P(e) V_e, S(e') ... with P aliased into S's TMEM columns, hence PV(e) is issued
        // before S(e') (tcgen05 executes in issue order).  The whole warp runs the loop so the
        // descriptors live in uniform registers; lane 0 issues.  K/V stages are released when
        // both groups are done with them (empty barriers count two arrivals; a group that skips
        // an entry arrives once the entry is resident).
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        // uniform values (see elect_one): descriptors stay in uniform registers
        const int g = __shfl_sync(0xffffffffu, warp - 1, 0);
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
        constexpr uint32_t idS = idesc_bf16(128, 128, false);
        constexpr uint32_t idO = idesc_bf16(128, D, true);
        const uint32_t sQ = smem_u32(smem + C::OFF_Q), sK = smem_u32(smem + C::OFF_K);
        const uint32_t sV = smem_u32(smem + C::OFF_V);
        const bool leader = lane == 0;
        const int use_bit = g == 0 ? kUseA : kUseB;
        const uint32_t s_tm = tmem_u + g * 128, o_tm = tmem_u + 256 + g * D;
        const uint32_t p_tm = SEP ? tmem_u + 384 + g * 64 : s_tm;
        int qi = 0;
        uint32_t qph = 0, pcnt = 0, scnt = 0;
        uint32_t gent = 0;                                   // global entry counter (ring position)
        UnitInfo nx = blockIdx.x < n_units ? SPLAT_FETCH(blockIdx.x) : UnitInfo{0, 0, 0, 0};
        EntRegs ner;
        load_ents(A, nx, lane, ner);
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            UnitInfo un = nx;
            un.pair = __shfl_sync(0xffffffffu, un.pair, 0);
            un.e0 = __shfl_sync(0xffffffffu, un.e0, 0);
            un.e1 = __shfl_sync(0xffffffffu, un.e1, 0);
            const EntRegs er = ner;
            if (u + (int)gridDim.x < n_units) nx = SPLAT_FETCH(u + gridDim.x);
            const bool active = 2 * un.pair + g < A.n_qt;
            const int slot = g * C::QS + qi;
            if (active) mbar_wait(&q_full[slot], qph);
            const uint32_t qb = sQ + slot * C::kTileBytes;
            bool pend = false, first = true;
            int pst = 0;
            uint32_t pph = 0;
            // O += P V of the pending entry (P written by the softmax over S's columns).  Issued
            // before anything waits on a later K/V stage: that stage may only be refilled after
            // this PV releases its V.
#define SPLAT_PV_PENDING()                                                                               \
    do {                                                                                                 \
        TRACE(1 + 3 * g, 19);                                                                            \
        mbar_wait(&p_full[g], pcnt & 1);                                                                 \
        TRACE(1 + 3 * g, 21);                                                                            \
        ++pcnt;                                                                                          \
        mbar_wait(&v_full[pst], pph);                                                                    \
        tc_fence_after();                                                                                \
        const uint32_t vbase = sV + pst * C::kTileBytes;                                                 \
        if (elect_one()) {                                                                               \
            _Pragma("unroll") for (int kk = 0; kk < 8; ++kk)                                             \
                if (!(DBG(1)))                                                                      \
                    mma_bf16_ts(o_tm, p_tm + kk * 8, sdesc_sw128(vbase + kk * 2048, kTileBytes64, 1024), \
                                idO, (first && kk == 0) ? 0u : 1u);                                      \
            mma_commit(&v_empty[pst]);                                                                   \
            if (SEP) mma_commit(&pv_done[g]);                                                            \
        }                                                                                                \
        __syncwarp();                                                                                    \
        TRACE(1 + 3 * g, 20);                                                                             \
        first = false;                                                                                   \
        pend = false;                                                                                    \
    } while (0)
            for (int e = un.e0; e < un.e1; ++e) {
                const int ent = __shfl_sync(0xffffffffu, ent_at(A, un, er, e), 0);
                const int st = gent % C::KS;
                const uint32_t ph = (gent / C::KS) & 1;
                ++gent;
                if (e == un.e0 + 1) load_ents(A, nx, lane, ner);
                const bool ours = active && (ent & use_bit);
                // non-SEP: P lives in S's columns, so the PV must precede the next S.  SEP: the next S
                // goes first (the PV waits for the softmax); a pending PV is still flushed before
                // waiting on a stage this group does not use (that stage may need its release).
                // (SEP, skipped entry in the pending PV's own stage: the stage cannot be refilled
                // before that PV releases it -- flush first)
                if (pend && (!SEP || (!ours && pst == st))) SPLAT_PV_PENDING();
                if (!ours) {
                    // Not ours: release the stages, but only once they hold this entry.  Every group
                    // observes every phase of every stage in order -- parity waits are ambiguous
                    // as soon as a waiter could lag two phases behind a barrier.  (SEP: a pending
                    // PV of an earlier entry uses another V stage, which cannot advance before that
                    // PV is issued, so it may stay pending.)
                    mbar_wait(&k_full[st], ph);
                    if (leader) mbar_arrive(&k_empty[st]);
                    mbar_wait(&v_full[st], ph);
                    if (leader) mbar_arrive(&v_empty[st]);
                    continue;
                }
                TRACE(1 + 3 * g, 9);
                mbar_wait(&k_full[st], ph);
                if (SEP && scnt > 0) mbar_wait(&s_empty[g], (scnt - 1) & 1);   // previous S loaded
                ++scnt;
                tc_fence_after();
                const uint32_t kbase = sK + st * C::kTileBytes;
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = (kk >> 2) * kTileBytes64 + (kk & 3) * 32;
                        if (!(DBG(1)))
                            mma_bf16_ss(s_tm, sdesc_sw128(qb + off, 16, 1024), sdesc_sw128(kbase + off, 16, 1024),
                                        idS, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(&s_full[g]);
                    mma_commit(&k_empty[st]);
                }
                __syncwarp();
                TRACE(1 + 3 * g, 10);
                if (SEP && pend) SPLAT_PV_PENDING();
                pend = true;
                pst = st;
                pph = ph;
            }
            if (pend) SPLAT_PV_PENDING();
#undef SPLAT_PV_PENDING
            if (un.e1 - un.e0 <= 1) load_ents(A, nx, lane, ner);
            if (active) {
                if (elect_one()) {
                    mma_commit(&epi[g]);
                    mma_commit(&q_empty[slot]);
                }
                __syncwarp();
                if (++qi == C::QS) { qi = 0; qph ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------------------ softmax warps (4..7: A, 8..11: B)
        // Each group walks only its own query tile's plan entries (qt_ptr range in pair_info);
        // the fast-index mask of the next entry is prefetched one entry ahead (across unit
        // boundaries too) so its L2 latency never sits on the critical path.
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
        const int g = (warp - 4) >> 2;          // tile group: 0 = A, 1 = B
        const int quad = warp & 3;              // TMEM lane quadrant of this warp
        const int r = quad * 32 + lane;         // row within the query tile
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const uint32_t s_tm = tmem + lane_off + g * 128;
        const uint32_t o_tm = tmem + lane_off + 256 + g * D;
        const uint32_t p_tm = SEP ? tmem + lane_off + 384 + g * 64 : s_tm;
        const float c2 = prm.scale_log2;
        const bool store_leader = quad == 0 && lane == 0;
        uint8_t *ostage = smem + C::OFF_O + g * kTileBytes64;
        const uint32_t ostage_u = smem_u32(ostage);
        uint32_t s_cnt = 0, e_cnt = 0;
        int dep_pend = -1;           // VM = 2: head whose strided-pass tile this group stored last, not yet signalled
        // VM = 2: the strided-pass O_s / lse of head dep_pend are complete in memory -> count it for the
        // band-pass units of that head (done before any wait of this group, so it can never wait on itself)
        auto dep_signal = [&]() {
            if (VM == 2 && dep_pend >= 0) {
                if (store_leader) {
                    bulk_wait0();                                   // this thread's TMA stores have landed
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    __threadfence();
                    atomicAdd(prm.dep + dep_pend, 1u);
                }
                dep_pend = -1;
            }
        };
        // O / l -> bf16 -> swizzled SMEM stage -> TMA store (rows beyond N clipped by the map)
        // uv: a residue-major (strided-pass) tile; VM = 2 merges every other tile
        auto epilogue = [&](float l, float m, int t, int bh, bool uv) {
            mbar_wait(&epi[g], e_cnt & 1);
            ++e_cnt;
            tc_fence_after();
            if (store_leader) TRACE(2 + g, 8);
            const bool merge = VM == 2 ? !uv : prm.merge != 0;
            dep_signal();
            if (VM == 2 && merge) {
                // the strided pass of this head must be complete (its units precede this one in the
                // sequence, so they are running or done on some CTA)
                if (lane == 0) {
                    unsigned v;
                    // relaxed polls (an acquire per poll would also invalidate the SM's L1), one acquire
                    // fence once the count is reached
                    for (long long n = 0;; ++n) {
                        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(prm.dep + bh) : "memory");
                        if (v >= (unsigned)prm.dep_target) break;
                        if (n > (1ll << 26)) __trap();      // a broken dependency fails loudly (~10 s), never hangs
                        __nanosleep(256);
                    }
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
                __syncwarp();
            }
            float inv = l > 0.f ? 1.f / l : 0.f;
            // residue decomposition: natural row of this thread's tile row
            // permuted row p = 128 t + r is residue class p / nk, position p % nk: natural p / nk + l (p % nk)
            const int nat = uv ? ((t * 128 + r) >> prm.rv_sh) + prm.rv_l * ((t * 128 + r) & (prm.rv_nk - 1))
                               : t * 128 + r;
            const bool in_range = nat < prm.N;
            float a_s = 0.f;                      // merge weight of the strided partial (pass 2)
            if (uv && prm.lse && in_range)
                prm.lse[(size_t)bh * prm.N + nat] = l > 0.f ? m + __log2f(l) : -INFINITY;
            if (merge) {
                // O = (O_b 2^(m_b - M) + O_s 2^(lse_s - M)) / (l_b 2^(m_b - M) + 2^(lse_s - M))
                const float lse_s = in_range ? prm.lse[(size_t)bh * prm.N + nat] : -INFINITY;
                const float lse_b = l > 0.f ? m + __log2f(l) : -INFINITY;
                const float M = fmaxf(lse_b, lse_s);
                const float a_b = l > 0.f ? ex2(m - M) : 0.f;
                a_s = lse_s == -INFINITY ? 0.f : ex2(lse_s - M);
                const float den = l * a_b + a_s;
                inv = den > 0.f ? a_b / den : 0.f;
                a_s = den > 0.f ? a_s / den : 0.f;
            }
#pragma unroll
            for (int c = 0; c < D / 64; ++c) {
                float o[64];
                tmem_ld32(o_tm + c * 64, o);
                tmem_ld32(o_tm + c * 64 + 32, o + 32);
                tmem_wait_ld();
                uint32_t w[32];
                if (merge) {
                    uint4 os[8];
                    const uint4 *src = reinterpret_cast<const uint4 *>(prm.O + ((size_t)bh * prm.N + nat) * D + 64 * c);
#pragma unroll
                    for (int q = 0; q < 8; ++q) os[q] = in_range ? src[q] : make_uint4(0u, 0u, 0u, 0u);
                    const uint32_t *ow = reinterpret_cast<const uint32_t *>(os);
#pragma unroll
                    for (int x = 0; x < 32; ++x) {
                        const float s0 = __uint_as_float(ow[x] << 16), s1 = __uint_as_float(ow[x] & 0xffff0000u);
                        w[x] = pack_bf16(o[2 * x] * inv + s0 * a_s, o[2 * x + 1] * inv + s1 * a_s);
                    }
                } else {
#pragma unroll
                    for (int x = 0; x < 32; ++x)
                        w[x] = inv == 0.f ? 0u : pack_bf16(o[2 * x] * inv, o[2 * x + 1] * inv);
                }
                if (store_leader) bulk_wait_read0();      // the stage's previous store has read it
                named_bar(1 + g, 128);
#pragma unroll
                for (int ch = 0; ch < 8; ++ch)
                    st_shared_v4(ostage_u + r * 128 + ((ch ^ (r & 7)) << 4), w[4 * ch], w[4 * ch + 1],
                                 w[4 * ch + 2], w[4 * ch + 3]);
                fence_proxy_async_smem();
                named_bar(1 + g, 128);
                if (store_leader) {
                    if (uv)
                        tma_store_4d(&tmO, ostage, 64 * c, (t << 7) & (prm.rv_nk - 1), (t << 7) >> prm.rv_sh, bh);
                    else tma_store_3d(VM == 2 ? &tmO2 : &tmO, ostage, 64 * c, t * 128, bh);
                    bulk_commit();
                }
            }
            if (VM == 2 && uv) dep_pend = bh;     // signalled at this group's next epilogue (or exit)
#ifdef SPLAT_X_DEPNOW
            dep_signal();                         // ablation (diagnostics build): signal immediately
#endif
            tc_fence_before();
            if (store_leader) TRACE(2 + g, 9);
        };
        bool pe_on = false;          // deferred epilogue of the previous unit (SEP)
        float pe_l = 0.f, pe_m = 0.f;
        int pe_t = 0, pe_bh = 0;
        bool pe_uv = false;
        UnitInfo nx{};
        if (blockIdx.x < n_units) nx = SPLAT_FETCH(blockIdx.x);
        TileRegs ntr;
        load_tile(A, nx.j0[g], nx.j0[g + 1], lane, ntr);
        uint4 pf = make_uint4(~0u, ~0u, ~0u, ~0u);     // mask of the next entry to process
        if (nx.j0[g] < nx.j0[g + 1]) pf = fetch_mask(A, ntr, nx.j0[g], nx.j0[g], quad, r);
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const UnitInfo un = nx;
            const TileRegs tr = ntr;
            const bool has_next = u + (int)gridDim.x < n_units;
            if (has_next) nx = SPLAT_FETCH(u + gridDim.x);
            const int j0 = un.j0[g], j1 = un.j0[g + 1];
            // next unit's entries and its first mask: issued during this unit's last entry
#define SPLAT_NEXT_UNIT_PREFETCH()                                                                      \
    do {                                                                                                \
        if (has_next) {                                                                                 \
            load_tile(A, nx.j0[g], nx.j0[g + 1], lane, ntr);                                            \
            if (nx.j0[g] < nx.j0[g + 1]) pf = fetch_mask(A, ntr, nx.j0[g], nx.j0[g], quad, r);          \
        }                                                                                               \
    } while (0)
            const int t = 2 * un.pair + g;
            if (t >= A.n_qt) {
                SPLAT_NEXT_UNIT_PREFETCH();
                continue;
            }
            const int bh = un.bh;
            const bool uv = VM == 1 || (VM == 2 && un.pass);
            if (VM == 2 ? !uv : (!VIEW && prm.merge)) {
                // the merging epilogue of this tile (deferred past the next unit's first tile) reads
                // this row's strided-pass O_s and lse: pull them into L2 now
                const int nat = t * 128 + r;
                if (nat < prm.N) {
                    const char *orow = reinterpret_cast<const char *>(prm.O + ((size_t)bh * prm.N + nat) * D);
#pragma unroll
                    for (int b = 0; b < D * 2; b += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(orow + b));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(prm.lse + (size_t)bh * prm.N + nat));
                }
            }
            float m_run = -INFINITY, l_run = 0.f;
            bool first = true;
            if (j0 == j1) SPLAT_NEXT_UNIT_PREFETCH();
            for (int j = j0; j < j1; ++j) {
                if (store_leader) TRACE(2 + g, 5);
                const uint4 m4 = pf;
                int mid;
                uint32_t bits;
                tile_at(A, tr, j0, j, mid, bits);
                if (j + 1 < j1) pf = fetch_mask(A, tr, j0, j + 1, quad, r);
                else SPLAT_NEXT_UNIT_PREFETCH();
                const uint32_t mk[4] = {m4.x, m4.y, m4.z, m4.w};
                uint32_t live = (bits >> (4 * quad)) & 0xFu;
                const uint32_t need = live & ~(bits >> (16 + 4 * quad));
                mbar_wait(&s_full[g], s_cnt & 1);
                ++s_cnt;
                tc_fence_after();
                if (store_leader) TRACE(2 + g, 2);
                float mx = -INFINITY;
                float sv[128];
                // the whole S row -> registers in two halves (the second half's load overlaps the
                // first half's mask + max); SEP: then S goes back to the MMA warp
                tmem_ld32(s_tm, sv);
                tmem_ld32(s_tm + 32, sv + 32);
                tmem_wait_ld();
                tmem_ld32(s_tm + 64, sv + 64);
                tmem_ld32(s_tm + 96, sv + 96);
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    if (w == 2) {
                        tmem_wait_ld();
                        if constexpr (SEP) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&s_empty[g]);
                        }
                    }
                    if (live & (1u << w)) {
                        if (need & (1u << w)) apply_mask(sv + 32 * w, mk[w]);
                        mx = fmax3(mx, max32(sv + 32 * w), -INFINITY);
                    }
                }
                if (store_leader) TRACE(2 + g, 12);
                mx *= c2;
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
                const uint64_t cc = pack2(c2, c2), mm = pack2(-mref, -mref);
                uint64_t acc0 = pack2(0.f, 0.f), acc1 = acc0;
                if DBG(2) live = 0;
                // exponentials first (registers): SEP -- the previous PV has long finished when O is
                // rescaled and P rewritten; non-SEP -- P overwrites S's columns (all of S is in
                // registers already) and S(j) was computed after PV(j-1), so O is final here
                uint32_t pw[64];
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    if (live & (1u << w)) {
                        exp32<D == 64 ? SPLAT_NEMU : SPLAT_NEMU128>(sv + 32 * w, cc, mm, acc0, acc1, pw + 16 * w);
                    } else {
#pragma unroll
                        for (int x = 0; x < 16; ++x) pw[16 * w + x] = 0u;
                    }
                }
                if (store_leader) TRACE(2 + g, 13);
                if constexpr (SEP) {
                    if (pe_on) {             // the previous unit's epilogue (first tile of a unit only)
                        epilogue(pe_l, pe_m, pe_t, pe_bh, pe_uv);
                        pe_on = false;
                    }
                    if (s_cnt > 1) {
                        // PV of this group's previous tile: complete before O is rescaled or P rewritten
                        mbar_wait(&pv_done[g], (s_cnt - 2) & 1);
                        tc_fence_after();
                    }
                }
                if (store_leader) TRACE(2 + g, 14);
                if (!first && __any_sync(0xffffffffu, resc)) {
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        float o[32];
                        tmem_ld32(o_tm + c * 32, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int x = 0; x < 32; ++x) o[x] *= alpha;
                        tmem_st32(o_tm + c * 32, o);
                    }
                }
                tmem_st32(p_tm, reinterpret_cast<const float *>(pw));
                tmem_st32(p_tm + 32, reinterpret_cast<const float *>(pw + 32));
                {
                    float a, b, c, d;
                    unpack2(acc0, a, b);
                    unpack2(acc1, c, d);
                    l_run += (a + b) + (c + d);
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[g]);
                if (store_leader) TRACE(2 + g, 4);
                first = false;
            }
#undef SPLAT_NEXT_UNIT_PREFETCH
            // epilogue.  SEP: deferred into the next unit's first tile (after its exponentials), so
            // the wait for this unit's last PV overlaps them; the first PV of the next unit
            // (accumulate = 0) is issued only after that tile's P, i.e. after O was read out.
            if constexpr (SEP) {
                if (j0 == j1) epilogue(l_run, m_run, t, bh, uv);      // degenerate: no entry to defer into
                else { pe_on = true; pe_l = l_run; pe_m = m_run; pe_t = t; pe_bh = bh; pe_uv = uv; }
            } else {
                epilogue(l_run, m_run, t, bh, uv);
            }
        }
        if (pe_on) epilogue(pe_l, pe_m, pe_t, pe_bh, pe_uv);
        dep_signal();
        if (store_leader) bulk_wait0();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
    if (VM == 2 && threadIdx.x == 0) {
        // the last CTA resets the dependency counters for the next launch on this launch slot
        __threadfence();
        if (atomicAdd(prm.dep + kLseHeads, 1u) == gridDim.x - 1u) {
            for (int i = 0; i < prm.BH; ++i) prm.dep[i] = 0u;
            prm.dep[kLseHeads] = 0u;
            __threadfence();
        }
    }
#undef SPLAT_FETCH
}

#ifdef SPLAT_FUSED_PROF
// Profiling aid (SPLAT_FUSED_PROF build): cycles each warp of CTA 0 spends in each barrier wait
// of the split kernel (by call site) and in total; read with splat_debug_fused_prof.
__device__ unsigned long long g_fprof[12][16];
#define FWAIT(SITE, BAR, PH)                                                                    \
    do {                                                                                        \
        const unsigned long long t0_ = clock64();                                               \
        mbar_wait(BAR, PH);                                                                     \
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)                                         \
            g_fprof[threadIdx.x >> 5][SITE] += clock64() - t0_;                                 \
    } while (0)
#else
#define FWAIT(SITE, BAR, PH) mbar_wait(BAR, PH)
#endif

// ================================================================ split-group kernel (d = 64)
//
// The two tile groups of a CTA run fully independent pipelines (own Q/K/V rings, own
// producer and MMA warps) over their own stream of single-query-tile work units (bucketed
// longest first, head-major inside a bucket; group g of CTA c takes units 2c + g + 2k * grid).
// Sharing K/V loads between two query tiles (the paired kernel above) couples the groups
// through one ring: a group that does not use an entry still has to wait for its loads, and a
// long tile stalls its partner.  At d = 64 both groups' rings fit in SMEM, so they are split.
//
//   warp 0 / 3 : TMA producer of group 0 / 1 (Q ring of 2, K and V rings of 2)
//   warp 1 / 2 : MMA issuer of group 0 / 1: S(j) = Q K_j^T as soon as K_j is resident and the
//                softmax has read S(j-1); then O += P(j-1) V_(j-1).  The pending PV carries
//                across unit boundaries, so the next unit's first S overlaps the last softmax.
//   warps 4-7 / 8-11 : softmax of group 0 / 1 (as in the paired kernel, deferred epilogue).
// TMEM: S_g [128g, 128g+128), O_g [256+64g, +64), P_g [384+64g, +64).
struct SCfg {
    static constexpr int QS = 2, KS = 2;
    static constexpr int TB = kTileBytes64;                      // 16 KB: 128 rows x 64 bf16
    static constexpr int OFF_Q = 0, OFF_K = QS * TB, OFF_V = OFF_K + KS * TB, OFF_O = OFF_V + KS * TB;
    static constexpr int GROUP = OFF_O + TB;                     // 112 KB per group
    static constexpr int OFF_BAR = 2 * GROUP;
    // per group: q_full[QS] q_empty[QS] k_full[KS] k_empty[KS] v_full[KS] v_empty[KS]
    //            s_full s_empty p_full pv_done epi
    static constexpr int NB = 2 * QS + 4 * KS + 5;
    // per group and Q slot: the unit's first kInfo plan entries (mask id, chunk bits), written by
    // the producer before it arms q_full -- the softmax reads them with one broadcast LDS
    static constexpr int kInfo = 32;
    static constexpr int OFF_INFO = OFF_BAR + 2 * NB * 8;        // [2 groups][QS][kInfo] int2
    static constexpr int OFF_HDR = OFF_INFO + 2 * QS * kInfo * 8;  // [2 groups][QS] int4: unit (t, bh, j0, j1)
    static constexpr int OFF_HDR2 = OFF_HDR + 2 * QS * 16 + 16;     // [2 groups][QS] int: split field; [2] merge flags
    // [2 groups][4 warps] int: split field of the warp's pending (deferred) epilogue, then [2][128] f32
    // its rows' running maxima
    static constexpr int OFF_PE = (OFF_HDR2 + 2 * QS * 4 + 2 * 4 + 15) / 16 * 16;
    // the dynamic buffer starts 1024-byte aligned (no static shared memory; checked with a trap)
    static constexpr int SMEM = OFF_PE + 32 + 2 * 128 * 4 + 8;
    static_assert(SMEM <= 232448, "shared memory budget");
};

struct TUnit {
    int t, bh, j0, j1;
    int split;      // split-K part: part | parts << 8 | split-tile index << 16; 0 = whole tile
};

__device__ __forceinline__ TUnit fetch_tunit(const DevAcsr &A, int BH, int v)
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
    return TUnit{x.x, bh, x.y, x.z, x.w};
}

// key-tile index of the unit's entries, cached in a (uniformly executing) warp's registers
struct KvRegs {
    int r[2];
};

__device__ __forceinline__ void load_kv(const DevAcsr &A, const TUnit &un, int lane, KvRegs &kr)
{
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int j = un.j0 + lane + 32 * k;
        kr.r[k] = j < un.j1 ? (A.kv[j] & (kKvMask | kCompBit)) : 0;
    }
}

__device__ __forceinline__ int kv_at(const DevAcsr &A, const TUnit &un, const KvRegs &kr, int j)
{
    const int i = j - un.j0;
    if (i < 64) return __shfl_sync(0xffffffffu, i < 32 ? kr.r[0] : kr.r[1], i & 31);
    return A.kv[j] & (kKvMask | kCompBit);
}

// The two 64-row key blocks of a split-kernel window: kv and kv + 1, or a composite's a and b
__device__ __forceinline__ int2 kv_blocks(int ent)
{
    return (ent & kCompBit) ? make_int2(ent & 0xFFF, (ent >> 12) & 0xFFF) : make_int2(ent, ent + 1);
}

// KS: the split-K unit list (long tiles in parts, merged by the last part); a separate instantiation
// so the whole-tile kernel carries none of the merge code
template <bool KS>
__global__ void __launch_bounds__(kThreads, 1)
mhsa_split_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                  const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmV64, const Params prm)
{
    using C = SCfg;
    constexpr int D = 64;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // No static shared memory precedes the dynamic buffer, so it starts 1024-byte aligned (checked
    // with a trap; SCfg reserves no slack).  Using smem_raw itself -- not an integer align-up --
    // keeps the shared state space visible to the compiler (LDS/STS, constant offsets).
    uint8_t *smem = smem_raw;
    if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u) != 0u) __trap();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // group of this warp: producers 0 / 3, MMA 1 / 2, softmax 4-7 / 8-11
    const int g = warp >= 4 ? (warp - 4) >> 2 : (warp == 0 || warp == 1 ? 0 : 1);
    uint8_t *gs = smem + g * C::GROUP;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR) + g * C::NB;
    uint64_t *q_full = bars, *q_empty = q_full + C::QS;
    uint64_t *k_full = q_empty + C::QS, *k_empty = k_full + C::KS;
    uint64_t *v_full = k_empty + C::KS, *v_empty = v_full + C::KS;
    uint64_t *s_full = v_empty + C::KS, *s_empty = s_full + 1, *p_full = s_empty + 1;
    uint64_t *pv_done = p_full + 1, *epi = pv_done + 1;
    int2 *info = reinterpret_cast<int2 *>(smem + C::OFF_INFO) + g * C::QS * C::kInfo;   // [QS][kInfo]
    int4 *hdr = reinterpret_cast<int4 *>(smem + C::OFF_HDR) + g * C::QS;               // [QS]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::OFF_HDR + 2 * C::QS * 16);
    const DevAcsr &A = prm.A;
    const int n_units = A.t_n * prm.BH;
#ifdef SPLAT_FUSED_PROF
    const unsigned long long t_start = clock64();
#endif
#ifdef SPLAT_TRACE
    int tr_n = 0;
#endif

    if (threadIdx.x == 0) {
        for (int gg = 0; gg < 2; ++gg) {
            uint64_t *b = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR) + gg * C::NB;
            for (int i = 0; i < 2 * C::QS + 4 * C::KS; ++i) mbar_init(&b[i], 1);
            // q_full: every lane of the producer warp publishes its writes of the unit's header /
            // entry table itself (lane 0's arrival carries the Q tile's bytes); q_empty: the unit's
            // last PV (MMA commit) and every softmax thread, done reading them -- the producer
            // rewrites both only after all of these
            for (int i = 0; i < C::QS; ++i) mbar_init(&b[i], 32);
            for (int i = 0; i < C::QS; ++i) mbar_init(&b[C::QS + i], 129);
            const int o = 2 * C::QS + 4 * C::KS;
            mbar_init(&b[o + 0], 1);   // s_full  (MMA commit)
            mbar_init(&b[o + 1], 4);   // s_empty (4 softmax warps)
            mbar_init(&b[o + 2], 4);   // p_full  (4 softmax warps)
            mbar_init(&b[o + 3], 1);   // pv_done (MMA commit)
            mbar_init(&b[o + 4], 1);   // epi     (MMA commit)
        }
        fence_mbar_init();
        tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); tma_prefetch(&tmO);
        tma_prefetch(&tmK64); tma_prefetch(&tmV64);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 || warp == 3) {
        // ------------------------------------------------------------ TMA producer of group g
        // Issue order K(j), V(j-1): V(j-1) waits for the PV of j-3 to free its stage, and the K
        // loads run one entry ahead of it so S never waits for a V release.
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        int qi = 0, qc = 0, ki = 0, kc = 0, vi = 0, vc = 0;
        uint32_t qph = 0, kph = 0, vph = 0;
        bool pv = false;            // V of the previous entry still to load
        int pv_kv = 0, pv_bh = 0;
        auto load_v = [&]() {
            if (vc >= C::KS) FWAIT(10, &v_empty[vi], vph ^ 1);
            if (lane == 0) {
                if DBG(16) {          // profiling aid: no TMA traffic (garbage K/V)
                    mbar_arrive(&v_full[vi]);
                } else {
                    mbar_expect_tx(&v_full[vi], C::TB);
                    if (pv_kv & kCompBit) {                    // composite window: two 64-row boxes
                        const int2 vb = kv_blocks(pv_kv);
                        tma_load_3d(gs + C::OFF_V + vi * C::TB, &tmV64, &v_full[vi], 0, vb.x * kKvUnit, pv_bh);
                        tma_load_3d(gs + C::OFF_V + vi * C::TB + C::TB / 2, &tmV64, &v_full[vi], 0, vb.y * kKvUnit, pv_bh);
                    } else {
                        tma_load_3d(gs + C::OFF_V + vi * C::TB, &tmV, &v_full[vi], 0, pv_kv * kKvUnit, pv_bh);
                    }
                }
            }
            ++vc;
            if (++vi == C::KS) { vi = 0; vph ^= 1; }
            pv = false;
        };
        // Dynamic schedule: the producer grabs the next unit from the handle's work counter (units
        // are bucketed longest first, so greedy grabbing balances the long global-row tiles) and
        // publishes it -- header (tile, bh, j0, j1) and entry table -- to the group's MMA and
        // softmax warps with the Q slot's q_full; a header with tile -1 ends the stream.
        auto grab = [&]() {
            int v = 0;
            if (lane == 0) v = (int)atomicAdd(prm.sched, 1ull);
            v = __shfl_sync(0xffffffffu, v, 0);
            return v < n_units ? fetch_tunit(A, prm.BH, v) : TUnit{-1, 0, 0, 0, 0};
        };
        TUnit nx = grab();
        KvRegs nkr;
        load_kv(A, nx, lane, nkr);
        while (true) {
            const TUnit un = nx;
            const KvRegs kr = nkr;
            if (qc >= C::QS) FWAIT(8, &q_empty[qi], qph ^ 1);
            if (un.t < 0) {
                if (lane == 0) hdr[qi] = make_int4(-1, 0, 0, 0);
                mbar_arrive(&q_full[qi]);
                break;
            }
            nx = grab();                      // next unit, fetched in the shadow of this one
            if (lane < un.j1 - un.j0 && lane < C::kInfo)
                info[qi * C::kInfo + lane] = make_int2(A.kv_mask[un.j0 + lane], (int)A.qt_bits[un.j0 + lane]);
            if (lane == 0) {
                hdr[qi] = make_int4(un.t, un.bh, un.j0, un.j1);
                if (KS) reinterpret_cast<int *>(smem + C::OFF_HDR2)[g * C::QS + qi] = un.split;   // split field
            }
            // header + table: each lane's arrival releases its own writes; lane 0's carries the Q bytes
            if (lane == 0) {
                // the tile's two 64-row segments (row classes, plan.cpp): rows 0-63 and 64-127
                mbar_expect_tx(&q_full[qi], C::TB);
                const int sa = A.row_classes ? (un.t & 0xFFFF) : 2 * un.t, sb = A.row_classes ? (un.t >> 16) : 2 * un.t + 1;
                tma_load_3d(gs + C::OFF_Q + qi * C::TB, &tmQ, &q_full[qi], 0, sa * 64, un.bh);
                tma_load_3d(gs + C::OFF_Q + qi * C::TB + C::TB / 2, &tmQ, &q_full[qi], 0, sb * 64, un.bh);
            } else {
                mbar_arrive(&q_full[qi]);
            }
            ++qc;
            if (++qi == C::QS) { qi = 0; qph ^= 1; }
            for (int j = un.j0; j < un.j1; ++j) {
                const int kv = kv_at(A, un, kr, j);
                if (j == un.j0 + 1) load_kv(A, nx, lane, nkr);   // next unit's entries, in the shadow
                TRACE(g == 0 ? 0 : 5, 30);
                if (kc >= C::KS) FWAIT(9, &k_empty[ki], kph ^ 1);
                TRACE(g == 0 ? 0 : 5, 31);
                if (lane == 0) {
                    if DBG(16) {
                        mbar_arrive(&k_full[ki]);
                    } else {
                        mbar_expect_tx(&k_full[ki], C::TB);
                        if (kv & kCompBit) {
                            const int2 kb = kv_blocks(kv);
                            tma_load_3d(gs + C::OFF_K + ki * C::TB, &tmK64, &k_full[ki], 0, kb.x * kKvUnit, un.bh);
                            tma_load_3d(gs + C::OFF_K + ki * C::TB + C::TB / 2, &tmK64, &k_full[ki], 0, kb.y * kKvUnit, un.bh);
                        } else {
                            tma_load_3d(gs + C::OFF_K + ki * C::TB, &tmK, &k_full[ki], 0, kv * kKvUnit, un.bh);
                        }
                    }
                }
                ++kc;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
                if (pv) load_v();
                pv = true;
                pv_kv = kv;
                pv_bh = un.bh;
            }
            if (un.j1 - un.j0 <= 1) load_kv(A, nx, lane, nkr);
        }
        if (pv) load_v();
    } else if (warp == 1 || warp == 2) {
        // ------------------------------------------------------------ MMA issuer of group g
        // Everything this role computes is made provably warp-uniform (group index, TMEM base and
        // unit fields broadcast with __shfl_sync) and MMAs / commits are issued under elect.sync,
        // so the descriptors live in uniform registers and the UTCHMMAs issue back to back.
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        const int gu = __shfl_sync(0xffffffffu, g, 0);
        const uint32_t tmu = __shfl_sync(0xffffffffu, tmem, 0);
        uint8_t *gsu = smem + gu * C::GROUP;
        uint64_t *bu = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR) + gu * C::NB;
        uint64_t *uq_full = bu, *uq_empty = uq_full + C::QS, *uk_full = uq_empty + C::QS, *uk_empty = uk_full + C::KS;
        uint64_t *uv_full = uk_empty + C::KS, *uv_empty = uv_full + C::KS;
        uint64_t *us_full = uv_empty + C::KS, *us_empty = us_full + 1, *up_full = us_empty + 1;
        uint64_t *upv_done = up_full + 1, *uepi = upv_done + 1;
        constexpr uint32_t idS = idesc_bf16(128, 128, false);
        constexpr uint32_t idO = idesc_bf16(128, D, true);
        const uint32_t sQ = smem_u32(gsu + C::OFF_Q), sK = smem_u32(gsu + C::OFF_K), sV = smem_u32(gsu + C::OFF_V);
        const uint32_t s_tm = tmu + gu * 128, o_tm = tmu + 256 + gu * D, p_tm = tmu + 384 + gu * 64;
        const bool no_mma = (DBG(1)) != 0;
        int qi = 0;
        uint32_t qph = 0, pcnt = 0, scnt = 0, gent = 0;
        // the pending PV (entry whose P the softmax is computing)
        bool pend = false, p_first = false, p_last = false;
        int pst = 0, pq = 0;
        uint32_t pph = 0;
        auto flush_pv = [&]() {
            FWAIT(6, up_full, pcnt & 1);
            ++pcnt;
            FWAIT(7, &uv_full[pst], pph);
            tc_fence_after();
            const uint32_t vbase = sV + pst * C::TB;
            if (elect_one()) {
                if (!no_mma) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16_ts(o_tm, p_tm + kk * 8, sdesc_sw128(vbase + kk * 2048, kTileBytes64, 1024), idO,
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
            TRACE(1 + 3 * g, 20);
            pend = false;
        };
        int4 *uhdr = reinterpret_cast<int4 *>(smem + C::OFF_HDR) + gu * C::QS;
        while (true) {
            FWAIT(11, &uq_full[qi], qph);
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
                TRACE(1 + 3 * g, 9);
                FWAIT(4, &uk_full[st], ph);
                TRACE(1 + 3 * g, 11);
                if (scnt > 0) FWAIT(5, us_empty, (scnt - 1) & 1);   // softmax has read the previous S
                ++scnt;
                tc_fence_after();
                const uint32_t kbase = sK + st * C::TB;
                if (elect_one()) {
                    if (!no_mma) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk)
                            mma_bf16_ss(s_tm, sdesc_sw128(qb + kk * 32, 16, 1024), sdesc_sw128(kbase + kk * 32, 16, 1024),
                                        idS, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(us_full);
                    mma_commit(&uk_empty[st]);
                }
                __syncwarp();
                TRACE(1 + 3 * g, 10);
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
        const uint32_t o_tm = tmem + lane_off + 256 + g * D;
        const uint32_t p_tm = tmem + lane_off + 384 + g * 64;
        const float c2 = prm.scale_log2;
        const bool store_leader = quad == 0 && lane == 0;
        uint8_t *ostage = gs + C::OFF_O;
        const uint32_t ostage_u = smem_u32(ostage);
        uint32_t s_cnt = 0, e_cnt = 0;
        // sp: split-K part of a long tile (0 = whole tile): the part publishes its normalised partial O
        // (bf16) and lse2 = m + log2(l) to the launch slot's scratch; the last part of the tile to
        // arrive merges all parts in part order (deterministic) and stores the tile
        auto epilogue = [&](float l, float m, int t, int bh, int sp) {
            FWAIT(2, epi, e_cnt & 1);
            ++e_cnt;
            tc_fence_after();
            if (store_leader) TRACE(2 + g, 8);
            const float inv = l > 0.f ? 1.f / l : 0.f;
            float o[64];
            tmem_ld32(o_tm, o);
            tmem_ld32(o_tm + 32, o + 32);
            tmem_wait_ld();
            uint32_t w[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) w[x] = inv == 0.f ? 0u : pack_bf16(o[2 * x] * inv, o[2 * x + 1] * inv);
            if (KS && sp != 0) {
                const int part = sp & 0xFF, np = (sp >> 8) & 0xFF, sid = sp >> 16;
                const size_t tix = (size_t)bh * A.n_ksplit + sid, base = tix * A.ks_pmax;
                uint4 *dst = reinterpret_cast<uint4 *>(A.ks_o) + ((base + part) * 128 + r) * 8;
#pragma unroll
                for (int q = 0; q < 8; ++q) dst[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
                A.ks_lse[(base + part) * 128 + r] = l > 0.f ? m + __log2f(l) : -INFINITY;
                named_bar(1 + g, 128);
                if (store_leader) {
                    __threadfence();
                    reinterpret_cast<int *>(smem + C::OFF_HDR2)[2 * C::QS + g] =
                        atomicAdd(A.ks_cnt + tix, 1u) == (unsigned)(np - 1) ? 1 : 0;
                }
                named_bar(1 + g, 128);
                if (!reinterpret_cast<const int *>(smem + C::OFF_HDR2)[2 * C::QS + g]) {
                    tc_fence_before();
                    return;
                }
                __threadfence();
                float M = -INFINITY;
                for (int q = 0; q < np; ++q) M = fmaxf(M, __ldcg(A.ks_lse + (base + q) * 128 + r));
                // two halves of 32 columns (register budget): weights recomputed per half
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float acc[32];
#pragma unroll
                    for (int x = 0; x < 32; ++x) acc[x] = 0.f;
                    float den = 0.f;
                    for (int q = 0; q < np; ++q) {
                        const float lq = __ldcg(A.ks_lse + (base + q) * 128 + r);
                        const float aq = lq == -INFINITY ? 0.f : ex2(lq - M);
                        den += aq;
                        const uint4 *src = reinterpret_cast<const uint4 *>(A.ks_o) + ((base + q) * 128 + r) * 8 + 4 * h;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint4 u4 = __ldcg(src + c);
                            const uint32_t uu[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
                            for (int y = 0; y < 4; ++y) {
                                acc[8 * c + 2 * y] += aq * __uint_as_float(uu[y] << 16);
                                acc[8 * c + 2 * y + 1] += aq * __uint_as_float(uu[y] & 0xffff0000u);
                            }
                        }
                    }
                    const float id = den > 0.f ? 1.f / den : 0.f;
#pragma unroll
                    for (int x = 0; x < 16; ++x)
                        w[16 * h + x] = den > 0.f ? pack_bf16(acc[2 * x] * id, acc[2 * x + 1] * id) : 0u;
                }
                if (store_leader) A.ks_cnt[tix] = 0u;      // for the next launch on this slot
            }
            if (store_leader) bulk_wait_read0();      // the stage's previous store has read it
            named_bar(1 + g, 128);
#pragma unroll
            for (int ch = 0; ch < 8; ++ch)
                st_shared_v4(ostage_u + r * 128 + ((ch ^ (r & 7)) << 4), w[4 * ch], w[4 * ch + 1], w[4 * ch + 2],
                             w[4 * ch + 3]);
            fence_proxy_async_smem();
            named_bar(1 + g, 128);
            if (store_leader) {
                const int sa = A.row_classes ? (t & 0xFFFF) : 2 * t, sb = A.row_classes ? (t >> 16) : 2 * t + 1;
                tma_store_3d(&tmO, ostage, 0, sa * 64, bh);
                tma_store_3d(&tmO, ostage + C::TB / 2, 0, sb * 64, bh);
                bulk_commit();
            }
            tc_fence_before();
            if (store_leader) TRACE(2 + g, 9);
        };
        bool pe_on = false;          // deferred epilogue of the previous unit
        float pe_l = 0.f;
        int pe_t = 0, pe_bh = 0;
        // the pending epilogue's split field and row maxima live in SMEM (register budget)
        int *pe_sp_s = reinterpret_cast<int *>(smem + C::OFF_PE) + g * 4 + quad;    // this warp's copy
        float *pe_m_s = reinterpret_cast<float *>(smem + C::OFF_PE + 32) + g * 128 + r;
        // the unit's entry table (mask id, bits) of Q slot qs, entry index i = j - j0
        int qs = 0;
        uint32_t qph = 0;
        auto entry = [&](int slot, int j0_, int j_) {
            const int i = j_ - j0_;
            return i < C::kInfo ? info[slot * C::kInfo + i] : make_int2(A.kv_mask[j_], (int)A.qt_bits[j_]);
        };
        auto mask_for = [&](int2 e) {       // row mask of this thread for entry e (ones if unneeded)
            const uint32_t bits = (uint32_t)e.y;
            const uint32_t need = (bits >> (4 * quad)) & ~(bits >> (16 + 4 * quad)) & 0xFu;
            uint4 m = make_uint4(~0u, ~0u, ~0u, ~0u);
            if (need && e.x >= 0) m = A.masks[(size_t)e.x * 128 + r];
            return m;
        };
        uint4 pf = make_uint4(~0u, ~0u, ~0u, ~0u);     // mask of the next entry to process
        {
            mbar_wait(&q_full[0], 0);
            const int4 h0 = hdr[0];
            if (h0.x >= 0 && h0.z < h0.w) pf = mask_for(entry(0, h0.z, h0.z));
        }
        while (true) {
            const int slot = qs;
            FWAIT(3, &q_full[slot], qph);            // the unit's header and entry table are published
            const int4 h4 = hdr[slot];
            if (h4.x < 0) break;
            const TUnit un{h4.x, h4.y, h4.z, h4.w, KS ? reinterpret_cast<const int *>(smem + C::OFF_HDR2)[g * C::QS + slot] : 0};
            if (++qs == C::QS) { qs = 0; qph ^= 1; }
            const int j0 = un.j0, j1 = un.j1;
#define SPLAT_NEXT_UNIT_PREFETCH()                                                                      \
    do {                                                                                                \
        mbar_wait(&q_full[qs], qph);                                                                    \
        const int4 hn = hdr[qs];                                                                        \
        if (hn.x >= 0 && hn.z < hn.w) pf = mask_for(entry(qs, hn.z, hn.z));                            \
    } while (0)
            float m_run = -INFINITY, l_run = 0.f;
            bool first = true;
            if (j0 == j1) {
                SPLAT_NEXT_UNIT_PREFETCH();
                if (pe_on) { epilogue(pe_l, KS ? *pe_m_s : 0.f, pe_t, pe_bh, KS ? *pe_sp_s : 0); pe_on = false; }
                epilogue(0.f, 0.f, un.t, un.bh, 0);
                mbar_arrive(&q_empty[slot]);
                continue;
            }
            for (int j = j0; j < j1; ++j) {
                if (store_leader) TRACE(2 + g, 5);
                const uint4 m4 = pf;
                const uint32_t bits = (uint32_t)entry(slot, j0, j).y;
                if (j + 1 < j1) pf = mask_for(entry(slot, j0, j + 1));
                else SPLAT_NEXT_UNIT_PREFETCH();
                const uint32_t mk[4] = {m4.x, m4.y, m4.z, m4.w};
                // chunk bits of this warp, broadcast so the per-chunk branches are provably uniform
                const uint32_t live4 = (bits >> (4 * quad)) & 0xFu, need4 = live4 & ~(bits >> (16 + 4 * quad));
                const uint32_t wbits = __shfl_sync(0xffffffffu, live4 | (need4 << 4), 0);
                uint32_t live = wbits & 0xFu;
                const uint32_t need = (wbits >> 4) & 0xFu;
                FWAIT(0, s_full, s_cnt & 1);
                ++s_cnt;
                tc_fence_after();
                if (store_leader) TRACE(2 + g, 2);
                float mx = -INFINITY;
                float sv[128];
                // the whole S row -> registers (one wait: under MMA traffic the TMEM load latency,
                // not the max, dominates), then S goes back to the MMA warp
                tmem_ld32(s_tm, sv);
                tmem_ld32(s_tm + 32, sv + 32);
                tmem_ld32(s_tm + 64, sv + 64);
                tmem_ld32(s_tm + 96, sv + 96);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(s_empty);
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    if (live & (1u << w)) {
                        if (need & (1u << w)) apply_mask(sv + 32 * w, mk[w]);
                        mx = fmax3(mx, max32(sv + 32 * w), -INFINITY);
                    }
                }
                if (store_leader) TRACE(2 + g, 12);
                mx *= c2;
#ifdef SPLAT_X_NOMAX
                mx = sv[0] * c2 + 1.f;      // ablation (diagnostics build only): no row max
#endif
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
                const uint64_t cc = pack2(c2, c2), mm = pack2(-mref, -mref);
                uint64_t acc0 = pack2(0.f, 0.f), acc1 = acc0;
                if DBG(2) live = 0;
                uint32_t pw[64];
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    if (live & (1u << w)) {
                        exp32(sv + 32 * w, cc, mm, acc0, acc1, pw + 16 * w);
                    } else {
#pragma unroll
                        for (int x = 0; x < 16; ++x) pw[16 * w + x] = 0u;
                    }
                }
                if (store_leader) TRACE(2 + g, 13);
                if (pe_on) {             // the previous unit's epilogue (first tile of a unit only)
                    epilogue(pe_l, KS ? *pe_m_s : 0.f, pe_t, pe_bh, KS ? *pe_sp_s : 0);
                    pe_on = false;
                }
                if (s_cnt > 1) {
                    // PV of this group's previous entry: complete before O is rescaled or P rewritten
                    FWAIT(1, pv_done, (s_cnt - 2) & 1);
                    tc_fence_after();
                }
                if (store_leader) TRACE(2 + g, 14);
                if (!first && __any_sync(0xffffffffu, resc)) {
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        float o[32];
                        tmem_ld32(o_tm + c * 32, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int x = 0; x < 32; ++x) o[x] *= alpha;
                        tmem_st32(o_tm + c * 32, o);
                    }
                }
                tmem_st32(p_tm, reinterpret_cast<const float *>(pw));
                tmem_st32(p_tm + 32, reinterpret_cast<const float *>(pw + 32));
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
                if (store_leader) TRACE(2 + g, 4);
                first = false;
            }
#undef SPLAT_NEXT_UNIT_PREFETCH
            mbar_arrive(&q_empty[slot]);   // header + entry table of this slot consumed (every thread)
            pe_on = true;
            pe_l = l_run;
            if (KS) *pe_m_s = m_run;
            pe_t = un.t;
            pe_bh = un.bh;
            if (KS) *pe_sp_s = un.split;  // every lane of the warp writes the same value
        }
        if (pe_on) epilogue(pe_l, KS ? *pe_m_s : 0.f, pe_t, pe_bh, KS ? *pe_sp_s : 0);
        if (store_leader) bulk_wait0();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
#ifdef SPLAT_FUSED_PROF
    if (blockIdx.x == 0 && lane == 0) g_fprof[warp][15] = clock64() - t_start;
#endif
    // the last CTA to finish resets the work counter for the next launch on this handle (every
    // grab of every CTA happened before its increment of the done counter)
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(prm.sched + 1, 1ull) == (unsigned long long)gridDim.x - 1ull) {
            prm.sched[0] = 0ull;
            prm.sched[1] = 0ull;
            __threadfence();
        }
    }
}

// ---------------------------------------------------------------- host side
// Residue-decomposition pass arguments (Params::view / merge); all zero for a plain launch.
struct ResidueArgs {
    int view = 0, merge = 0, R = 0, nk = 0, l = 0;
    float *lse = nullptr;
    // one-launch decomposition (view = 2): pairs of the strided / band pass in the merged plan,
    // lag in heads, dependency counters of the launch slot
    int u1 = 0, u2 = 0, lag = 0;
    unsigned *dep = nullptr;
};

template <int D, int VM>
cudaError_t set_smem_once()
{
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        const cudaError_t e = cudaFuncSetAttribute(mhsa_tc_kernel<D, VM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   Cfg<D>::SMEM);
        if (e != cudaSuccess) return e;
        attr_set[dev & 63] = true;
    }
    return cudaSuccess;
}

template <int D>
cudaError_t launch_d(const DevAcsr &A, const void *Q, const void *K, const void *V, int BH, float scale, void *O,
                     cudaStream_t st, const ResidueArgs &ra = ResidueArgs())
{
    CUtensorMap mq, mk, mv, mo, mq2, mk2, mv2, mo2;
    if (ra.view) {
        if (!make_map_residue(&mq, Q, BH, A.n, D, ra.l, ra.nk, ra.R) || !make_map_residue(&mk, K, BH, A.n, D, ra.l, ra.nk, ra.R) ||
            !make_map_residue(&mv, V, BH, A.n, D, ra.l, ra.nk, ra.R) || !make_map_residue(&mo, O, BH, A.n, D, ra.l, ra.nk, ra.R))
            return cudaErrorInvalidValue;
    } else if (!make_map(&mq, Q, BH, A.n, D) || !make_map(&mk, K, BH, A.n, D) || !make_map(&mv, V, BH, A.n, D) ||
               !make_map(&mo, O, BH, A.n, D)) {
        return cudaErrorInvalidValue;
    }
    if (ra.view == 2) {
        if (!make_map(&mq2, Q, BH, A.n, D) || !make_map(&mk2, K, BH, A.n, D) || !make_map(&mv2, V, BH, A.n, D) ||
            !make_map(&mo2, O, BH, A.n, D))
            return cudaErrorInvalidValue;
    } else {
        mq2 = mq; mk2 = mk; mv2 = mv; mo2 = mo;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    {
        cudaError_t e;
#ifdef SPLAT_DIAG
        if constexpr (D == 128) e = ra.view == 2 ? set_smem_once<D, 2>() : ra.view ? set_smem_once<D, 1>() : set_smem_once<D, 0>();
        else
#endif
            e = ra.view == 2 ? cudaErrorNotSupported : ra.view ? set_smem_once<D, 1>() : set_smem_once<D, 0>();
        if (e != cudaSuccess) return e;
    }
    Params p{};
    p.A = A;
    p.BH = BH;
    p.N = A.n;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.O = reinterpret_cast<__nv_bfloat16 *>(O);
    static const int dbg = diag_env("SPLAT_TC_DEBUG");
    p.dbg = dbg;
    p.view = ra.view;
    p.merge = ra.merge;
    p.rv_R = ra.R;
    p.rv_nk = ra.nk;
    p.rv_sh = 0;
    while ((1 << p.rv_sh) < ra.nk) ++p.rv_sh;
    p.rv_l = ra.l;
    p.lse = ra.lse;
    p.mix_u1 = ra.u1;
    p.mix_u2 = ra.u2;
    p.mix_lag = ra.lag;
    p.dep = ra.dep;
    p.dep_target = A.n_qt;          // strided-pass tiles per head
    const long long units = (long long)A.n_pairs * BH;
    const int grid = (int)(units < num_sms(dev) ? units : num_sms(dev));
    if (ra.view == 2) {
#ifdef SPLAT_DIAG
        if constexpr (D == 128)
            mhsa_tc_kernel<D, 2><<<grid, kThreads, Cfg<D>::SMEM, st>>>(mq, mk, mv, mo, mq2, mk2, mv2, mo2, p);
        else
#endif
            return cudaErrorNotSupported;
    } else if (ra.view)
        mhsa_tc_kernel<D, 1><<<grid, kThreads, Cfg<D>::SMEM, st>>>(mq, mk, mv, mo, mq2, mk2, mv2, mo2, p);
    else
        mhsa_tc_kernel<D, 0><<<grid, kThreads, Cfg<D>::SMEM, st>>>(mq, mk, mv, mo, mq2, mk2, mv2, mo2, p);
    return cudaGetLastError();
}

cudaError_t launch_split64(const DevAcsr &A, const void *Q, const void *K, const void *V, int BH, float scale,
                           void *O, cudaStream_t st)
{
    CUtensorMap mq, mk, mv, mo, mk64, mv64;
    // Q and O move as two 64-row segments per tile (row classes), K and V as 128-row key windows, or as
    // two 64-row key blocks for a composite window (two distant half-live blocks, plan.cpp)
    if (!make_map(&mq, Q, BH, A.n, 64, 64) || !make_map(&mk, K, BH, A.n, 64) || !make_map(&mv, V, BH, A.n, 64) ||
        !make_map(&mo, O, BH, A.n, 64, 64) || !make_map(&mk64, K, BH, A.n, 64, 64) || !make_map(&mv64, V, BH, A.n, 64, 64))
        return cudaErrorInvalidValue;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(mhsa_split_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCfg::SMEM);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(mhsa_split_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCfg::SMEM);
        if (e != cudaSuccess) return e;
        attr_set[dev & 63] = true;
    }
    Params p{};
    p.A = A;
    p.BH = BH;
    p.N = A.n;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.O = reinterpret_cast<__nv_bfloat16 *>(O);
    static const int dbg = diag_env("SPLAT_TC_DEBUG");
    p.dbg = dbg;
    p.sched = A.sched;
    if (!p.sched) return cudaErrorInvalidValue;
    p.A.n_ksplit = 0;
    static const int no_ks = diag_env("SPLAT_NO_KSPLIT");      // diagnostics build only
    if (A.n_ksplit > 0 && A.t_n_ks > 0 && !no_ks) {
        // split-K list when the longest whole tile would outlast a tile group's average share of the
        // work (few heads per GPU, e.g. a rank of a sharded job): DESIGN.md section 8
        const double avg = (double)BH * A.t_entries / (2.0 * num_sms(dev));
        if ((double)A.t_max_len > avg && BH <= kSplitHeads) {     // the slot's scratch holds kSplitHeads heads
            if (!A.ks_o || !A.ks_lse || !A.ks_cnt) return cudaErrorInvalidValue;
            p.A.n_ksplit = A.n_ksplit;
            p.A.t_info = A.t_info_ks;
            p.A.t_n = A.t_n_ks;
            p.A.t_n_buckets = A.t_n_buckets_ks;
            for (int b = 0; b <= A.t_n_buckets_ks && b <= kMaxBuckets; ++b) p.A.t_bucket_start[b] = A.t_bucket_start_ks[b];
        }
    }
    const long long units = (long long)p.A.t_n * BH;
    const long long ctas = (units + 1) / 2;
    const int grid = (int)(ctas < num_sms(dev) ? ctas : num_sms(dev));
    if (p.A.n_ksplit > 0) mhsa_split_kernel<true><<<grid, kThreads, SCfg::SMEM, st>>>(mq, mk, mv, mo, mk64, mv64, p);
    else mhsa_split_kernel<false><<<grid, kThreads, SCfg::SMEM, st>>>(mq, mk, mv, mo, mk64, mv64, p);
    return cudaGetLastError();
}

}  // namespace

#ifdef SPLAT_DIAG
extern "C" int splat_debug_hang(unsigned long long *out)
{
#ifdef SPLAT_HANG_DEBUG
    cudaMemcpyFromSymbol(out, sm100::g_hang, sizeof(sm100::g_hang));
    return 1;
#else
    (void)out;
    return 0;
#endif
}

extern "C" int splat_debug_fused_prof(unsigned long long *out)
{
#ifdef SPLAT_FUSED_PROF
    cudaMemcpyFromSymbol(out, g_fprof, sizeof(g_fprof));
    static const unsigned long long z[12 * 16] = {};
    cudaMemcpyToSymbol(g_fprof, z, sizeof(z));
    return 0;
#else
    (void)out;
    return 1;
#endif
}

extern "C" int splat_debug_trace(unsigned long long *out, int *counts)
{
    cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace));
    cudaMemcpyFromSymbol(counts, g_trace_n, sizeof(g_trace_n));
    int z[6] = {0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_trace_n, z, sizeof(z));
    return 0;
}
#endif  // SPLAT_DIAG

cudaError_t launch_mhsa_tc_residue1(const DevAcsr &mix, int u1, int u2, int l, int nk, int R, float *lse, unsigned *dep,
                                    const void *Q, const void *K, const void *V, int BH, int d, float scale, void *O,
                                    cudaStream_t st, int *n_launch)
{
    *n_launch = 1;
    if (d != 128 || BH > kLseHeads || !dep) return cudaErrorNotSupported;
    ResidueArgs r;
    r.view = 2;
    r.R = R;
    r.nk = nk;
    r.l = l;
    r.lse = lse;
    r.u1 = u1;
    r.u2 = u2;
    r.dep = dep;
    // lag: about 1.5 waves of units between a head's strided units and its band units, so the band
    // units rarely wait and the head's Q / K / V / O_s are still in L2 when they run
    int dev = 0;
    cudaGetDevice(&dev);
    const int per_head = u1 + u2 > 0 ? u1 + u2 : 1;
    r.lag = (3 * num_sms(dev) / 2 + per_head - 1) / per_head;
    if (const int lag = diag_env("SPLAT_MIX_LAG"); lag > 0) r.lag = lag;     // diagnostics build only
    if (r.lag < 1) r.lag = 1;
    return launch_d<128>(mix, Q, K, V, BH, scale, O, st, r);
}

cudaError_t launch_mhsa_tc_residue(const DevAcsr &band, const DevAcsr &str, int l, int nk, int R, float *lse,
                                   const void *Q, const void *K, const void *V, int BH, int d, float scale, void *O,
                                   cudaStream_t st, int *n_launch)
{
    *n_launch = 2;
    if (d != 128) return cudaErrorNotSupported;
    ResidueArgs r1;
    r1.view = 1;
    r1.R = R;
    r1.nk = nk;
    r1.l = l;
    r1.lse = lse;
    cudaError_t e = launch_d<128>(str, Q, K, V, BH, scale, O, st, r1);     // pass 1: strided keys, residue-major
    if (e != cudaSuccess) return e;
    ResidueArgs r2;
    r2.merge = 1;
    r2.lse = lse;
    return launch_d<128>(band, Q, K, V, BH, scale, O, st, r2);           // pass 2: causal band + merge
}

// Plain STRIDED(l) with nk | 128 (R whole classes per 128-row tile) or 128 | nk (a tile inside one
// class): the BLOCKED(nk) handle of the permuted mask on residue-major views; no lse, the
// epilogue writes O / l directly.
cudaError_t launch_mhsa_tc_permuted(const DevAcsr &perm, int l, int nk, int R, const void *Q, const void *K,
                                    const void *V, int BH, int d, float scale, void *O, cudaStream_t st,
                                    int *n_launch)
{
    *n_launch = 1;
    ResidueArgs r;
    r.view = 1;
    r.R = R;
    r.nk = nk;
    r.l = l;
    if (d == 64) return launch_d<64>(perm, Q, K, V, BH, scale, O, st, r);
    if (d == 128) return launch_d<128>(perm, Q, K, V, BH, scale, O, st, r);
    return cudaErrorNotSupported;
}

cudaError_t launch_mhsa_tc(const DevAcsr &A, const void *Q, const void *K, const void *V, int BH, int d,
                           float scale, void *O, cudaStream_t st, int *n_launch)
{
    *n_launch = 1;
    // d = 64: the split-group kernel.  Diagnostics build only: SPLAT_TC_PAIRED64=1 runs the paired
    // kernel, =3 the half-row double-buffered kernel of tc_fused64.cu (experimental)
    static const int alt64 = diag_env("SPLAT_TC_PAIRED64");
    if (d == 64 && alt64 == 0) return launch_split64(A, Q, K, V, BH, scale, O, st);
#ifdef SPLAT_DIAG
    if (d == 64 && alt64 == 3) return launch_mhsa64(A, Q, K, V, BH, scale, O, st);
#endif
    if (d == 64) return launch_d<64>(A, Q, K, V, BH, scale, O, st);
    if (d == 128) return launch_d<128>(A, Q, K, V, BH, scale, O, st);
    return cudaErrorNotSupported;
}

}  // namespace splat
