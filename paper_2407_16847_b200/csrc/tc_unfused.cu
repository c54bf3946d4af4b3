// tc_unfused.cu -- R-SDDMM and R-SpMM on sm_100a tensor cores, bf16.
//
// The paper's primitives (Listing 1 P:412-431 and the R-SpMM listing P:553-568) run one SIMT
// thread per output point.  Here the dense 128x128 sub-tiles of the contractions named by the
// tile plan (span specialisation) go through tcgen05, and the sparse side (the ACSR
// value arrays S and P, laid out row by row) is moved with coalesced accesses:
//
//   R-SDDMM : S_tile^T = K_j Q_t^T (TMA -> 128B-swizzled SMEM -> tcgen05.mma -> TMEM).  In the
//             transposed accumulator a TMEM lane is a key column and a TMEM column a query row,
//             so after tcgen05.ld a warp holds 32 consecutive key columns of each query row and
//             writes scale * S of the row's non-zeros with one coalesced store per row.  The
//             position of (row i, column c) is row_ptr[i] + (runs of row i left of the tile,
//             closed form) + (popcount of the pattern's row mask left of c).
//   R-SpMM  : a query row's non-zeros inside key tile j are one contiguous span of P (ACSR order),
//             copied with one bulk copy per (row, tile) into an SMEM staging ring and expanded into
//             a dense bf16 P tile in 128B-swizzled SMEM (zeros off the mask); O += P V_j is an
//             SS-MMA (V an MN-major operand), O accumulated in TMEM over the tile's key tiles and
//             written once as bf16.
//
// R-SDDMM runs 4 epilogue warpgroups that take the S tiles round robin (four tiles in flight per
// SM).  Work units: (b*H+h, 128-row query tile), head-major, query tiles in LPT order; persistent
// CTAs, one per SM.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sm100.cuh"

namespace splat {
namespace {

using namespace sm100;

#ifndef SPLAT_UNF_NWG
#define SPLAT_UNF_NWG 4
#endif
constexpr int kNWG = SPLAT_UNF_NWG;               // epilogue / gather warpgroups
constexpr int kThreadsU = 64 + 128 * kNWG;        // warp 0 TMA, warp 1 MMA, then the warpgroups
constexpr int kSub = 128 * 128;                   // [128 rows x 64 bf16] swizzle-128B sub-tile (16 KB)

struct ParamsU {
    DevAcsr A;
    int BH;
    float scale;
    float *S;                    // SDDMM output
    const __nv_bfloat16 *P;      // SpMM input (ACSR order)
    __nv_bfloat16 *O;            // SpMM output
    // residue decomposition of STRIDED_LOCAL (splat_acsr_s::sub_band): A is a sub-handle, the
    // S / P arrays are in the NATURAL handle's ACSR order.  pass 1: strided component on
    // residue-major views (tile row r -> natural row (t R + r / nk) + l (r % nk)); its keys are
    // the first i / l entries of the natural row.  pass 2: causal band in natural order, after
    // the row's i / l stride entries; R-SpMM adds pass 1's O.
    int pass, rv_l, rv_nk, rv_R;
    int rv_sh;                   // log2(rv_nk) (a power of two)
    const int64_t *nat_row_ptr;
    long long nat_nnz;
};

#if defined(SPLAT_UNF_PROF) && !defined(SPLAT_DIAG)
#error "SPLAT_UNF_PROF needs the diagnostics build (-DSPLAT_DIAG)"
#endif
#ifdef SPLAT_UNF_PROF
// Profiling aid (SPLAT_UNF_PROF build): cycles each warp of CTA 0 spends in barrier waits, by
// call site, and in total; read with splat_debug_unf_prof.
__device__ unsigned long long g_unf_prof[32][8];
#define PWAIT(SITE, BAR, PH)                                                                    \
    do {                                                                                        \
        const unsigned long long t0_ = clock64();                                               \
        mbar_wait(BAR, PH);                                                                     \
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)                                         \
            g_unf_prof[threadIdx.x >> 5][SITE] += clock64() - t0_;                              \
    } while (0)
// time of a code region into a wait slot of the profile (SPLAT_UNF_PROF build only)
#define PSPAN_BEGIN(V) const unsigned long long V = clock64()
#define PSPAN_END(SITE, V)                                                                      \
    do {                                                                                        \
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)                                         \
            g_unf_prof[threadIdx.x >> 5][SITE] += clock64() - (V);                              \
    } while (0)
#else
#define PWAIT(SITE, BAR, PH) mbar_wait(BAR, PH)
#define PSPAN_BEGIN(V) do { } while (0)
#define PSPAN_END(SITE, V) do { } while (0)
#endif

// predicated 4-byte global store (no branch / reconvergence per element)
__device__ __forceinline__ void st_pred_f32(float *addr, float v, uint32_t pred)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.global.f32 [%0], %1;\n\t}" ::"l"(addr), "f"(v),
                 "r"(pred)
                 : "memory");
}

// natural row of tile row r (pass 1: residue-major tile; permuted row p = 128 t + r is residue
// class p / nk, position p % nk, natural row p / nk + l (p % nk))
__device__ __forceinline__ int nat_row(const ParamsU &prm, int t, int r)
{
    const int p = t * 128 + r;
    return prm.pass == 1 ? (p >> prm.rv_sh) + prm.rv_l * (p & (prm.rv_nk - 1)) : p;
}

// 3-D (natural) or 4-D (residue-major, pass 1) load of the 128 rows starting at row `row0` (a query
// tile: 128 t; a key window: 64 kv)
__device__ __forceinline__ void load_tile_rows(const ParamsU &prm, void *dst, const CUtensorMap *m, uint64_t *bar,
                                               int c0, int row0, int bh)
{
    if (prm.pass == 1) tma_load_4d(dst, m, bar, c0, row0 & (prm.rv_nk - 1), row0 >> prm.rv_sh, bh);
    else tma_load_3d(dst, m, bar, c0, row0, bh);
}

__device__ __forceinline__ void unit_tile(const DevAcsr &A, int u, int &bh, int &t)
{
    bh = u / A.n_qt;
    t = A.order[u % A.n_qt];
}

__device__ __forceinline__ void wg_sync(int id)
{
    asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}

// number of columns of run g that lie left of column c0
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

// (b,h) element offset of tile row r's ACSR row in S / P, and the runs of the row in A's pattern
// (residue passes: the runs of the sub-pattern row, the base of the natural row)
__device__ __forceinline__ long long row_offset(const ParamsU &prm, int bh, int t, int r, RowRuns &R)
{
    const DevAcsr &A = prm.A;
    long long base;
    row_info(A, t * 128 + r, base, R);
    if (prm.pass == 0) return (long long)bh * A.nnz + base;
    const int i = nat_row(prm, t, r);
    if (i >= A.n) return 0;
    return (long long)bh * prm.nat_nnz + prm.nat_row_ptr[i] + (prm.pass == 2 ? i / prm.rv_l : 0);
}

// (b,h) element offset of tile row r's ACSR row in S / P (row_offset without the runs)
__device__ __forceinline__ long long row_base(const ParamsU &prm, int bh, int t, int r)
{
    const DevAcsr &A = prm.A;
    if (prm.pass == 0) return t * 128 + r < A.n ? (long long)bh * A.nnz + A.row_ptr[t * 128 + r] : 0ll;
    const int i = nat_row(prm, t, r);
    if (i >= A.n) return 0;
    return (long long)bh * prm.nat_nnz + prm.nat_row_ptr[i] + (prm.pass == 2 ? i / prm.rv_l : 0);
}

// ============================================================================ R-SDDMM
template <int D>
struct CfgS {
    static constexpr int kChunks = D / 64;
    static constexpr int kTileBytes = kChunks * kSub;
    static constexpr int QS = 2;
    static constexpr int KS = D == 64 ? 4 : 3;
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + QS * kTileBytes;
    // per (epilogue group, buffer, query row, key quad): {offset of the quad's first non-zero
    // relative to the tile base, row mask word of the quad} -- one LDS.64 per stored row
    static constexpr int OFF_TQ = OFF_K + KS * kTileBytes;                   // [kNWG][2][128][4] int2
    static constexpr int OFF_TBASE = OFF_TQ + kNWG * 2 * 128 * 4 * 8;       // [kNWG][2] int64
    static constexpr int OFF_BAR = OFF_TBASE + kNWG * 2 * 8;
    static constexpr int NBAR = 2 * QS + 2 * KS + 2 * kNWG;
    static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
    static_assert(SMEM <= 232448, "shared memory budget");
};

template <int D>
__global__ void __launch_bounds__(kThreadsU, 1)
rsddmm_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK, const ParamsU prm)
{
    using C = CfgS<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // pointer arithmetic on the __shared__ array keeps the state space known (LDS/STS, not generic)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *q_full = bars, *q_empty = bars + C::QS;
    uint64_t *k_full = q_empty + C::QS, *k_empty = k_full + C::KS;
    uint64_t *s_full = k_empty + C::KS, *s_empty = s_full + kNWG;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + C::NBAR);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const DevAcsr &A = prm.A;
    const int n_units = A.n_qt * prm.BH;
#ifdef SPLAT_UNF_PROF
    const unsigned long long t_start = clock64();
#endif

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::QS; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
        for (int i = 0; i < C::KS; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
        for (int i = 0; i < kNWG; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4); }
        fence_mbar_init();
        tma_prefetch(&tmQ); tma_prefetch(&tmK);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 128 * kNWG);
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
            if (qc >= C::QS) PWAIT(0, &q_empty[qi], qph ^ 1);
            if (lane == 0) {
                mbar_expect_tx(&q_full[qi], C::kTileBytes);
#pragma unroll
                for (int c = 0; c < C::kChunks; ++c)
                    load_tile_rows(prm, smem + C::OFF_Q + qi * C::kTileBytes + c * kSub, &tmQ, &q_full[qi], 64 * c, t * 128, bh);
            }
            ++qc;
            if (++qi == C::QS) { qi = 0; qph ^= 1; }
            for (int e = A.qt_ptr[t]; e < A.qt_ptr[t + 1]; ++e) {
                const int kv = A.kv[e] & kKvMask;
                if (kc >= C::KS) PWAIT(1, &k_empty[ki], kph ^ 1);
                if (lane == 0) {
                    mbar_expect_tx(&k_full[ki], C::kTileBytes);
#pragma unroll
                    for (int c = 0; c < C::kChunks; ++c)
                        load_tile_rows(prm, smem + C::OFF_K + ki * C::kTileBytes + c * kSub, &tmK, &k_full[ki], 64 * c,
                                       kv * kKvUnit, bh);
                }
                ++kc;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // S^T = K Q^T: A = K tile (M = 128 key rows), B = Q tile (N = 128 query rows), both K-major
        constexpr uint32_t idS = idesc_bf16(128, 128, false);
        const uint32_t sQ = smem_u32(smem + C::OFF_Q), sK = smem_u32(smem + C::OFF_K);
        int qi = 0, ki = 0;
        uint32_t qph = 0, kph = 0, ns = 0;   // ns: S tiles issued so far (buffer ns % kNWG)
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int bh, t;
            unit_tile(A, u, bh, t);
            PWAIT(2, &q_full[qi], qph);
            const uint32_t qb = sQ + qi * C::kTileBytes;
            for (int e = A.qt_ptr[t]; e < A.qt_ptr[t + 1]; ++e) {
                const int sb = ns % kNWG;
                PWAIT(3, &k_full[ki], kph);
                if (ns >= kNWG) PWAIT(4, &s_empty[sb], ((ns / kNWG) - 1) & 1);
                tc_fence_after();
                const uint32_t kb = sK + ki * C::kTileBytes;
                if (lane == 0) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = (kk >> 2) * kSub + (kk & 3) * 32;
                        mma_bf16_ss(tmem + sb * 128, sdesc_sw128(kb + off, 16, 1024), sdesc_sw128(qb + off, 16, 1024),
                                    idS, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(&s_full[sb]);
                    mma_commit(&k_empty[ki]);
                }
                __syncwarp();
                ++ns;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
            }
            if (lane == 0) mma_commit(&q_empty[qi]);
            __syncwarp();
            if (++qi == C::QS) { qi = 0; qph ^= 1; }
        }
    } else {
        // epilogue warpgroup eg takes S tiles i = eg, eg + kNWG, ...  Thread r of the group first
        // publishes its query row's ACSR offset and column mask for the tile; then warp quad
        // (TMEM lanes = key columns 32 quad .. 32 quad + 31) stores every query row's values.
        const int eg = (warp - 2) >> 2, quad = warp & 3, r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        int2 *tq = reinterpret_cast<int2 *>(smem + C::OFF_TQ) + eg * 2 * 128 * 4;
        const uint32_t below = (1u << lane) - 1u, lanebit = 1u << lane;
        float *const Sg = prm.S;
        const float scale = prm.scale;
        uint32_t i = 0, k = 0;   // i: CTA tile counter, k: this group's tile counter
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int bh, t;
            unit_tile(A, u, bh, t);
            const int e0 = A.qt_ptr[t], e1 = A.qt_ptr[t + 1];
            // first tile of this unit owned by eg
            int e = e0 + (int)((eg - (int)(i % kNWG) + kNWG) % kNWG);
            i += (uint32_t)(e1 - e0);
            if (e >= e1) continue;
            const int row = t * 128 + r;
            // element offset of this (b, h) slice in S: every row offset of the slice is relative to it
            const long long hbase = (long long)bh * (prm.pass ? prm.nat_nnz : A.nnz);
            RowRuns R;
            PSPAN_BEGIN(t_row);
            const long long rowoff = row_offset(prm, bh, t, r, R);
            PSPAN_END(6, t_row);
            for (; e < e1; e += kNWG) {
                PSPAN_BEGIN(t_meta);              // wait profile (SPLAT_UNF_PROF): per-tile metadata phase
                const int ent = A.kv[e];
                const int c0 = (ent & kKvMask) * kKvUnit;
                const bool partial = (ent & kPartialBit) != 0;
                const int tb = k & 1;
                uint4 m4 = make_uint4(~0u, ~0u, ~0u, ~0u);
                if (partial) m4 = A.masks[(size_t)A.kv_mask[e] * 128 + r];
                if (row >= A.n) m4 = make_uint4(0u, 0u, 0u, 0u);
                // Thread r publishes, per key quad q, the offset of row r's first non-zero in the
                // quad's 32 columns (relative to the (b, h) slice base, < 2^32 entries per head) and the
                // row mask word: one LDS.64 per stored row.
                const long long o0 = row < A.n ? rowoff + rank_before(R, c0) : hbase;
                int2 *dst = tq + (tb * 128 + r) * 4;
                const int p1 = __popc(m4.x), p2 = p1 + __popc(m4.y), p3 = p2 + __popc(m4.z);
                const int rel = (int)(uint32_t)(o0 - hbase);
                dst[0] = make_int2(rel, (int)m4.x);
                dst[1] = make_int2(rel + p1, (int)m4.y);
                dst[2] = make_int2(rel + p2, (int)m4.z);
                dst[3] = make_int2(rel + p3, (int)m4.w);
                wg_sync(1 + eg);
                PSPAN_END(6, t_meta);
                PWAIT(5, &s_full[eg], k & 1);
                tc_fence_after();
                const unsigned long long baddr = reinterpret_cast<unsigned long long>(Sg + hbase);
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    float v[32];
                    tmem_ld32(tmem + lane_off + eg * 128 + 32 * c, v);
                    tmem_wait_ld();
                    if (c == 3) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&s_empty[eg]);
                    }
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int2 q = tq[(tb * 128 + 32 * c + j) * 4 + quad];
                        const uint32_t mw = (uint32_t)q.y;
                        // unsigned 32-bit element offset from the tile base: one IMAD.WIDE.U32 per address
                        const uint32_t eo = (uint32_t)q.x + (uint32_t)__popc(mw & below);
                        st_pred_f32(reinterpret_cast<float *>(baddr + (unsigned long long)eo * 4ull), scale * v[j], mw & lanebit);
                    }
                }
                ++k;
            }
        }
    }
#ifdef SPLAT_UNF_PROF
    if (blockIdx.x == 0 && lane == 0) g_unf_prof[warp][7] = clock64() - t_start;
#endif
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 128 * kNWG);
    }
}

// ============================================================================ R-SpMM
//
// The sparse operand is P in ACSR order: the non-zeros of row i inside key tile [c0, c0 + 128) are
// the contiguous values P[row_ptr[i] + rank_before(i, c0) ...] (columns ascending, Fig. 5(b)), so a
// (row, key tile) span is one contiguous run of <= 256 bytes.  The P producer warpgroup (thread =
// query row) publishes the row's column mask and alignment shift, and each producer warp copies
// its 32 rows' spans (16-byte aligned supersets, one coalesced cp.async request per row) into a
// staging ring in SMEM -- a tile (up to 32 KB) in flight while the previous one completes, no
// registers held.  (One
// cp.async.bulk per row was tried: the TMA unit takes ~80 cycles per small copy, 0.71 ms on
// Longformer.)  Two expander warpgroups take the
// staged tiles in turn and scatter them into a dense 128B-swizzled bf16 P tile (lane = 4 columns:
// one unaligned 8-byte read from the staged row, a byte permute by the 4-bit mask nibble, zeros
// off the mask).  O += P V_j is an SS-MMA (V an MN-major operand), O accumulated in TMEM over the
// query tile's key tiles and written once as bf16.
//
//   warp 0 : V producer (TMA)            warp 1 : MMA issuer
//   warps 4-7   : epilogue (thread = query row = TMEM lane)
//   warps 8-15          : P producer (warp w: rows 16 (w - 8) .. +15, lane = row for the row table;
//                         a stage is published one entry late, when its cp.async group completes;
//                         one warp's copies issue at ~one 272-byte request per 125 cycles, so eight
//                         warps share each tile)
//   warps 16-19, 20-23  : expanders (entry k -> expander k % 2, dense P buffer k % 2)
constexpr int kNExp = 2;
constexpr int kThreadsP = 768;
constexpr int kStgRow = 272;                      // staged row: 256 bytes + 16-byte alignment slack

template <int D>
struct CfgP {
    static constexpr int kChunks = D / 64;
    static constexpr int kTileBytes = kChunks * kSub;                 // V tile
#ifndef SPLAT_SPMM_KS64
#define SPLAT_SPMM_KS64 3
#endif
#ifndef SPLAT_SPMM_NSTG
#define SPLAT_SPMM_NSTG 4
#endif
    static constexpr int KS = D == 64 ? SPLAT_SPMM_KS64 : 2;          // V ring
    static constexpr int NSTG = D == 64 ? SPLAT_SPMM_NSTG : 4;        // P staging ring
    static constexpr int OFF_V = 0;
    static constexpr int OFF_STG = OFF_V + KS * kTileBytes;           // [NSTG][128 rows][kStgRow]
    // [NSTG][128 rows][16 column groups of 8] u16: low byte = staged element index of the group's
    // first live value, high byte = the group's 8 mask bits
    static constexpr int OFF_RM = OFF_STG + NSTG * 128 * kStgRow;
    static constexpr int OFF_BAR = OFF_RM + NSTG * 128 * 32;
    static constexpr int NBAR = 2 * KS + 2 * NSTG + 2 * kNExp + 4;
    static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16;   // the dynamic buffer is 1024-aligned (checked)
    // TMEM: O double buffer [0, 2D), then the dense P tile of each expander (128 keys as 64
    // columns of bf16 pairs) at 2D + 64 x
    static constexpr int TMEM_COLS = 2 * D + kNExp * 64 <= 256 ? 256 : 512;
    static_assert(SMEM <= 232448, "shared memory budget");
    static_assert(OFF_STG % 16 == 0 && OFF_RM % 16 == 0 && OFF_BAR % 8 == 0, "alignment");
};

template <int D>
__global__ void __launch_bounds__(kThreadsP, 1)
rspmm_tc_kernel(const __grid_constant__ CUtensorMap tmV, const ParamsU prm)
{
    using C = CfgP<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // no static shared memory precedes the dynamic buffer, so it starts 1024-byte aligned (checked)
    uint8_t *smem = smem_raw;
    if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u) != 0u) __trap();
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *v_full = bars, *v_empty = bars + C::KS;
    uint64_t *stg_full = v_empty + C::KS, *stg_empty = stg_full + C::NSTG;
    uint64_t *p_full = stg_empty + C::NSTG, *p_empty = p_full + kNExp;
    uint64_t *o_full = p_empty + kNExp, *o_empty = o_full + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + C::NBAR);
    uint8_t *rrec = smem + C::OFF_RM;      // [NSTG][128][32] bytes
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const DevAcsr &A = prm.A;
    const int n_units = A.n_qt * prm.BH;
#ifdef SPLAT_UNF_PROF
    const unsigned long long t_start = clock64();
#endif

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::KS; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); }
        // every producer thread publishes its own copies and row-record writes (stg_full), every
        // expander thread its reads of the stage (stg_empty): each writer / reader arrives itself
        // stg_full: per producer thread one arrival (its row-record writes) and one cp.async arrive-on
        // (its copies) per stage use
        for (int i = 0; i < C::NSTG; ++i) { mbar_init(&stg_full[i], 512); mbar_init(&stg_empty[i], 128); }
        for (int i = 0; i < kNExp; ++i) { mbar_init(&p_full[i], 128); mbar_init(&p_empty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&o_full[i], 1); mbar_init(&o_empty[i], 4); }
        fence_mbar_init();
        tma_prefetch(&tmV);
    }
    if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;     // O buffers at columns [0, D), [D, 2D)

    if (warp == 0) {
        int ki = 0, kc = 0;
        uint32_t kph = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int bh, t;
            unit_tile(A, u, bh, t);
            for (int e = A.qt_ptr[t]; e < A.qt_ptr[t + 1]; ++e) {
                const int kv = A.kv[e] & kKvMask;
                if (kc >= C::KS) PWAIT(0, &v_empty[ki], kph ^ 1);
                if (lane == 0) {
                    mbar_expect_tx(&v_full[ki], C::kTileBytes);
#pragma unroll
                    for (int c = 0; c < C::kChunks; ++c)
                        load_tile_rows(prm, smem + C::OFF_V + ki * C::kTileBytes + c * kSub, &tmV, &v_full[ki], 64 * c,
                                       kv * kKvUnit, bh);
                }
                ++kc;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idO = idesc_bf16(128, D, true);
        const uint32_t sV = smem_u32(smem + C::OFF_V);
        int ki = 0;
        uint32_t kph = 0, np = 0, uo = 0;   // np: P tiles consumed; uo: units started
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++uo) {
            int bh, t;
            unit_tile(A, u, bh, t);
            const int ob = uo & 1;
            if (uo >= 2) PWAIT(1, &o_empty[ob], ((uo >> 1) - 1) & 1);
            bool first = true;
            for (int e = A.qt_ptr[t]; e < A.qt_ptr[t + 1]; ++e) {
                const int pb = np % kNExp;
                PWAIT(2, &v_full[ki], kph);
                PWAIT(3, &p_full[pb], (np / kNExp) & 1);
                ++np;
                tc_fence_after();
                const uint32_t vb = sV + ki * C::kTileBytes, pt = tmem + 2 * D + 64 * pb;
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16_ts(tmem + ob * D, pt + kk * 8, sdesc_sw128(vb + kk * 2048, kSub, 1024), idO,
                                    (first && kk == 0) ? 0u : 1u);
                    mma_commit(&v_empty[ki]);
                    mma_commit(&p_empty[pb]);
                }
                __syncwarp();
                first = false;
                if (++ki == C::KS) { ki = 0; kph ^= 1; }
            }
            if (elect_one()) mma_commit(&o_full[ob]);
            __syncwarp();
        }
    } else if (warp >= 8 && warp < 16) {
        // ---------------------------------------------------------------- P producers: thread = row r
        const int r = (warp - 8) * 16 + (lane & 15);   // lanes 16-31 mirror lanes 0-15
        const unsigned char *Pb = reinterpret_cast<const unsigned char *>(prm.P);
        const long long total_b = 2ll * (long long)prm.BH * (prm.pass ? prm.nat_nnz : A.nnz);   // bytes of P
        const long long end_a = total_b & ~15ll;       // bulk copies stay below this (16-byte granules)
        uint32_t k = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int bh, t;
            unit_tile(A, u, bh, t);
            const int e0 = A.qt_ptr[t], e1 = A.qt_ptr[t + 1];
            PSPAN_BEGIN(t_unit);
            // The unit's entries are in ascending key-tile order and cover each row's non-zeros
            // exactly once, so the rank of the row's first non-zero in entry e is the running sum of
            // its non-zero counts in the entries before it.
            const long long rowoff = row_base(prm, bh, t, r);
            const bool rvalid = t * 128 + r < A.n;
            long long run = 0;
            // the unit's plan words and mask ids, lane l holding entry e0 + l (the warp's copy is
            // broadcast by shuffle; entries past 32 are read from global memory); a PARTIAL entry's
            // row record (precomputed per mask by the planner: live columns before each 8-column
            // group, the group's bits) and live count are loaded one entry ahead
            const int ne = e1 - e0;
            const int ent_l = lane < ne ? A.kv[e0 + lane] : 0;
            const int mid_l = lane < ne ? A.kv_mask[e0 + lane] : -1;
            auto ent_of = [&](int i) { return i < 32 ? __shfl_sync(0xffffffffu, ent_l, i) : A.kv[e0 + i]; };
            auto rec_of = [&](int i, int en, uint4 &rc, int &cn) {
                if (en & kPartialBit) {
                    const int mid = i < 32 ? __shfl_sync(0xffffffffu, mid_l, i) : A.kv_mask[e0 + i];
                    rc = A.mask_rec[((size_t)mid * 128 + r) * 2 + (lane >> 4)];
                    cn = A.mask_cnt[(size_t)mid * 128 + r];
                } else {
                    // FULL entry: every group of a valid row is live, group g starts at 8 g
                    const uint32_t b8 = rvalid ? 0xFF00u : 0u, g0 = lane < 16 ? 0u : 64u;
                    rc = make_uint4((g0 | b8) | ((g0 + 8u) | b8) << 16, ((g0 + 16u) | b8) | ((g0 + 24u) | b8) << 16,
                                    ((g0 + 32u) | b8) | ((g0 + 40u) | b8) << 16, ((g0 + 48u) | b8) | ((g0 + 56u) | b8) << 16);
                    cn = rvalid ? 128 : 0;
                }
            };
            int ent = ne > 0 ? ent_of(0) : 0;
            uint4 rc4 = make_uint4(0u, 0u, 0u, 0u);
            int cn4 = 0;
            if (ne > 0) rec_of(0, ent, rc4, cn4);
            PSPAN_END(3, t_unit);
            for (int e = e0; e < e1; ++e, ++k) {
                const uint4 rc = rc4;
                const int cnt = cn4;
                if (e + 1 < e1) {
                    ent = ent_of(e + 1 - e0);
                    rec_of(e + 1 - e0, ent, rc4, cn4);
                }
                const int s = k % C::NSTG;
                if (k >= C::NSTG) PWAIT(4, &stg_empty[s], ((k / C::NSTG) - 1) & 1);
                const long long b0 = 2ll * (rowoff + run), b1 = b0 + 2ll * cnt;
                run += cnt;
                const long long a0 = b0 & ~15ll;
                long long a1 = (b1 + 15) & ~15ll;
                uint8_t *srow = smem + C::OFF_STG + (s * 128 + r) * kStgRow;
                uint32_t bytes = 0;
                if (cnt > 0) {
                    if (a1 > end_a && lane < 16) {
                        // the last row of P: the bytes past the last full 16-byte granule are copied
                        // by this thread (a bulk copy may not read past the end of the buffer)
                        for (long long x = (a0 > end_a ? a0 : end_a); x < b1; x += 2)
                            *reinterpret_cast<unsigned short *>(srow + (x - a0)) =
                                *reinterpret_cast<const unsigned short *>(Pb + x);
                        a1 = end_a > a0 ? end_a : a0;
                    }
                    bytes = (uint32_t)(a1 - a0);
                }
                {
                    // row record: lanes 0-15 write column groups 0-7, lanes 16-31 groups 8-15 of row r;
                    // the span's element shift in its staged row is added to every group's index
                    const uint32_t sh2 = (uint32_t)((b0 - a0) >> 1) * 0x00010001u;
                    *reinterpret_cast<uint4 *>(rrec + (s * 128 + r) * 32 + (lane >> 4) * 16) =
                        make_uint4(rc.x + sh2, rc.y + sh2, rc.z + sh2, rc.w + sh2);
                }
                // The warp copies its 16 rows' spans (16-byte granules, <= 17 per row, coalesced).
                PSPAN_BEGIN(t_copy);
                const uint32_t ng = bytes >> 4;
                const uint32_t stg_row0 = (uint32_t)(s * 128 + (warp - 8) * 16) * kStgRow;
                // two rows per instruction (half-warp hh: row rr + 8 hh, lane l16: granule l16), then
                // the 17th granule of all 16 rows (a span not 16-byte aligned) in one instruction
                {
                    const int hh = lane >> 4, l16 = lane & 15;
#pragma unroll 4
                    for (int rr = 0; rr < 8; ++rr) {
                        const int row = rr + 8 * hh;
                        const uint32_t n_rr = __shfl_sync(0xffffffffu, ng, row);
                        const long long a_rr = __shfl_sync(0xffffffffu, a0, row);
                        if ((uint32_t)l16 < n_rr)
                            cp_async16(smem + C::OFF_STG + stg_row0 + row * kStgRow + 16 * l16, Pb + a_rr + 16 * l16);
                    }
                    if (lane < 16 && ng > 16u)
                        cp_async16(smem + C::OFF_STG + stg_row0 + lane * kStgRow + 256, Pb + a0 + 256);
                }
                cp_async_mbar_arrive_noinc(&stg_full[s]);   // fires when this thread's copies land
                mbar_arrive(&stg_full[s]);                  // releases this thread's record writes
                PSPAN_END(5, t_copy);
            }
        }
    } else if (warp >= 16) {
        // ---------------------------------------------------------------- expanders
        // expander x takes entries k = x, x + 2, ...; warp q of it fills rows q, q + 4, ... (rows
        // with many non-zeros, e.g. Longformer's global rows, all in the first 32 rows of tile 0,
        // are spread over the four warps).  Lane l owns columns 4l .. 4l + 3.
        // Thread = query row = TMEM lane (warp q of the expander owns lanes 32 q .. 32 q + 31): the
        // thread expands its own row, 8 columns (one group of its row record) at a time, from the
        // staged span into bf16 pairs and writes them to the expander's P tile in TMEM (64 columns)
        // with tcgen05.st; the MMA reads P from TMEM (TS form).
        const int x = (warp - 16) >> 2, q = warp & 3, r = q * 32 + lane;
        const uint32_t p_tm = tmem + ((uint32_t)(q * 32) << 16) + 2 * D + 64 * x;
        uint32_t k = 0, j = 0;     // k: CTA entry counter, j: this expander's tile counter
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
          int bh, t;
          unit_tile(A, u, bh, t);
          const uint32_t kend = k + (uint32_t)(A.qt_ptr[t + 1] - A.qt_ptr[t]);
          for (k += (uint32_t)((x - (int)(k % kNExp) + kNExp) % kNExp); k < kend; k += kNExp, ++j) {
            const int s = k % C::NSTG;
            PWAIT(5, &stg_full[s], (k / C::NSTG) & 1);
            if (j >= 1) PWAIT(6, &p_empty[x], (j - 1) & 1);
            tc_fence_after();
            PSPAN_BEGIN(t_rows);
            const uint8_t *srow = smem + C::OFF_STG + (s * 128 + r) * kStgRow;
            const uint4 *rp4 = reinterpret_cast<const uint4 *>(rrec + (s * 128 + r) * 32);
            const uint4 ra = rp4[0], rb = rp4[1];
            const uint32_t rw[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {          // 4 groups = 32 keys = 16 TMEM columns per store
                uint32_t pk[16];
#pragma unroll
                for (int gg = 0; gg < 4; ++gg) {
                    const int g = 4 * c4 + gg;
                    const uint32_t rc = (rw[g >> 1] >> (16 * (g & 1))) & 0xFFFFu;
                    const uint32_t byte = rc >> 8, qq = rc & 0xFFu;           // staged element index
                    // 8 values from element qq: an 8-byte-aligned 24-byte window (three LDS.64), the
                    // words shifted by the window offset (0 / 1 word, 0 / 16 bits)
                    const uint32_t b0 = 2u * qq, a8 = b0 & ~7u, o = b0 - a8;   // o in {0, 2, 4, 6}
                    const uint2 *wp = reinterpret_cast<const uint2 *>(srow + a8);
                    const uint2 u0 = wp[0], u1 = wp[1], u2 = wp[2];
                    const uint32_t w[6] = {u0.x, u0.y, u1.x, u1.y, u2.x, u2.y};
                    const uint32_t sw = o >> 2, sb = (o & 3u) * 8u;
                    uint32_t v[4];
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const uint32_t lo = sw ? w[jj + 1] : w[jj], hi = sw ? w[jj + 2] : w[jj + 1];
                        v[jj] = __funnelshift_r(lo, hi, sb);
                    }
                    if (byte != 0xFFu) {
                        if (byte == 0u) {
                            v[0] = v[1] = v[2] = v[3] = 0u;
                        } else {
                            // a group straddling a run boundary: value popc(byte & ((1 << c) - 1))
                            // into each live column c
                            const unsigned short *e = reinterpret_cast<const unsigned short *>(srow) + qq;
                            uint32_t h[8];
#pragma unroll
                            for (int c = 0; c < 8; ++c)
                                h[c] = ((byte >> c) & 1u) ? (uint32_t)e[__popc(byte & ((1u << c) - 1u))] : 0u;
#pragma unroll
                            for (int jj = 0; jj < 4; ++jj) v[jj] = h[2 * jj] | (h[2 * jj + 1] << 16);
                        }
                    }
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) pk[4 * gg + jj] = v[jj];
                }
                tmem_st16(p_tm + 16 * c4, pk);
            }
            tmem_wait_st();
            PSPAN_END(3, t_rows);
            tc_fence_before();
            // every thread publishes its own row (P tile) and releases its staged row
            mbar_arrive(&stg_empty[s]);
            mbar_arrive(&p_full[x]);
          }
          k = kend;
        }
    } else if (warp >= 4) {
        // epilogue warpgroup (warps 4..7): O of unit uo (the plain sum P V) -> bf16 -> HBM;
        // thread = query row.  O is double buffered in TMEM so the MMA runs one unit ahead.
        const int quad = warp & 3, r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        uint32_t uo = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++uo) {
            int bh, t;
            unit_tile(A, u, bh, t);
            const int row = t * 128 + r;
            const int e0 = A.qt_ptr[t], e1 = A.qt_ptr[t + 1];
            {
                const int ob = uo & 1;
                PWAIT(6, &o_full[ob], (uo >> 1) & 1);
                tc_fence_after();
                const bool empty = e0 == e1;   // no key tile: O = 0
                const int nrow = nat_row(prm, t, r);
                __nv_bfloat16 *orow = prm.O + ((size_t)bh * A.n + nrow) * D;
#pragma unroll
                for (int c = 0; c < D / 32; ++c) {
                    float o[32];
                    tmem_ld32(tmem + lane_off + ob * D + c * 32, o);
                    tmem_wait_ld();
                    if (empty) {
#pragma unroll
                        for (int x = 0; x < 32; ++x) o[x] = 0.f;
                    }
                    if (prm.pass == 2 && row < A.n) {
                        // O = O_band + O_strided (pass 1 wrote the strided part to this row)
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const uint4 w4 = *reinterpret_cast<const uint4 *>(orow + c * 32 + 8 * v);
                            const uint32_t ww[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                o[8 * v + 2 * q] += __uint_as_float(ww[q] << 16);
                                o[8 * v + 2 * q + 1] += __uint_as_float(ww[q] & 0xffff0000u);
                            }
                        }
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
                __syncwarp();
                if (lane == 0) mbar_arrive(&o_empty[ob]);
            }
        }
    }
#ifdef SPLAT_UNF_PROF
    if (blockIdx.x == 0 && lane == 0) g_unf_prof[warp][7] = clock64() - t_start;
#endif
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

int grid_for(long long units)
{
    int dev = 0;
    cudaGetDevice(&dev);
    const int sms = num_sms(dev);
    return (int)(units < sms ? units : sms);
}

template <int D>
cudaError_t launch_sddmm_d(const DevAcsr &A, const void *Q, const void *K, int BH, float scale, float *S,
                           cudaStream_t st)
{
    CUtensorMap mq, mk;
    if (!make_map(&mq, Q, BH, A.n, D) || !make_map(&mk, K, BH, A.n, D)) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(rsddmm_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgS<D>::SMEM);
    if (e != cudaSuccess) return e;
    ParamsU p{};
    p.A = A;
    p.BH = BH;
    p.scale = scale;
    p.S = S;
    rsddmm_tc_kernel<D><<<grid_for((long long)A.n_qt * BH), kThreadsU, CfgS<D>::SMEM, st>>>(mq, mk, p);
    return cudaGetLastError();
}

template <int D>
cudaError_t launch_spmm_d(const DevAcsr &A, const void *P, const void *V, int BH, void *O, cudaStream_t st)
{
    CUtensorMap mv;
    if (!make_map(&mv, V, BH, A.n, D)) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(rspmm_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgP<D>::SMEM);
    if (e != cudaSuccess) return e;
    ParamsU p{};
    p.A = A;
    p.BH = BH;
    p.P = reinterpret_cast<const __nv_bfloat16 *>(P);
    p.O = reinterpret_cast<__nv_bfloat16 *>(O);
    rspmm_tc_kernel<D><<<grid_for((long long)A.n_qt * BH), kThreadsP, CfgP<D>::SMEM, st>>>(mv, p);
    return cudaGetLastError();
}

struct UPass {
    int pass = 0, l = 0, nk = 0, R = 0;
    const int64_t *nat_row_ptr = nullptr;
    long long nat_nnz = 0;
};

void apply_pass(ParamsU &p, const UPass &ps)
{
    p.pass = ps.pass;
    p.rv_l = ps.l;
    p.rv_nk = ps.nk;
    p.rv_sh = 0;
    while ((1 << p.rv_sh) < ps.nk) ++p.rv_sh;
    p.rv_R = ps.R;
    p.nat_row_ptr = ps.nat_row_ptr;
    p.nat_nnz = ps.nat_nnz;
}

bool maps_for(CUtensorMap *m, const void *X, int BH, int N, int D, const UPass &ps)
{
    return ps.pass == 1 ? make_map_residue(m, X, BH, N, D, ps.l, ps.nk, ps.R) : make_map(m, X, BH, N, D);
}

template <int D>
cudaError_t launch_sddmm_pass(const DevAcsr &A, const UPass &ps, const void *Q, const void *K, int BH, float scale,
                              float *S, cudaStream_t st)
{
    CUtensorMap mq, mk;
    if (!maps_for(&mq, Q, BH, A.n, D, ps) || !maps_for(&mk, K, BH, A.n, D, ps)) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(rsddmm_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgS<D>::SMEM);
    if (e != cudaSuccess) return e;
    ParamsU p{};
    p.A = A;
    p.BH = BH;
    p.scale = scale;
    p.S = S;
    apply_pass(p, ps);
    rsddmm_tc_kernel<D><<<grid_for((long long)A.n_qt * BH), kThreadsU, CfgS<D>::SMEM, st>>>(mq, mk, p);
    return cudaGetLastError();
}

template <int D>
cudaError_t launch_spmm_pass(const DevAcsr &A, const UPass &ps, const void *P, const void *V, int BH, void *O,
                             cudaStream_t st)
{
    CUtensorMap mv;
    if (!maps_for(&mv, V, BH, A.n, D, ps)) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(rspmm_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgP<D>::SMEM);
    if (e != cudaSuccess) return e;
    ParamsU p{};
    p.A = A;
    p.BH = BH;
    p.P = reinterpret_cast<const __nv_bfloat16 *>(P);
    p.O = reinterpret_cast<__nv_bfloat16 *>(O);
    apply_pass(p, ps);
    rspmm_tc_kernel<D><<<grid_for((long long)A.n_qt * BH), kThreadsP, CfgP<D>::SMEM, st>>>(mv, p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_unfused_residue(bool sddmm, const DevAcsr &band, const DevAcsr &str, const DevAcsr &nat, int l,
                                   int nk, int R, const void *X, const void *Y, int BH, int d, float scale, void *out,
                                   cudaStream_t st, int *n_launch)
{
    *n_launch = 2;
    UPass p1, p2;
    p1.pass = 1;
    p2.pass = 2;
    p1.l = p2.l = l;
    p1.nk = p2.nk = nk;
    p1.R = p2.R = R;
    p1.nat_row_ptr = p2.nat_row_ptr = nat.row_ptr;
    p1.nat_nnz = p2.nat_nnz = nat.nnz;
    cudaError_t e;
    if (sddmm) {
        float *S = reinterpret_cast<float *>(out);
        if (d == 64) {
            if ((e = launch_sddmm_pass<64>(str, p1, X, Y, BH, scale, S, st)) != cudaSuccess) return e;
            return launch_sddmm_pass<64>(band, p2, X, Y, BH, scale, S, st);
        }
        if (d == 128) {
            if ((e = launch_sddmm_pass<128>(str, p1, X, Y, BH, scale, S, st)) != cudaSuccess) return e;
            return launch_sddmm_pass<128>(band, p2, X, Y, BH, scale, S, st);
        }
    } else {
        if (d == 64) {
            if ((e = launch_spmm_pass<64>(str, p1, X, Y, BH, out, st)) != cudaSuccess) return e;
            return launch_spmm_pass<64>(band, p2, X, Y, BH, out, st);
        }
        if (d == 128) {
            if ((e = launch_spmm_pass<128>(str, p1, X, Y, BH, out, st)) != cudaSuccess) return e;
            return launch_spmm_pass<128>(band, p2, X, Y, BH, out, st);
        }
    }
    return cudaErrorNotSupported;
}

// Plain STRIDED(l): only the residue-major pass, on the BLOCKED(nk) handle of the permuted mask.  The
// natural ACSR row of i holds exactly its stride keys, in the order m of the permuted block row, so
// pass 1's addressing (natural row base + rank within the sub-pattern row) is the whole S / P.
cudaError_t launch_unfused_permuted(bool sddmm, const DevAcsr &perm, const DevAcsr &nat, int l, int nk, int R,
                                    const void *X, const void *Y, int BH, int d, float scale, void *out,
                                    cudaStream_t st, int *n_launch)
{
    *n_launch = 1;
    UPass p1;
    p1.pass = 1;
    p1.l = l;
    p1.nk = nk;
    p1.R = R;
    p1.nat_row_ptr = nat.row_ptr;
    p1.nat_nnz = nat.nnz;
    if (sddmm) {
        float *S = reinterpret_cast<float *>(out);
        if (d == 64) return launch_sddmm_pass<64>(perm, p1, X, Y, BH, scale, S, st);
        if (d == 128) return launch_sddmm_pass<128>(perm, p1, X, Y, BH, scale, S, st);
    } else {
        if (d == 64) return launch_spmm_pass<64>(perm, p1, X, Y, BH, out, st);
        if (d == 128) return launch_spmm_pass<128>(perm, p1, X, Y, BH, out, st);
    }
    return cudaErrorNotSupported;
}

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

#ifdef SPLAT_UNF_PROF
extern "C" int splat_debug_unf_prof(unsigned long long *out)
{
    cudaMemcpyFromSymbol(out, splat::g_unf_prof, sizeof(splat::g_unf_prof));
    static const unsigned long long z[32 * 8] = {};
    cudaMemcpyToSymbol(splat::g_unf_prof, z, sizeof(z));
    return 0;
}
#endif
