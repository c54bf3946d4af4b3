// splat_internal.h -- internal types of the SPLAT B200 library (not part of the ABI).
#pragma once

#include <atomic>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "splat.h"

#if defined(__CUDACC__)
#define SPLAT_HD __host__ __device__ __forceinline__
#else
#define SPLAT_HD inline
#endif

namespace splat {

// Query-tile rows and key-tile columns of the tile plan (tcgen05 M = 128,
// 128-column key tiles).
constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kKvUnit = 64;          // plan entries: key window [64 kv, 64 kv + kBN)
constexpr int kPartialBit = 1 << 24;
constexpr int kKvMask = (1 << 24) - 1;
// classed (split-kernel) entries only: a composite window of two 64-column key blocks a | b << 12
constexpr int kCompBit = 1 << 25;

struct Seg {
    int32_t start, step, count;
};

// Internal pattern kind (never accepted from the ABI): the strided component of STRIDED_LOCAL(l)
// in residue-major row order.  With nk = N / l rows per residue (field `block`), permuted row
// r = rho * nk + k is natural row rho + l k, and it attends permuted keys rho * nk + m, m < k
// (natural keys j = rho + l m = i - l (k - m)): one affine run (rho nk, 1, k) per row.
constexpr int32_t kKindResiduePrev = 100;
// handles built from an explicit bit mask (splat_acsr_from_mask): no descriptor, metadata only
constexpr int32_t kKindMask = 101;
constexpr int32_t kMaxMaskN = 1 << 17;

// Diagnostics build (-DSPLAT_DIAG -> libsplat_diag.so, tools/ only): environment knobs that change
// the plan or switch kernels off for profiling.  The product library (libsplat.so) is built
// without SPLAT_DIAG: there every knob reads as 0 and no environment variable is consulted.
#ifdef SPLAT_DIAG
constexpr bool kDiag = true;
inline int diag_env(const char *name)
{
    const char *e = getenv(name);
    return e ? atoi(e) : 0;
}
#else
constexpr bool kDiag = false;
inline int diag_env(const char *) { return 0; }
#endif

SPLAT_HD int imin(int a, int b) { return a < b ? a : b; }
SPLAT_HD int imax(int a, int b) { return a > b ? a : b; }

// Canonical affine runs of row i in closed form (
// SURVEY §8(c) C-2b).  Equal, row by row, to the paper's construction --
// 2x2 solve on the first two columns, extension while consecutive
// columns pass the check of P:219, restart at the first failing column --
// applied to the row's column set; a run of one column has step 1
// (SPEC S:96).  Returns the number of runs written to s (<= 3).
// Preconditions: pattern validated by validate_pattern(), 0 <= i < N.
SPLAT_HD int row_segments(const splat_pattern &p, int i, Seg *s)
{
    const int N = p.seq_len;
    int n = 0;
#define SPLAT_ADD(st, sp, ct)                                   \
    do {                                                        \
        int c_ = (ct);                                          \
        if (c_ > 0) {                                           \
            s[n].start = (st);                                  \
            s[n].step = c_ == 1 ? 1 : (sp);                     \
            s[n].count = c_;                                    \
            ++n;                                                \
        }                                                       \
    } while (0)
    switch (p.kind) {
    case SPLAT_WINDOW: {
        int a = imax(0, i - p.lo), e = imin(N - 1, i + p.hi);
        SPLAT_ADD(a, 1, e - a + 1);
        break;
    }
    case SPLAT_BLOCKED: {
        int b0 = (i / p.block) * p.block;
        SPLAT_ADD(b0, 1, imin(p.block, N - b0));
        break;
    }
    case SPLAT_STRIDED: {
        int r = i % p.stride;
        SPLAT_ADD(r, p.stride, (N - 1 - r) / p.stride + 1);
        break;
    }
    case SPLAT_DILATED: {
        int dl = p.stride;
        int st = i - dl * imin(p.radius, i / dl);
        int en = i + dl * imin(p.radius, (N - 1 - i) / dl);
        SPLAT_ADD(st, dl, (en - st) / dl + 1);
        break;
    }
    case SPLAT_GLOBAL_LOCAL: {
        int g = p.n_global;
        int a = imax(0, i - p.lo), e = imin(N - 1, i + p.hi);
        if (i < g) {
            SPLAT_ADD(0, 1, N);
        } else if (a <= g) {
            SPLAT_ADD(0, 1, imax(e, g - 1) + 1);
        } else {
            SPLAT_ADD(0, 1, g);
            SPLAT_ADD(a, 1, e - a + 1);
        }
        break;
    }
    case SPLAT_BIGBIRD: {
        int bs = p.block, nb = (N + bs - 1) / bs, qb = i / bs;
        if (qb == 0 || qb == nb - 1) {
            SPLAT_ADD(0, 1, N);
            break;
        }
        // block runs: [0,0], [lo_b, hi_b] (sliding), [nb-1, nb-1]; merge neighbours
        int lo_b = imax(0, qb - p.radius), hi_b = imin(nb - 1, qb + p.radius);
        const int r1a = lo_b, r1b = hi_b, r2a = nb - 1;
        const bool m01 = r1a <= 1, m12 = r2a <= r1b + 1;
        if (m01 && m12) {
            SPLAT_ADD(0, 1, N);
        } else if (m01) {
            SPLAT_ADD(0, 1, imin(N, (r1b + 1) * bs));
            SPLAT_ADD(r2a * bs, 1, N - r2a * bs);
        } else if (m12) {
            SPLAT_ADD(0, 1, imin(N, bs));
            SPLAT_ADD(r1a * bs, 1, N - r1a * bs);
        } else {
            SPLAT_ADD(0, 1, imin(N, bs));
            SPLAT_ADD(r1a * bs, 1, imin(N, (r1b + 1) * bs) - r1a * bs);
            SPLAT_ADD(r2a * bs, 1, N - r2a * bs);
        }
        break;
    }
    case kKindResiduePrev: {
        const int nk = p.block;
        SPLAT_ADD((i / nk) * nk, 1, i % nk);
        break;
    }
    case SPLAT_STRIDED_LOCAL: {
        int l = p.stride;
        if (i < l || l == 1) {
            SPLAT_ADD(0, 1, i + 1);
        } else if (i / l == 1) {
            SPLAT_ADD(i - l, 1, l + 1);
        } else {
            SPLAT_ADD(i % l, l, i / l);
            SPLAT_ADD(i - l + 1, 1, l);
        }
        break;
    }
    default:
        break;
    }
#undef SPLAT_ADD
    return n;
}

// Pair-plan entry flags (the fused kernel runs two adjacent query tiles A = 2p
// and B = 2p+1 against the union of their key-tile lists, sharing K/V loads).
constexpr int kUseA = 1 << 24, kUseB = 1 << 25, kPartA = 1 << 26, kPartB = 1 << 27;
constexpr int kMaxBuckets = 24;

struct Plan {
    int bm = kBM, bn = kBN, n_qt = 0, n_entries = 0, n_kt = 0;
    int kv_align = 1;                     // window starts: multiples of kv_align * 64 columns
    int row_classes = 0;                  // split-kernel tiles regrouped by row class (plan.cpp)
    int n_split_tiles = 0;                // split-kernel work units per (b, h)
    int n_ksplit = 0, ksplit_pmax = 0;    // split-K: long tiles per (b, h) split into parts, max parts
    int t_max_len = 0;                    // entries of the longest whole-tile unit
    int t_n_buckets_ks = 0;               // the split-K unit list (t_info_ks), bucketed like t_info
    std::vector<int32_t> t_bucket_start_ks, t_info_ks;
    int32_t *d_t_info_ks = nullptr;
    std::vector<int32_t> qt_ptr, kv, order;          // per query tile (ABI: splat_plan_copy)
    // query-tile pairs
    int n_pairs = 0, n_pair_entries = 0, n_buckets = 0, n_masks = 0;
    std::vector<int32_t> pair_ptr, pair_ent, pair_order, bucket_start;
    std::vector<int32_t> pair_info;   // [n_pairs][8]: pair, e0, e1, jA0, jA1, jB1, 0, 0 -- in pair_order order
    std::vector<int32_t> pair_mask;   // [n_pair_entries][2]: mask id of tile A / B (-1: FULL or unused)
    std::vector<uint32_t> masks;      // [n_masks][128 rows][4 words]: column mask of each row
    std::vector<uint16_t> mask_rec;   // [n_masks][128 rows][16 groups]: live columns before the group | group bits << 8
    std::vector<uint8_t> mask_cnt;    // [n_masks][128 rows]: live columns of the row
    std::vector<int32_t> kv_mask;     // [n_entries]: mask id of each (query tile, key tile) entry (-1: FULL)
    std::vector<uint32_t> qt_bits;    // [n_entries]: per-warp chunk live (bits 0-15) / full (bits 16-31)
    int t_n_buckets = 0;
    std::vector<int32_t> t_bucket_start;  // single-tile units: bucket boundaries in t_info order
    std::vector<int32_t> t_info;          // [n_qt][4]: tile, j0, j1, 0 -- bucketed longest first
    int32_t *d_qt_ptr = nullptr, *d_kv = nullptr, *d_order = nullptr;
    int32_t *d_pair_ent = nullptr, *d_pair_info = nullptr;
    uint32_t *d_masks = nullptr;
    uint16_t *d_mask_rec = nullptr;
    uint8_t *d_mask_cnt = nullptr;
    int32_t *d_kv_mask = nullptr;
    uint32_t *d_qt_bits = nullptr;
    int32_t *d_t_info = nullptr;
    unsigned long long *d_sched = nullptr;   // [kLaunchSlots][2] split-kernel work / done counters
};

// Per-call device resources of a compute call (the split kernel's work counter, the residue
// decomposition's lse scratch) come from one of kLaunchSlots slots, allocated at build time.  A
// call takes the next slot round robin; the calling stream first waits for the slot's previous
// user (an event), so two streams sharing one handle never share a slot's resources at the same
// time -- correct by construction, with up to kLaunchSlots calls in flight concurrently.
constexpr int kLaunchSlots = 8;
// heads (b, h) per launch of the residue decomposition (lse scratch per slot: kLseHeads x N floats)
constexpr int kLseHeads = 64;
// split-K of the d = 64 fused kernel's long tiles (plan.cpp): entries per part, parts per tile, and
// heads per launch (the per-slot partial-result scratch holds kSplitHeads heads)
constexpr int kSplitMax = 8;
constexpr int kSplitPartsMax = 16;
constexpr int kSplitHeads = 128;
constexpr size_t kSplitScratchMax = (size_t)256 << 20;   // per handle (all launch slots)

struct LaunchSlot {
    std::mutex mu;
    void *ev = nullptr;          // cudaEvent_t recorded after the slot's last use
    bool used = false;
};

}  // namespace splat

struct splat_acsr_s {
    splat_pattern pat;
    int device = -1;
    int32_t n = 0;
    int64_t nnz = 0;
    int32_t max_segs = 0;
    // host copies (always present)
    std::vector<int32_t> seg_h;       // [N][4][4]: start, step, count, offset-in-row
    std::vector<uint8_t> nseg_h;      // [N]
    std::vector<int64_t> row_ptr_h;   // [N+1]
    // device copies (device >= 0)
    int32_t *d_seg = nullptr;         // [N][4][4] (int4 per run)
    uint8_t *d_nseg = nullptr;
    int64_t *d_row_ptr = nullptr;
    splat::Plan plan;
    // Residue decomposition of STRIDED_LOCAL(l): the mask is the
    // disjoint union of a causal band WINDOW(l-1, 0) (natural order) and the strided keys
    // i - l m, m >= 1, which become a dense strictly-causal block per residue class i mod l
    // (row classes by residue of the stride).  The fused kernel runs the
    // strided part on residue-major views of Q/K/V/O (4-D tensor maps) and merges the two
    // partial softmaxes in the band pass's epilogue.  Null when not applicable.
    splat_acsr_s *sub_band = nullptr, *sub_str = nullptr;
    // Plain STRIDED(X) with N = X nk, nk | 128 or 128 | nk: rows and keys permuted residue-major
    // (r' = (i mod X) nk + i div X) make the mask block diagonal, BLOCKED(nk) -- the residue
    // classes of the paper's stretched thread blocks (Sec. 7.3.1, App. B).  The fused bf16 path
    // runs this handle on residue-major views of Q/K/V/O; the other paths use the natural one.
    splat_acsr_s *sub_perm = nullptr;
    int32_t rv_l = 0, rv_nk = 0, rv_R = 0;   // stride, rows per residue (N / l), residues per 128-row tile
    float *d_lse = nullptr;                   // [kLaunchSlots][kLseHeads * N] log2-sum-exp of the strided pass
    // split-K scratch of the d = 64 fused kernel (plan.n_ksplit > 0), [kLaunchSlots][kSplitHeads][n_ksplit]
    // x [ksplit_pmax][128 rows]: partial O (bf16 x 64) and lse2; counters per split tile
    void *d_ks_o = nullptr;
    float *d_ks_lse = nullptr;
    unsigned *d_ks_cnt = nullptr;
    // merged plan of the one-launch decomposition (strided-pass pairs, then band-pass pairs; entry,
    // entry-table and mask indices of the band part offset past the strided part's) and the per-slot
    // dependency counters [kLaunchSlots][kLseHeads + 1]; null when not built
    int32_t *d_mix_ent = nullptr, *d_mix_info = nullptr, *d_mix_kv_mask = nullptr;
    uint32_t *d_mix_masks = nullptr, *d_mix_qt_bits = nullptr;
    unsigned *d_dep = nullptr;
    int32_t mix_u1 = 0, mix_u2 = 0;
    // launch slots (top-level device handles only)
    splat::LaunchSlot slots[splat::kLaunchSlots];
    std::atomic<unsigned> next_slot{0};
    // splat_sparse_mhsa_host pipeline: copy-in, compute and copy-out streams + per-chunk events,
    // created at build time (top-level device handles only)
    std::mutex host_mu;
    void *hs[3] = {nullptr, nullptr, nullptr};
    void *hev[2][16] = {};
};

namespace splat {
cudaError_t dev_alloc_bytes(void **p, size_t bytes);
cudaError_t dev_alloc_async(void **p, size_t bytes, cudaStream_t st);
template <typename T>
inline cudaError_t dev_alloc(T **p, size_t bytes) { return dev_alloc_bytes(reinterpret_cast<void **>(p), bytes); }
splat_status set_error(splat_status st, const char *fmt, ...);
void clear_error();
void note_launches(int n);
splat_status validate_pattern(const splat_pattern &p);
void build_plan(splat_acsr_s &a);
}  // namespace splat
