// api.cu -- the C ABI of include/splat.h: argument validation, handle
// lifetime, ACSR build orchestration and kernel dispatch.  No arithmetic of
// the method lives here; every step runs in the kernels (acsr.cu, simt.cu,
// tc_fused.cu) or the planner (plan.cpp).
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <new>
#include <stdexcept>

#include "kernels.h"
#include "splat_internal.h"

namespace splat {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_allocs{0};

// Every device allocation of the library goes through here (build time only: compute calls never
// allocate; splat_device_alloc_count lets the tests check that).
cudaError_t dev_alloc_bytes(void **p, size_t bytes)
{
    g_allocs.fetch_add(1, std::memory_order_relaxed);
    return cudaMalloc(p, bytes);
}
cudaError_t dev_alloc_async(void **p, size_t bytes, cudaStream_t st)
{
    g_allocs.fetch_add(1, std::memory_order_relaxed);
    return cudaMallocAsync(p, bytes, st);
}
static thread_local int g_launches = 0;

splat_status set_error(splat_status st, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

void clear_error() { g_err[0] = 0; }
void note_launches(int n) { g_launches = n; }

static bool in_range(int v, int lo, int hi) { return v >= lo && v <= hi; }

splat_status validate_pattern(const splat_pattern &p)
{
    const int N = p.seq_len;
    if (!in_range(N, 1, 1 << 24))
        return set_error(SPLAT_ERR_INVALID_ARG, "seq_len %d outside [1, 2^24]", N);
    for (int r = 0; r < 7; ++r)
        if (p.reserved[r] != 0) return set_error(SPLAT_ERR_INVALID_ARG, "reserved[%d] must be 0", r);
    // which fields each kind reads; every other field must be 0
    bool use_lohi = false, use_block = false, use_g = false, use_stride = false, use_radius = false,
         use_causal = false;
    switch (p.kind) {
    case SPLAT_WINDOW: use_lohi = true; break;
    case SPLAT_BLOCKED: use_block = true; break;
    case SPLAT_STRIDED: use_stride = true; break;
    case SPLAT_DILATED: use_stride = use_radius = true; break;
    case SPLAT_GLOBAL_LOCAL: use_lohi = use_g = true; break;
    case SPLAT_BIGBIRD: use_block = use_radius = true; break;
    case SPLAT_STRIDED_LOCAL: use_stride = use_causal = true; break;
    default: return set_error(SPLAT_ERR_INVALID_ARG, "unknown pattern kind %d", p.kind);
    }
    if (!use_lohi && (p.lo || p.hi)) return set_error(SPLAT_ERR_INVALID_ARG, "lo/hi unused by kind %d", p.kind);
    if (!use_block && p.block) return set_error(SPLAT_ERR_INVALID_ARG, "block unused by kind %d", p.kind);
    if (!use_g && p.n_global) return set_error(SPLAT_ERR_INVALID_ARG, "n_global unused by kind %d", p.kind);
    if (!use_stride && p.stride) return set_error(SPLAT_ERR_INVALID_ARG, "stride unused by kind %d", p.kind);
    if (!use_radius && p.radius) return set_error(SPLAT_ERR_INVALID_ARG, "radius unused by kind %d", p.kind);
    if (!use_causal && p.causal) return set_error(SPLAT_ERR_INVALID_ARG, "causal unused by kind %d", p.kind);
    if (use_lohi && !(in_range(p.lo, 0, N) && in_range(p.hi, 0, N)))
        return set_error(SPLAT_ERR_INVALID_ARG, "window lo=%d hi=%d outside [0, N=%d]", p.lo, p.hi, N);
    if (use_block && !in_range(p.block, 1, N))
        return set_error(SPLAT_ERR_INVALID_ARG, "block %d outside [1, N=%d]", p.block, N);
    if (use_stride && !in_range(p.stride, 1, N))
        return set_error(SPLAT_ERR_INVALID_ARG, "stride %d outside [1, N=%d]", p.stride, N);
    if (use_radius && !in_range(p.radius, 0, N))
        return set_error(SPLAT_ERR_INVALID_ARG, "radius %d outside [0, N=%d]", p.radius, N);
    if (use_g && !in_range(p.n_global, 0, N))
        return set_error(SPLAT_ERR_INVALID_ARG, "n_global %d outside [0, N=%d]", p.n_global, N);
    if (p.kind == SPLAT_GLOBAL_LOCAL && p.n_global == 1)
        return set_error(SPLAT_ERR_UNSUPPORTED,
                         "GLOBAL_LOCAL with n_global=1: canonical greedy runs pair column 0 with the window");
    if (p.kind == SPLAT_BIGBIRD && p.block == 1)
        return set_error(SPLAT_ERR_UNSUPPORTED, "BIGBIRD with block=1: canonical greedy runs differ");
    if (p.kind == SPLAT_STRIDED_LOCAL && p.causal != 1)
        return set_error(SPLAT_ERR_UNSUPPORTED, "STRIDED_LOCAL requires causal=1");
    return SPLAT_OK;
}

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

splat_status cuda_fail(cudaError_t e, const char *what)
{
    return set_error(e == cudaErrorMemoryAllocation ? SPLAT_ERR_OOM : SPLAT_ERR_CUDA, "%s: %s", what,
                     cudaGetErrorString(e));
}

void free_device(splat_acsr_s *a)
{
    if (a->device < 0) return;
    DeviceGuard g(a->device);
    for (splat_acsr_s *sub : {a->sub_band, a->sub_str, a->sub_perm}) {
        if (sub) {
            free_device(sub);
            delete sub;
        }
    }
    a->sub_band = a->sub_str = a->sub_perm = nullptr;
    cudaFree(a->d_lse);
    a->d_lse = nullptr;
    cudaFree(a->d_ks_o);
    cudaFree(a->d_ks_lse);
    cudaFree(a->d_ks_cnt);
    a->d_ks_o = nullptr;
    a->d_ks_lse = nullptr;
    a->d_ks_cnt = nullptr;
    for (void *q : {(void *)a->d_mix_ent, (void *)a->d_mix_info, (void *)a->d_mix_kv_mask, (void *)a->d_mix_masks,
                    (void *)a->d_mix_qt_bits, (void *)a->d_dep})
        cudaFree(q);
    a->d_mix_ent = a->d_mix_info = a->d_mix_kv_mask = nullptr;
    a->d_mix_masks = a->d_mix_qt_bits = nullptr;
    a->d_dep = nullptr;
    for (int i = 0; i < kLaunchSlots; ++i)
        if (a->slots[i].ev) cudaEventDestroy((cudaEvent_t)a->slots[i].ev);
    for (int i = 0; i < 3; ++i)
        if (a->hs[i]) cudaStreamDestroy((cudaStream_t)a->hs[i]);
    for (int i = 0; i < 2; ++i)
        for (int c = 0; c < 16; ++c)
            if (a->hev[i][c]) cudaEventDestroy((cudaEvent_t)a->hev[i][c]);
    cudaFree(a->d_seg);
    cudaFree(a->d_nseg);
    cudaFree(a->d_row_ptr);
    cudaFree(a->plan.d_qt_ptr);
    cudaFree(a->plan.d_kv);
    cudaFree(a->plan.d_order);
    cudaFree(a->plan.d_pair_ent);
    cudaFree(a->plan.d_pair_info);
    cudaFree(a->plan.d_masks);
    cudaFree(a->plan.d_mask_rec);
    cudaFree(a->plan.d_mask_cnt);
    cudaFree(a->plan.d_kv_mask);
    cudaFree(a->plan.d_qt_bits);
    cudaFree(a->plan.d_t_info);
    cudaFree(a->plan.d_t_info_ks);
    cudaFree(a->plan.d_sched);
}

void finish_host_meta(splat_acsr_s *a)
{
    a->nnz = a->row_ptr_h[a->n];
    int mx = 0;
    for (int i = 0; i < a->n; ++i) mx = a->nseg_h[i] > mx ? a->nseg_h[i] : mx;
    a->max_segs = mx;
}

DevAcsr dev_view(const splat_acsr_s *a, int slot = 0)
{
    DevAcsr A;
    A.seg = reinterpret_cast<const int4 *>(a->d_seg);
    A.pat = a->pat;
    A.has_pat = a->pat.kind >= SPLAT_WINDOW && a->pat.kind <= SPLAT_STRIDED_LOCAL;
    A.nseg = a->d_nseg;
    A.row_ptr = a->d_row_ptr;
    A.n = a->n;
    A.nnz = a->nnz;
    A.qt_ptr = a->plan.d_qt_ptr;
    A.kv = a->plan.d_kv;
    A.order = a->plan.d_order;
    A.n_qt = a->plan.n_qt;
    A.pair_ent = a->plan.d_pair_ent;
    A.pair_info = reinterpret_cast<const int4 *>(a->plan.d_pair_info);
    A.masks = reinterpret_cast<const uint4 *>(a->plan.d_masks);
    A.mask_rec = reinterpret_cast<const uint4 *>(a->plan.d_mask_rec);
    A.mask_cnt = a->plan.d_mask_cnt;
    A.kv_mask = a->plan.d_kv_mask;
    A.qt_bits = a->plan.d_qt_bits;
    A.n_pairs = a->plan.n_pairs;
    A.n_buckets = a->plan.n_buckets;
    for (int b = 0; b <= a->plan.n_buckets && b <= kMaxBuckets; ++b) A.bucket_start[b] = a->plan.bucket_start[b];
    A.t_info = reinterpret_cast<const int4 *>(a->plan.d_t_info);
    A.sched = a->plan.d_sched ? a->plan.d_sched + 2 * slot : nullptr;
    A.t_n = (int)(a->plan.t_info.size() / 4);
    A.t_max_len = a->plan.t_max_len;
    A.t_entries = 0;
    for (size_t k = 0; k < a->plan.t_info.size(); k += 4) A.t_entries += a->plan.t_info[k + 2] - a->plan.t_info[k + 1];
    A.t_info_ks = reinterpret_cast<const int4 *>(a->plan.d_t_info_ks);
    A.t_n_ks = (int)(a->plan.t_info_ks.size() / 4);
    A.t_n_buckets_ks = a->plan.t_n_buckets_ks;
    for (int b = 0; b < (int)a->plan.t_bucket_start_ks.size() && b <= kMaxBuckets; ++b)
        A.t_bucket_start_ks[b] = a->plan.t_bucket_start_ks[b];
    A.n_ksplit = a->plan.n_ksplit;
    A.ks_pmax = a->plan.ksplit_pmax;
    {
        const size_t tiles = (size_t)kSplitHeads * a->plan.n_ksplit, parts = tiles * a->plan.ksplit_pmax;
        A.ks_o = a->d_ks_o ? static_cast<char *>(a->d_ks_o) + (size_t)slot * parts * 128 * 64 * 2 : nullptr;
        A.ks_lse = a->d_ks_lse ? a->d_ks_lse + (size_t)slot * parts * 128 : nullptr;
        A.ks_cnt = a->d_ks_cnt ? a->d_ks_cnt + (size_t)slot * tiles : nullptr;
    }
    A.t_n_buckets = a->plan.t_n_buckets;
    A.row_classes = a->plan.row_classes;
    for (int b = 0; b <= a->plan.t_n_buckets && b <= kMaxBuckets; ++b) A.t_bucket_start[b] = a->plan.t_bucket_start[b];
    return A;
}

splat_status check_compute(splat_acsr a, int B, int H)
{
    clear_error();
    if (!a) return set_error(SPLAT_ERR_INVALID_ARG, "null handle");
    if (a->device < 0)
        return set_error(SPLAT_ERR_INVALID_ARG, "host-only inspection handle: no device path (no CPU fallback)");
    if (B < 1 || H < 1) return set_error(SPLAT_ERR_SHAPE, "B=%d H=%d must be >= 1", B, H);
    if ((long long)B * H * a->n > (1LL << 31) - 1)
        return set_error(SPLAT_ERR_SHAPE, "B*H*N exceeds 2^31-1 rows");
    return SPLAT_OK;
}

splat_status check_d(splat_dtype dt, int d)
{
    if (dt == SPLAT_BF16) {
        if (d != 64 && d != 128) return set_error(SPLAT_ERR_UNSUPPORTED, "bf16 path needs d in {64,128}, got %d", d);
    } else if (dt == SPLAT_FP32) {
        if (d < 1 || d > 256) return set_error(SPLAT_ERR_UNSUPPORTED, "fp32 path needs 1 <= d <= 256, got %d", d);
    } else {
        return set_error(SPLAT_ERR_INVALID_ARG, "unknown dtype %d", (int)dt);
    }
    return SPLAT_OK;
}

bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

// residue decomposition available and not disabled (diagnostics build only: SPLAT_NO_RESIDUE_SPLIT=1
// runs the single-pass natural-order plan)
bool use_residue_split(const splat_acsr_s *a)
{
    static const bool off = diag_env("SPLAT_NO_RESIDUE_SPLIT") != 0;
    return a->sub_band != nullptr && !off;
}

// One launch for the residue decomposition: an experiment, selected only in the diagnostics build
// (SPLAT_RESIDUE_1PASS=1).  It cuts the DRAM traffic of the Sparse-Transformer step from 1.16 GB to
// 0.70 GB but runs ~40 % slower than the two launches: the product keeps two.
bool use_residue1(const splat_acsr_s *a)
{
    static const bool on = diag_env("SPLAT_RESIDUE_1PASS") != 0;
    return a->d_dep != nullptr && on;
}

// Device view of the merged plan of the one-launch residue decomposition
DevAcsr mix_view(const splat_acsr_s *a)
{
    DevAcsr A = dev_view(a->sub_str);
    A.pair_ent = a->d_mix_ent;
    A.pair_info = reinterpret_cast<const int4 *>(a->d_mix_info);
    A.kv_mask = a->d_mix_kv_mask;
    A.masks = reinterpret_cast<const uint4 *>(a->d_mix_masks);
    A.qt_bits = a->d_mix_qt_bits;
    A.n_pairs = a->mix_u1 + a->mix_u2;
    A.n_buckets = 0;
    return A;
}

bool use_perm()
{
    static const bool off = diag_env("SPLAT_NO_RESIDUE_SPLIT") != 0;
    return !off;
}

}  // namespace
}  // namespace splat

using namespace splat;

namespace {

// Device metadata is in a->d_seg / d_nseg / d_row_ptr (queued on cs): copy it to the host,
// build the tile plan and upload it.  Frees `a` on failure.
// The tile plan, with host allocation failures and oversize plans reported instead of thrown
// through the C ABI.
splat_status plan_or_error(splat_acsr_s &a)
{
    try {
        build_plan(a);
    } catch (const std::bad_alloc &) {
        return set_error(SPLAT_ERR_OOM, "host allocation of the tile plan failed");
    } catch (const std::length_error &e) {
        return set_error(SPLAT_ERR_UNSUPPORTED, "tile plan: %s", e.what());
    }
    return SPLAT_OK;
}

splat_status finish_device_build(splat_acsr_s *a, cudaStream_t cs, splat_acsr *out)
{
    const int N = a->n;
    cudaError_t e = cudaMemcpyAsync(a->seg_h.data(), a->d_seg, sizeof(int32_t) * 16 * (size_t)N,
                                    cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(a->nseg_h.data(), a->d_nseg, (size_t)N, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(a->row_ptr_h.data(), a->d_row_ptr, sizeof(int64_t) * ((size_t)N + 1),
                            cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) {
        free_device(a);
        delete a;
        return cuda_fail(e, "acsr build");
    }
    finish_host_meta(a);
    if (const splat_status ps = plan_or_error(*a); ps != SPLAT_OK) {
        free_device(a);
        delete a;
        return ps;
    }
    Plan &P = a->plan;
    if ((e = dev_alloc(&P.d_qt_ptr, sizeof(int32_t) * (P.n_qt + 1))) != cudaSuccess ||
        (e = dev_alloc(&P.d_kv, sizeof(int32_t) * (P.kv.empty() ? 1 : P.kv.size()))) != cudaSuccess ||
        (e = dev_alloc(&P.d_order, sizeof(int32_t) * P.n_qt)) != cudaSuccess ||
        (e = dev_alloc(&P.d_pair_ent, sizeof(int32_t) * (P.n_pair_entries > 0 ? P.n_pair_entries : 1))) != cudaSuccess ||
        (e = dev_alloc(&P.d_pair_info, sizeof(int32_t) * 8 * P.n_pairs)) != cudaSuccess ||
        (e = dev_alloc(&P.d_masks, sizeof(uint32_t) * (P.masks.empty() ? 4 : P.masks.size()))) != cudaSuccess ||
        (e = dev_alloc(&P.d_mask_rec, sizeof(uint16_t) * (P.mask_rec.empty() ? 16 : P.mask_rec.size()))) != cudaSuccess ||
        (e = dev_alloc(&P.d_mask_cnt, P.mask_cnt.empty() ? 16 : P.mask_cnt.size())) != cudaSuccess ||
        (e = dev_alloc(&P.d_kv_mask, sizeof(int32_t) * (P.kv_mask.empty() ? 1 : P.kv_mask.size()))) != cudaSuccess ||
        (e = dev_alloc(&P.d_qt_bits, sizeof(uint32_t) * (P.qt_bits.empty() ? 1 : P.qt_bits.size()))) != cudaSuccess ||
        (e = dev_alloc(&P.d_t_info, sizeof(int32_t) * (P.t_info.empty() ? 4 : P.t_info.size()))) != cudaSuccess ||
        (e = dev_alloc(&P.d_t_info_ks, sizeof(int32_t) * (P.t_info_ks.empty() ? 4 : P.t_info_ks.size()))) != cudaSuccess ||
        (e = dev_alloc(&P.d_sched, kLaunchSlots * 2 * sizeof(unsigned long long))) != cudaSuccess) {
        free_device(a);
        delete a;
        return cuda_fail(e, "plan allocation");
    }
    e = cudaMemcpyAsync(P.d_qt_ptr, P.qt_ptr.data(), sizeof(int32_t) * (P.n_qt + 1), cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess && !P.kv.empty())
        e = cudaMemcpyAsync(P.d_kv, P.kv.data(), sizeof(int32_t) * P.kv.size(), cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(P.d_order, P.order.data(), sizeof(int32_t) * P.n_qt, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess && P.n_pair_entries > 0)
        e = cudaMemcpyAsync(P.d_pair_ent, P.pair_ent.data(), sizeof(int32_t) * P.n_pair_entries, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(P.d_pair_info, P.pair_info.data(), sizeof(int32_t) * 8 * P.n_pairs, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess && !P.masks.empty())
        e = cudaMemcpyAsync(P.d_masks, P.masks.data(), sizeof(uint32_t) * P.masks.size(), cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess && !P.mask_rec.empty())
        e = cudaMemcpyAsync(P.d_mask_rec, P.mask_rec.data(), sizeof(uint16_t) * P.mask_rec.size(), cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess && !P.mask_cnt.empty())
        e = cudaMemcpyAsync(P.d_mask_cnt, P.mask_cnt.data(), P.mask_cnt.size(), cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess && !P.kv_mask.empty())
        e = cudaMemcpyAsync(P.d_kv_mask, P.kv_mask.data(), sizeof(int32_t) * P.kv_mask.size(), cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess && !P.qt_bits.empty())
        e = cudaMemcpyAsync(P.d_qt_bits, P.qt_bits.data(), sizeof(uint32_t) * P.qt_bits.size(), cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(P.d_t_info, P.t_info.data(), sizeof(int32_t) * P.t_info.size(), cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess && !P.t_info_ks.empty())
        e = cudaMemcpyAsync(P.d_t_info_ks, P.t_info_ks.data(), sizeof(int32_t) * P.t_info_ks.size(), cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaMemsetAsync(P.d_sched, 0, kLaunchSlots * 2 * sizeof(unsigned long long), cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) {
        free_device(a);
        delete a;
        return cuda_fail(e, "plan upload");
    }
    *out = a;
    return SPLAT_OK;
}

// Host INSPECTION variant of the mask ingest (mask_ingest.cu): the same greedy runs, column by
// column.  Returns false with the first offending column if row i needs more than max_runs runs.
bool host_mask_row(const uint32_t *row, int N, int max_runs, int32_t *seg, uint8_t *nseg, int64_t *cnt,
                   int32_t *bad_col)
{
    auto bit = [&](int x) { return (row[x >> 5] >> (x & 31)) & 1u; };
    int nr = 0, off = 0, x = 0;
    while (true) {
        while (x < N && !bit(x)) ++x;
        if (x >= N) break;
        if (nr == max_runs) {
            *bad_col = x;
            return false;
        }
        int c0 = x, step = 1, n = 1;
        int c1 = c0 + 1;
        while (c1 < N && !bit(c1)) ++c1;
        if (c1 < N) {
            step = c1 - c0;
            n = 2;
            int last = c1;
            while (true) {
                int nx = last + 1;
                while (nx < N && !bit(nx)) ++nx;
                if (nx >= N || nx - last != step) break;
                last = nx;
                ++n;
            }
            x = last + 1;
        } else {
            x = N;
        }
        int32_t *g = seg + 4 * nr;
        g[0] = c0; g[1] = step; g[2] = n; g[3] = off;
        off += n;
        ++nr;
    }
    for (int k = nr; k < 4; ++k) seg[4 * k + 3] = off;
    *nseg = (uint8_t)nr;
    *cnt = off;
    return true;
}

// The whole handle build (metadata + plan, device copies); `internal` patterns (the residue
// decomposition's sub-patterns) skip the public descriptor validation.
splat_status build_impl(const splat_pattern *p, int device, void *stream, splat_acsr *out, bool internal)
{
    clear_error();
    if (!p || !out) return set_error(SPLAT_ERR_INVALID_ARG, "null pattern or out pointer");
    *out = nullptr;
    splat_status st = internal ? SPLAT_OK : validate_pattern(*p);
    if (st != SPLAT_OK) return st;
    splat_acsr_s *a = new (std::nothrow) splat_acsr_s();
    if (!a) return set_error(SPLAT_ERR_OOM, "host allocation failed");
    a->pat = *p;
    a->n = p->seq_len;
    // sub-handles of the residue decomposition / permuted strided path run residue-major views whose
    // tile arithmetic needs 128-aligned key windows
    a->plan.kv_align = internal ? 2 : 1;
    const int N = a->n;
    a->seg_h.assign((size_t)N * 16, 0);
    a->nseg_h.assign(N, 0);
    a->row_ptr_h.assign((size_t)N + 1, 0);
    if (device < 0) {
        // host INSPECTION handle: same closed form, evaluated on the host
        for (int i = 0; i < N; ++i) {
            Seg s[4];
            const int n = row_segments(*p, i, s);
            int off = 0;
            for (int k = 0; k < n; ++k) {
                int32_t *g = &a->seg_h[(size_t)i * 16 + 4 * k];
                g[0] = s[k].start; g[1] = s[k].step; g[2] = s[k].count; g[3] = off;
                off += s[k].count;
            }
            for (int k = n; k < 4; ++k) a->seg_h[(size_t)i * 16 + 4 * k + 3] = off;
            a->nseg_h[i] = (uint8_t)n;
            a->row_ptr_h[i + 1] = a->row_ptr_h[i] + off;
        }
        finish_host_meta(a);
        if (const splat_status ps = plan_or_error(*a); ps != SPLAT_OK) {
            delete a;
            return ps;
        }
        *out = a;
        return SPLAT_OK;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev) {
        delete a;
        cudaGetLastError();
        return set_error(SPLAT_ERR_INVALID_ARG, "device %d not available (%d devices)", device, ndev);
    }
    a->device = device;
    DeviceGuard g(device);
    cudaStream_t cs = (cudaStream_t)stream;
    cudaError_t e;
    if ((e = dev_alloc(&a->d_seg, sizeof(int32_t) * 16 * (size_t)N)) != cudaSuccess ||
        (e = dev_alloc(&a->d_nseg, (size_t)N)) != cudaSuccess ||
        (e = dev_alloc(&a->d_row_ptr, sizeof(int64_t) * ((size_t)N + 1))) != cudaSuccess) {
        free_device(a);
        delete a;
        return cuda_fail(e, "acsr allocation");
    }
    e = launch_acsr_build(*p, reinterpret_cast<int4 *>(a->d_seg), a->d_nseg, a->d_row_ptr, cs);
    if (e != cudaSuccess) {
        free_device(a);
        delete a;
        return cuda_fail(e, "acsr build");
    }
    return finish_device_build(a, cs, out);
}

#ifdef SPLAT_DIAG
// Merged plan of the one-launch residue decomposition: the strided pass's pairs, then the band
// pass's, with the band part's entry (pair_ent), entry-table (kv_mask / qt_bits) and mask indices
// offset past the strided part's; plus zeroed dependency counters per launch slot.  Optional: on
// any failure the two-launch form is used.
void build_residue_merged(splat_acsr_s *a, cudaStream_t cs)
{
    const Plan &P1 = a->sub_str->plan, &P2 = a->sub_band->plan;
    if (P1.n_qt != P2.n_qt || P1.n_pairs <= 0 || P2.n_pairs <= 0) return;
    std::vector<int32_t> ent, info, kvm;
    std::vector<uint32_t> masks, bits;
    try {
        ent.assign(P1.pair_ent.begin(), P1.pair_ent.begin() + P1.n_pair_entries);
        ent.insert(ent.end(), P2.pair_ent.begin(), P2.pair_ent.begin() + P2.n_pair_entries);
        info.assign(P1.pair_info.begin(), P1.pair_info.begin() + 8 * (size_t)P1.n_pairs);
        const int n_ent1 = (int)P1.kv_mask.size();
        for (int k = 0; k < P2.n_pairs; ++k) {
            const int32_t *x = &P2.pair_info[8 * (size_t)k];
            // pair, e0, e1, jA0, jA1, jB1, 0, 0
            info.insert(info.end(), {x[0], x[1] + P1.n_pair_entries, x[2] + P1.n_pair_entries, x[3] + n_ent1,
                                     x[4] + n_ent1, x[5] + n_ent1, x[6], x[7]});
        }
        kvm = P1.kv_mask;
        for (int32_t m : P2.kv_mask) kvm.push_back(m >= 0 ? m + P1.n_masks : m);
        bits = P1.qt_bits;
        bits.insert(bits.end(), P2.qt_bits.begin(), P2.qt_bits.end());
        masks.assign(P1.masks.begin(), P1.masks.begin() + (size_t)P1.n_masks * 128 * 4);
        masks.insert(masks.end(), P2.masks.begin(), P2.masks.begin() + (size_t)P2.n_masks * 128 * 4);
    } catch (const std::bad_alloc &) {
        return;
    }
    if (masks.empty()) masks.assign(4, 0u);
    const size_t n_dep = (size_t)kLaunchSlots * (kLseHeads + 1);
    cudaError_t e = cudaSuccess;
    if ((e = dev_alloc(&a->d_mix_ent, sizeof(int32_t) * ent.size())) != cudaSuccess ||
        (e = dev_alloc(&a->d_mix_info, sizeof(int32_t) * info.size())) != cudaSuccess ||
        (e = dev_alloc(&a->d_mix_kv_mask, sizeof(int32_t) * kvm.size())) != cudaSuccess ||
        (e = dev_alloc(&a->d_mix_qt_bits, sizeof(uint32_t) * bits.size())) != cudaSuccess ||
        (e = dev_alloc(&a->d_mix_masks, sizeof(uint32_t) * masks.size())) != cudaSuccess ||
        (e = dev_alloc(&a->d_dep, sizeof(unsigned) * n_dep)) != cudaSuccess) {
    } else if ((e = cudaMemcpyAsync(a->d_mix_ent, ent.data(), sizeof(int32_t) * ent.size(), cudaMemcpyHostToDevice, cs)) != cudaSuccess ||
               (e = cudaMemcpyAsync(a->d_mix_info, info.data(), sizeof(int32_t) * info.size(), cudaMemcpyHostToDevice, cs)) != cudaSuccess ||
               (e = cudaMemcpyAsync(a->d_mix_kv_mask, kvm.data(), sizeof(int32_t) * kvm.size(), cudaMemcpyHostToDevice, cs)) != cudaSuccess ||
               (e = cudaMemcpyAsync(a->d_mix_qt_bits, bits.data(), sizeof(uint32_t) * bits.size(), cudaMemcpyHostToDevice, cs)) != cudaSuccess ||
               (e = cudaMemcpyAsync(a->d_mix_masks, masks.data(), sizeof(uint32_t) * masks.size(), cudaMemcpyHostToDevice, cs)) != cudaSuccess ||
               (e = cudaMemsetAsync(a->d_dep, 0, sizeof(unsigned) * n_dep, cs)) != cudaSuccess) {
    } else {
        e = cudaStreamSynchronize(cs);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        for (void *q : {(void *)a->d_mix_ent, (void *)a->d_mix_info, (void *)a->d_mix_kv_mask, (void *)a->d_mix_masks,
                        (void *)a->d_mix_qt_bits, (void *)a->d_dep})
            cudaFree(q);
        a->d_mix_ent = a->d_mix_info = a->d_mix_kv_mask = nullptr;
        a->d_mix_masks = a->d_mix_qt_bits = nullptr;
        a->d_dep = nullptr;
        return;
    }
    a->mix_u1 = P1.n_pairs;
    a->mix_u2 = P2.n_pairs;
}
#endif  // SPLAT_DIAG

// Residue decomposition of STRIDED_LOCAL(l) (see splat_acsr_s::sub_band): applicable when the
// residue classes tile the sequence exactly (N % l == 0) and whole classes fill a 128-row tile
// (nk = N / l divides 128, nk >= 2).
void build_residue_split(splat_acsr_s *a, void *stream)
{
    const splat_pattern &p = a->pat;
    if (p.kind == SPLAT_STRIDED && a->device >= 0) {
        const int N = a->n, X = p.stride;
        if (X < 2 || N % X != 0) return;
        const int nk = N / X;
        if (nk < 2 || (nk & (nk - 1)) != 0) return;   // power of two: nk | 128 or 128 | nk
        splat_pattern blk{};
        blk.kind = SPLAT_BLOCKED;
        blk.seq_len = N;
        blk.block = nk;
        splat_acsr hp = nullptr;
        if (build_impl(&blk, a->device, stream, &hp, true) != SPLAT_OK) { clear_error(); return; }
        a->sub_perm = hp;
        a->rv_l = X;
        a->rv_nk = nk;
        a->rv_R = nk <= 128 ? 128 / nk : 1;
        return;
    }
    if (p.kind != SPLAT_STRIDED_LOCAL || a->device < 0) return;
    const int N = a->n, l = p.stride;
    if (l < 2 || N % l != 0) return;
    const int nk = N / l;
    if (nk < 2 || nk > 128 || 128 % nk != 0) return;
    splat_pattern band{}, str{};
    band.kind = SPLAT_WINDOW;
    band.seq_len = N;
    band.lo = l - 1;
    band.hi = 0;
    str.kind = kKindResiduePrev;
    str.seq_len = N;
    str.block = nk;
    splat_acsr hb = nullptr, hs = nullptr;
    if (build_impl(&band, a->device, stream, &hb, true) != SPLAT_OK) { clear_error(); return; }
    if (build_impl(&str, a->device, stream, &hs, true) != SPLAT_OK) {
        clear_error();
        free_device(hb);
        delete hb;
        return;
    }
    float *lse = nullptr;
    if (dev_alloc(&lse, sizeof(float) * (size_t)kLaunchSlots * kLseHeads * N) != cudaSuccess) {
        cudaGetLastError();
        free_device(hb);
        delete hb;
        free_device(hs);
        delete hs;
        return;
    }
    a->d_lse = lse;
    a->sub_band = hb;
    a->sub_str = hs;
    a->rv_l = l;
    a->rv_nk = nk;
    a->rv_R = 128 / nk;
#ifdef SPLAT_DIAG
    build_residue_merged(a, (cudaStream_t)stream);    // the one-launch experiment (DESIGN 9g)
#endif
}

// Launch slots and the host pipeline's streams / events of a top-level device handle (build time,
// so that compute calls never allocate).
splat_status create_call_resources(splat_acsr_s *a)
{
    if (a->device < 0) return SPLAT_OK;
    DeviceGuard g(a->device);
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < kLaunchSlots && e == cudaSuccess; ++i)
        e = cudaEventCreateWithFlags(reinterpret_cast<cudaEvent_t *>(&a->slots[i].ev), cudaEventDisableTiming);
    for (int i = 0; i < 3 && e == cudaSuccess; ++i)
        e = cudaStreamCreateWithFlags(reinterpret_cast<cudaStream_t *>(&a->hs[i]), cudaStreamNonBlocking);
    if (e == cudaSuccess && a->plan.n_ksplit > 0 &&
        (size_t)kLaunchSlots * kSplitHeads * a->plan.n_ksplit * a->plan.ksplit_pmax * 128 * (64 * 2 + 4) > kSplitScratchMax) {
        // too many long tiles for a bounded scratch: the launches keep the whole-tile list
        a->plan.n_ksplit = 0;
        a->plan.t_info_ks.clear();
    }
    if (e == cudaSuccess && a->plan.n_ksplit > 0) {
        // split-K partial results of the d = 64 fused kernel, per launch slot (bf16 O + lse2 per part
        // and row, one counter per split tile), zeroed once: the merging part resets its counter
        const size_t tiles = (size_t)kLaunchSlots * kSplitHeads * a->plan.n_ksplit;
        const size_t parts = tiles * a->plan.ksplit_pmax;
        if ((e = dev_alloc_bytes(&a->d_ks_o, parts * 128 * 64 * 2)) == cudaSuccess &&
            (e = dev_alloc(&a->d_ks_lse, parts * 128 * sizeof(float))) == cudaSuccess &&
            (e = dev_alloc(&a->d_ks_cnt, tiles * sizeof(unsigned))) == cudaSuccess)
            e = cudaMemset(a->d_ks_cnt, 0, tiles * sizeof(unsigned));
    }
    for (int i = 0; i < 2 && e == cudaSuccess; ++i)
        for (int c = 0; c < 16 && e == cudaSuccess; ++c)
            e = cudaEventCreateWithFlags(reinterpret_cast<cudaEvent_t *>(&a->hev[i][c]), cudaEventDisableTiming);
    return e == cudaSuccess ? SPLAT_OK : cuda_fail(e, "call resources");
}

// RAII use of a launch slot on `s`: waits for the slot's previous user, records the slot's event
// after the work queued while held.  Under stream capture the event ordering is skipped (a captured
// graph must not be replayed concurrently with another use of the same handle).
struct SlotUse {
    LaunchSlot *slot = nullptr;
    int index = 0;
    cudaStream_t s;
    bool capturing = false;
    SlotUse(splat_acsr_s *a, cudaStream_t st) : s(st)
    {
        index = (int)(a->next_slot.fetch_add(1u, std::memory_order_relaxed) % kLaunchSlots);
        slot = &a->slots[index];
        slot->mu.lock();
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cap);
        capturing = cap != cudaStreamCaptureStatusNone;
        if (slot->used && !capturing) cudaStreamWaitEvent(s, (cudaEvent_t)slot->ev, 0);
    }
    ~SlotUse()
    {
        if (!capturing && cudaEventRecord((cudaEvent_t)slot->ev, s) == cudaSuccess) slot->used = true;
        slot->mu.unlock();
    }
};

}  // namespace

namespace {

#ifndef SPLAT_HOST_CHUNKS
#define SPLAT_HOST_CHUNKS 12
#endif
constexpr int kHostChunks = SPLAT_HOST_CHUNKS;     // (b, h) chunks of the host pipeline (<= 15 events)

// argument checks of splat_sparse_mhsa (also applied once to a whole host-path call)
splat_status check_mhsa(splat_acsr a, const void *Q, const void *K, const void *V, splat_dtype dt, int B, int H,
                        int d, float scale, const void *O)
{
    splat_status st = check_compute(a, B, H);
    if (st == SPLAT_OK) st = check_d(dt, d);
    if (st != SPLAT_OK) return st;
    if (!Q || !K || !V || !O) return set_error(SPLAT_ERR_INVALID_ARG, "null tensor pointer");
    if (!aligned16(Q) || !aligned16(K) || !aligned16(V) || !aligned16(O))
        return set_error(SPLAT_ERR_INVALID_ARG, "tensors must be 16-byte aligned");
    if (!(scale > 0.f) || scale == INFINITY) return set_error(SPLAT_ERR_INVALID_ARG, "scale must be positive and finite");
    return SPLAT_OK;
}

// dispatch of a validated fused call (sets the launch count); no allocation, no host sync
// allow_ksplit: the d = 64 kernel may take the split-K unit list for few heads (off for the host
// pipeline's chunks, whose kernels hide behind the PCIe copies: measured 3.56 vs 3.27 ms per step)
cudaError_t launch_mhsa(splat_acsr a, const void *Q, const void *K, const void *V, splat_dtype dt, int BH, int d,
                        float scale, void *O, cudaStream_t s, bool allow_ksplit = true)
{
    int nl = 1;
    cudaError_t e;
    if (dt == SPLAT_BF16 && d == 128 && use_residue_split(a)) {
        // heads in chunks of kLseHeads: the slot's lse scratch holds one chunk
        SlotUse su(a, s);
        float *lse = a->d_lse + (size_t)su.index * kLseHeads * a->n;
        const size_t slice = (size_t)a->n * d * 2;
        e = cudaSuccess;
        nl = 0;
        for (int h0 = 0; h0 < BH && e == cudaSuccess; h0 += kLseHeads) {
            const int nh = BH - h0 < kLseHeads ? BH - h0 : kLseHeads;
            const size_t off = slice * h0;
            int n1 = 0;
            if (use_residue1(a))
                e = launch_mhsa_tc_residue1(mix_view(a), a->mix_u1, a->mix_u2, a->rv_l, a->rv_nk, a->rv_R, lse,
                                            a->d_dep + (size_t)su.index * (kLseHeads + 1), (const char *)Q + off,
                                            (const char *)K + off, (const char *)V + off, nh, d, scale,
                                            (char *)O + off, s, &n1);
            else
                e = launch_mhsa_tc_residue(dev_view(a->sub_band), dev_view(a->sub_str), a->rv_l, a->rv_nk, a->rv_R,
                                           lse, (const char *)Q + off, (const char *)K + off, (const char *)V + off,
                                           nh, d, scale, (char *)O + off, s, &n1);
            nl += n1;
        }
    } else if (dt == SPLAT_BF16 && a->sub_perm && use_perm())
        e = launch_mhsa_tc_permuted(dev_view(a->sub_perm), a->rv_l, a->rv_nk, a->rv_R, Q, K, V, BH, d, scale, O, s,
                                    &nl);
    else if (dt == SPLAT_BF16 && d == 64) {
        SlotUse su(a, s);                // the split kernel's work counter (and split-K scratch)
        DevAcsr A = dev_view(a, su.index);
        if (!allow_ksplit) A.n_ksplit = 0;
        e = launch_mhsa_tc(A, Q, K, V, BH, d, scale, O, s, &nl);
    } else if (dt == SPLAT_BF16)
        e = launch_mhsa_tc(dev_view(a), Q, K, V, BH, d, scale, O, s, &nl);
    else
        e = launch_mhsa_simt(dev_view(a), Q, K, V, false, BH, d, scale, O, s);
    note_launches(nl);
    return e;
}

}  // namespace

extern "C" {

splat_status splat_acsr_build(const splat_pattern *p, int device, void *stream, splat_acsr *out)
{
    splat_status st;
    try {
        st = build_impl(p, device, stream, out, false);
    } catch (const std::bad_alloc &) {
        // host metadata of a huge N (the per-row vectors are allocated before the plan)
        if (out) *out = nullptr;
        return set_error(SPLAT_ERR_OOM, "host allocation of the ACSR metadata failed");
    }
    if (st == SPLAT_OK) build_residue_split(*out, stream);
    if (st == SPLAT_OK && (st = create_call_resources(*out)) != SPLAT_OK) {
        free_device(*out);
        delete *out;
        *out = nullptr;
    }
    return st;
}

splat_status splat_acsr_from_mask(const uint32_t *mask, int32_t n, int32_t max_runs, int device, void *stream,
                                  splat_acsr *out, int32_t *bad_row, int32_t *bad_col)
{
    clear_error();
    if (bad_row) *bad_row = -1;
    if (bad_col) *bad_col = -1;
    if (!mask || !out) return set_error(SPLAT_ERR_INVALID_ARG, "null mask or out pointer");
    *out = nullptr;
    if (n < 1 || n > kMaxMaskN) return set_error(SPLAT_ERR_INVALID_ARG, "n = %d outside [1, %d]", n, kMaxMaskN);
    if (max_runs < 1 || max_runs > SPLAT_MAX_SEGS)
        return set_error(SPLAT_ERR_INVALID_ARG, "max_runs = %d outside [1, %d]", max_runs, SPLAT_MAX_SEGS);
    splat_acsr_s *a = new (std::nothrow) splat_acsr_s();
    if (!a) return set_error(SPLAT_ERR_OOM, "host allocation failed");
    a->pat = splat_pattern{};
    a->pat.kind = kKindMask;
    a->pat.seq_len = n;
    a->n = n;
    a->seg_h.assign((size_t)n * 16, 0);
    a->nseg_h.assign(n, 0);
    a->row_ptr_h.assign((size_t)n + 1, 0);
    auto not_regular = [&](long long r, long long c) {
        if (bad_row) *bad_row = (int32_t)r;
        if (bad_col) *bad_col = (int32_t)c;
        return set_error(SPLAT_ERR_NOT_REGULAR, "row %lld needs more than %d affine runs (column %lld)", r,
                         max_runs, c);
    };
    const int W = (n + 31) / 32;
    if (device < 0) {
        for (int i = 0; i < n; ++i) {
            int64_t cnt = 0;
            int32_t bc = -1;
            if (!host_mask_row(mask + (size_t)i * W, n, max_runs, &a->seg_h[(size_t)i * 16], &a->nseg_h[i], &cnt,
                               &bc)) {
                delete a;
                return not_regular(i, bc);
            }
            a->row_ptr_h[i + 1] = a->row_ptr_h[i] + cnt;
        }
        finish_host_meta(a);
        if (const splat_status ps = plan_or_error(*a); ps != SPLAT_OK) {
            delete a;
            return ps;
        }
        *out = a;
        return SPLAT_OK;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev) {
        delete a;
        cudaGetLastError();
        return set_error(SPLAT_ERR_INVALID_ARG, "device %d not available (%d devices)", device, ndev);
    }
    a->device = device;
    DeviceGuard g(device);
    cudaStream_t cs = (cudaStream_t)stream;
    cudaError_t e;
    unsigned long long *d_bad = nullptr, bad = 0;
    if ((e = dev_alloc(&a->d_seg, sizeof(int32_t) * 16 * (size_t)n)) != cudaSuccess ||
        (e = dev_alloc(&a->d_nseg, (size_t)n)) != cudaSuccess ||
        (e = dev_alloc(&a->d_row_ptr, sizeof(int64_t) * ((size_t)n + 1))) != cudaSuccess ||
        (e = dev_alloc(&d_bad, sizeof(unsigned long long))) != cudaSuccess) {
        cudaFree(d_bad);
        free_device(a);
        delete a;
        return cuda_fail(e, "acsr allocation");
    }
    e = launch_acsr_from_mask(mask, n, max_runs, reinterpret_cast<int4 *>(a->d_seg), a->d_nseg, a->d_row_ptr,
                              d_bad, cs);
    note_launches(n > 32 * 8192 ? 4 : 2);     // row kernel + row_ptr scan (multi-CTA above 32 tiles)
    if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    cudaFree(d_bad);
    if (e != cudaSuccess) {
        free_device(a);
        delete a;
        return cuda_fail(e, "mask ingest");
    }
    if (bad != ~0ull) {
        free_device(a);
        delete a;
        return not_regular((long long)(bad >> 32), (long long)(bad & 0xffffffffull));
    }
    splat_status st = finish_device_build(a, cs, out);
    if (st == SPLAT_OK && (st = create_call_resources(*out)) != SPLAT_OK) {
        free_device(*out);
        delete *out;
        *out = nullptr;
    }
    return st;
}

splat_status splat_acsr_info(splat_acsr a, int32_t *n, int64_t *nnz, int32_t *max_segs, double *density)
{
    clear_error();
    if (!a) return set_error(SPLAT_ERR_INVALID_ARG, "null handle");
    if (n) *n = a->n;
    if (nnz) *nnz = a->nnz;
    if (max_segs) *max_segs = a->max_segs;
    if (density) *density = (double)a->nnz / ((double)a->n * (double)a->n);
    return SPLAT_OK;
}

splat_status splat_acsr_copy_meta(splat_acsr a, int32_t *seg, uint8_t *nseg, int64_t *row_ptr)
{
    clear_error();
    if (!a) return set_error(SPLAT_ERR_INVALID_ARG, "null handle");
    if (seg)
        for (size_t i = 0; i < (size_t)a->n; ++i)
            for (int k = 0; k < 4; ++k)
                for (int c = 0; c < 3; ++c) seg[i * 12 + k * 3 + c] = a->seg_h[i * 16 + k * 4 + c];
    if (nseg) memcpy(nseg, a->nseg_h.data(), (size_t)a->n);
    if (row_ptr) memcpy(row_ptr, a->row_ptr_h.data(), sizeof(int64_t) * ((size_t)a->n + 1));
    return SPLAT_OK;
}

splat_status splat_plan_info(splat_acsr a, int32_t *bm, int32_t *bn, int32_t *n_qtiles, int32_t *n_entries)
{
    clear_error();
    if (!a) return set_error(SPLAT_ERR_INVALID_ARG, "null handle");
    if (bm) *bm = a->plan.bm;
    if (bn) *bn = a->plan.bn;
    if (n_qtiles) *n_qtiles = a->plan.n_qt;
    if (n_entries) *n_entries = a->plan.n_entries;
    return SPLAT_OK;
}

splat_status splat_plan_split_info(splat_acsr a, int32_t *row_classes, int32_t *n_split_entries)
{
    clear_error();
    if (!a) return set_error(SPLAT_ERR_INVALID_ARG, "null handle");
    const Plan &P = a->plan;
    if (row_classes) *row_classes = P.row_classes;
    if (n_split_entries) *n_split_entries = P.row_classes ? (int32_t)(P.kv.size() - (size_t)P.n_entries) : P.n_entries;
    return SPLAT_OK;
}

int64_t splat_plan_sizes(splat_acsr a, int32_t which)
{
    if (!a) return -1;
    const Plan &P = a->plan;
    switch (which) {
    case 0: return (int64_t)P.t_info.size() / 4;   // split-kernel units per (b, h)
    case 1: return (int64_t)P.kv.size();           // all entries (natural, then classed)
    case 2: return (int64_t)P.n_masks;
    case 3: return (int64_t)P.t_info_ks.size() / 4;   // split-K units per (b, h)
    default: return -1;
    }
}

splat_status splat_plan_split_copy(splat_acsr a, int32_t *units, int32_t *kv, int32_t *mask_id, uint32_t *masks)
{
    clear_error();
    if (!a) return set_error(SPLAT_ERR_INVALID_ARG, "null handle");
    const Plan &P = a->plan;
    if (units) memcpy(units, P.t_info.data(), sizeof(int32_t) * P.t_info.size());
    if (kv) memcpy(kv, P.kv.data(), sizeof(int32_t) * P.kv.size());
    if (mask_id) memcpy(mask_id, P.kv_mask.data(), sizeof(int32_t) * P.kv_mask.size());
    if (masks) memcpy(masks, P.masks.data(), sizeof(uint32_t) * P.masks.size());
    return SPLAT_OK;
}

splat_status splat_plan_ksplit_copy(splat_acsr a, int32_t *units)
{
    clear_error();
    if (!a || !units) return set_error(SPLAT_ERR_INVALID_ARG, "null handle or output");
    const Plan &P = a->plan;
    if (!P.t_info_ks.empty()) memcpy(units, P.t_info_ks.data(), sizeof(int32_t) * P.t_info_ks.size());
    return SPLAT_OK;
}

splat_status splat_plan_copy(splat_acsr a, int32_t *qt_ptr, int32_t *kv, int32_t *order)
{
    clear_error();
    if (!a) return set_error(SPLAT_ERR_INVALID_ARG, "null handle");
    const Plan &P = a->plan;
    if (qt_ptr) memcpy(qt_ptr, P.qt_ptr.data(), sizeof(int32_t) * (P.n_qt + 1));
    if (kv && P.n_entries) memcpy(kv, P.kv.data(), sizeof(int32_t) * P.n_entries);
    if (order) memcpy(order, P.order.data(), sizeof(int32_t) * P.n_qt);
    return SPLAT_OK;
}

splat_status splat_acsr_destroy(splat_acsr a)
{
    clear_error();
    if (!a) return SPLAT_OK;
    free_device(a);
    delete a;
    return SPLAT_OK;
}

splat_status splat_rsddmm(splat_acsr a, const void *Q, const void *K, splat_dtype dt, int32_t B, int32_t H,
                          int32_t d, float scale, float *S, void *stream)
{
    splat_status st = check_compute(a, B, H);
    if (st == SPLAT_OK) st = check_d(dt, d);
    if (st != SPLAT_OK) return st;
    if (!Q || !K || !S) return set_error(SPLAT_ERR_INVALID_ARG, "null tensor pointer");
    if (!aligned16(Q) || !aligned16(K) || !aligned16(S)) return set_error(SPLAT_ERR_INVALID_ARG, "tensors must be 16-byte aligned");
    DeviceGuard g(a->device);
    int nl = 1;
    cudaError_t e;
    if (dt == SPLAT_BF16 && use_residue_split(a))
        e = launch_unfused_residue(true, dev_view(a->sub_band), dev_view(a->sub_str), dev_view(a), a->rv_l, a->rv_nk,
                                   a->rv_R, Q, K, B * H, d, scale, S, (cudaStream_t)stream, &nl);
    else if (dt == SPLAT_BF16 && a->sub_perm && use_perm())
        e = launch_unfused_permuted(true, dev_view(a->sub_perm), dev_view(a), a->rv_l, a->rv_nk, a->rv_R, Q, K, B * H,
                                    d, scale, S, (cudaStream_t)stream, &nl);
    else
        e = dt == SPLAT_BF16 ? launch_rsddmm_tc(dev_view(a), Q, K, B * H, d, scale, S, (cudaStream_t)stream)
                             : launch_rsddmm_simt(dev_view(a), Q, K, false, B * H, d, scale, S, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "splat_rsddmm launch");
    note_launches(nl);
    return SPLAT_OK;
}

splat_status splat_sparse_softmax(splat_acsr a, const float *S, void *P, splat_dtype p_dt, int32_t B, int32_t H,
                                  void *stream)
{
    splat_status st = check_compute(a, B, H);
    if (st != SPLAT_OK) return st;
    if (p_dt != SPLAT_BF16 && p_dt != SPLAT_FP32) return set_error(SPLAT_ERR_INVALID_ARG, "unknown dtype %d", (int)p_dt);
    if (!S || !P) return set_error(SPLAT_ERR_INVALID_ARG, "null tensor pointer");
    if ((const void *)S == P) return set_error(SPLAT_ERR_INVALID_ARG, "P may not alias S");
    DeviceGuard g(a->device);
    cudaError_t e = launch_softmax(dev_view(a), S, P, p_dt == SPLAT_BF16, B * H, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "splat_sparse_softmax launch");
    note_launches(1);
    return SPLAT_OK;
}

splat_status splat_rspmm(splat_acsr a, const void *P, const void *V, splat_dtype dt, int32_t B, int32_t H,
                         int32_t d, void *O, void *stream)
{
    splat_status st = check_compute(a, B, H);
    if (st == SPLAT_OK) st = check_d(dt, d);
    if (st != SPLAT_OK) return st;
    if (!P || !V || !O) return set_error(SPLAT_ERR_INVALID_ARG, "null tensor pointer");
    if (!aligned16(P) || !aligned16(V) || !aligned16(O)) return set_error(SPLAT_ERR_INVALID_ARG, "tensors must be 16-byte aligned");
    DeviceGuard g(a->device);
    int nl = 1;
    cudaError_t e;
    if (dt == SPLAT_BF16 && use_residue_split(a))
        e = launch_unfused_residue(false, dev_view(a->sub_band), dev_view(a->sub_str), dev_view(a), a->rv_l, a->rv_nk,
                                   a->rv_R, P, V, B * H, d, 0.f, O, (cudaStream_t)stream, &nl);
    else if (dt == SPLAT_BF16 && a->sub_perm && use_perm())
        e = launch_unfused_permuted(false, dev_view(a->sub_perm), dev_view(a), a->rv_l, a->rv_nk, a->rv_R, P, V,
                                    B * H, d, 0.f, O, (cudaStream_t)stream, &nl);
    else
        e = dt == SPLAT_BF16 ? launch_rspmm_tc(dev_view(a), P, V, B * H, d, O, (cudaStream_t)stream)
                             : launch_rspmm_simt(dev_view(a), P, V, false, B * H, d, O, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "splat_rspmm launch");
    note_launches(nl);
    return SPLAT_OK;
}

splat_status splat_sparse_mhsa(splat_acsr a, const void *Q, const void *K, const void *V, splat_dtype dt,
                               int32_t B, int32_t H, int32_t d, float scale, void *O, void *stream)
{
    splat_status st = check_mhsa(a, Q, K, V, dt, B, H, d, scale, O);
    if (st != SPLAT_OK) return st;
    DeviceGuard g(a->device);
    cudaError_t e = launch_mhsa(a, Q, K, V, dt, B * H, d, scale, O, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "splat_sparse_mhsa launch");
    return SPLAT_OK;
}

splat_status splat_sparse_mhsa_host(splat_acsr a, const void *Qh, const void *Kh, const void *Vh, splat_dtype dt,
                                    int32_t B, int32_t H, int32_t d, float scale, void *Oh, void *dQ, void *dK,
                                    void *dV, void *dO, void *stream)
{
    splat_status st = check_mhsa(a, dQ, dK, dV, dt, B, H, d, scale, dO);
    if (st != SPLAT_OK) return st;
    if (!Qh || !Kh || !Vh || !Oh) return set_error(SPLAT_ERR_INVALID_ARG, "null host pointer");
    if (!a->hs[0]) return set_error(SPLAT_ERR_INVALID_ARG, "handle has no host pipeline (internal sub-handle)");
    const int BH = B * H;
    const size_t slice = (size_t)a->n * d * (dt == SPLAT_BF16 ? 2 : 4);    // bytes per (b, h)
    // chunk boundaries only at slice indices whose byte offset is 16-byte aligned (the kernels'
    // alignment contract): multiples of `unit` slices
    size_t gs = slice & 15u ? slice & 15u : 16u, g16 = 16;
    while (gs) { const size_t t = g16 % gs; g16 = gs; gs = t; }          // gcd(slice mod 16, 16)
    const int unit = (int)(16 / g16);
    const int n_units = (BH + unit - 1) / unit;
    const int nch = n_units >= kHostChunks ? kHostChunks : n_units;
    DeviceGuard g(a->device);
    cudaStream_t cs = (cudaStream_t)stream;
    cudaStream_t s_in = (cudaStream_t)a->hs[0], s_k = (cudaStream_t)a->hs[1], s_out = (cudaStream_t)a->hs[2];
    cudaEvent_t start = (cudaEvent_t)a->hev[0][15], fin = (cudaEvent_t)a->hev[1][15];
    // everything the caller enqueued on `stream` before this call happens first
    cudaError_t e = cudaEventRecord(start, cs);
    if (e != cudaSuccess) return cuda_fail(e, "event");
    cudaStreamWaitEvent(s_in, start, 0);
    cudaStreamWaitEvent(s_k, start, 0);
    cudaStreamWaitEvent(s_out, start, 0);
    int nl = 0;
    for (int c = 0; c < nch && e == cudaSuccess; ++c) {
        const int b0 = (int)std::min<long long>(BH, (long long)unit * ((long long)n_units * c / nch));
        const int b1 = (int)std::min<long long>(BH, (long long)unit * ((long long)n_units * (c + 1) / nch));
        if (b1 <= b0) continue;
        const size_t off = slice * b0, bytes = slice * (b1 - b0);
        auto hp = [&](const void *p) { return static_cast<const char *>(p) + off; };
        auto dp = [&](void *p) { return static_cast<char *>(p) + off; };
        cudaEvent_t done_in = (cudaEvent_t)a->hev[0][c], done_k = (cudaEvent_t)a->hev[1][c];
        e = cudaMemcpyAsync(dp(dQ), hp(Qh), bytes, cudaMemcpyHostToDevice, s_in);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dp(dK), hp(Kh), bytes, cudaMemcpyHostToDevice, s_in);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dp(dV), hp(Vh), bytes, cudaMemcpyHostToDevice, s_in);
        if (e == cudaSuccess) e = cudaEventRecord(done_in, s_in);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s_k, done_in, 0);
        if (e == cudaSuccess) e = launch_mhsa(a, dp(dQ), dp(dK), dp(dV), dt, b1 - b0, d, scale, dp(dO), s_k, false);
        nl += g_launches;
        if (e == cudaSuccess) e = cudaEventRecord(done_k, s_k);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s_out, done_k, 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(static_cast<char *>(Oh) + off, static_cast<char *>(dO) + off, bytes,
                                cudaMemcpyDeviceToHost, s_out);
    }
    // the caller's stream waits for the last copy-out and, through it, for everything queued above --
    // also after an error, so a caller that frees its buffers afterwards cannot race the copies
    cudaEventRecord(fin, s_in);
    cudaStreamWaitEvent(s_out, fin, 0);
    cudaEventRecord(fin, s_k);
    cudaStreamWaitEvent(s_out, fin, 0);
    const cudaError_t ej = cudaEventRecord(fin, s_out);
    const cudaError_t ew = ej == cudaSuccess ? cudaStreamWaitEvent(cs, fin, 0) : ej;
    if (e != cudaSuccess) return cuda_fail(e, "splat_sparse_mhsa_host");
    if (ew != cudaSuccess) return cuda_fail(ew, "pipeline join");
    note_launches(nl);
    return SPLAT_OK;
}

// ---- data-layout reordering (NEXT #3): column-compressed ACSR values for R-SpMM
splat_status splat_acsr_transpose(splat_acsr a, void *stream, splat_acsr *at)
{
    clear_error();
    if (!a || !at) return set_error(SPLAT_ERR_INVALID_ARG, "null handle or out pointer");
    *at = nullptr;
    const int n = a->n;
    if (n > kMaxMaskN) return set_error(SPLAT_ERR_UNSUPPORTED, "transpose needs N <= %d, got %d", kMaxMaskN, n);
    const size_t W = ((size_t)n + 31) / 32;
    std::vector<uint32_t> mt;
    try {
        mt.assign((size_t)n * W, 0u);
    } catch (const std::exception &) {
        return set_error(SPLAT_ERR_OOM, "host allocation of the transposed mask failed");
    }
    // M^T as an explicit bit mask: row c of M^T holds bit i for every non-zero (i, c) of M
    for (int i = 0; i < n; ++i)
        for (int s = 0; s < a->nseg_h[i]; ++s) {
            const int32_t *g = &a->seg_h[(size_t)i * 16 + 4 * s];
            for (int x = 0; x < g[2]; ++x) {
                const int c = g[0] + g[1] * x;
                mt[(size_t)c * W + (size_t)(i >> 5)] |= 1u << (i & 31);
            }
        }
    if (a->device < 0) return splat_acsr_from_mask(mt.data(), n, SPLAT_MAX_SEGS, -1, stream, at, nullptr, nullptr);
    DeviceGuard g(a->device);
    uint32_t *d = nullptr;
    cudaError_t e = dev_alloc(&d, mt.size() * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemcpy(d, mt.data(), mt.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(d);
        return cuda_fail(e, "transposed mask upload");
    }
    const splat_status st = splat_acsr_from_mask(d, n, SPLAT_MAX_SEGS, a->device, stream, at, nullptr, nullptr);
    cudaFree(d);      // the build is synchronous
    return st;
}

splat_status splat_transpose_values(splat_acsr a, splat_acsr at, const void *X, void *Y, splat_dtype dt, int32_t B,
                                    int32_t H, void *stream)
{
    splat_status st = check_compute(a, B, H);
    if (st != SPLAT_OK) return st;
    if (!at || at->device != a->device || at->n != a->n || at->nnz != a->nnz)
        return set_error(SPLAT_ERR_INVALID_ARG, "at is not the transpose handle of a (splat_acsr_transpose)");
    if (dt != SPLAT_BF16 && dt != SPLAT_FP32) return set_error(SPLAT_ERR_INVALID_ARG, "unknown dtype %d", (int)dt);
    if (!X || !Y) return set_error(SPLAT_ERR_INVALID_ARG, "null tensor pointer");
    DeviceGuard g(a->device);
    const cudaError_t e = launch_transpose_values(dev_view(a), dev_view(at), X, Y, dt == SPLAT_BF16, B * H,
                                                  (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "splat_transpose_values launch");
    note_launches(1);
    return SPLAT_OK;
}

splat_status splat_rspmm_cc(splat_acsr a, splat_acsr at, const void *PT, const void *V, splat_dtype dt, int32_t B,
                            int32_t H, int32_t d, void *O, void *stream)
{
    splat_status st = check_compute(a, B, H);
    if (st != SPLAT_OK) return st;
    if (!at || at->device != a->device || at->n != a->n || at->nnz != a->nnz)
        return set_error(SPLAT_ERR_INVALID_ARG, "at is not the transpose handle of a (splat_acsr_transpose)");
    if (dt != SPLAT_BF16 && dt != SPLAT_FP32) return set_error(SPLAT_ERR_INVALID_ARG, "unknown dtype %d", (int)dt);
    if (d < 1 || d > 256) return set_error(SPLAT_ERR_UNSUPPORTED, "splat_rspmm_cc needs 1 <= d <= 256, got %d", d);
    if (!PT || !V || !O) return set_error(SPLAT_ERR_INVALID_ARG, "null tensor pointer");
    // Fig. 14 ablation knob (diagnostics build only; 0 in the product build): SPLAT_CC_ALIGN = X runs
    // the lanes along the stride lattice of STRIDED(X)
    const int align_x = diag_env("SPLAT_CC_ALIGN");
    if (align_x > 1 && a->n % align_x != 0) return set_error(SPLAT_ERR_INVALID_ARG, "SPLAT_CC_ALIGN must divide N");
    DeviceGuard g(a->device);
    const cudaError_t e = launch_rspmm_cc(dev_view(a), dev_view(at), PT, V, dt == SPLAT_BF16, B * H, d, O,
                                          (cudaStream_t)stream, align_x);
    if (e != cudaSuccess) return cuda_fail(e, "splat_rspmm_cc launch");
    note_launches(1);
    return SPLAT_OK;
}

int32_t splat_layout_choice(splat_acsr a, double alpha)
{
    if (!a || a->n < 1) return 0;
    const double density = (double)a->nnz / ((double)a->n * (double)a->n);
    return density >= alpha ? 1 : 0;
}

double splat_flops(splat_acsr a, int32_t B, int32_t H, int32_t d)
{
    if (!a) return 0.0;
    return 4.0 * (double)a->nnz * (double)d * (double)B * (double)H;
}

int32_t splat_last_launch_count(void) { return g_launches; }

int64_t splat_device_alloc_count(void) { return g_allocs.load(); }

const char *splat_last_error(void) { return g_err; }

}  // extern "C"
