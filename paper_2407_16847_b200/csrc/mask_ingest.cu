// mask_ingest.cu -- ACSR build from an explicit bit mask.
//
// The paper's analysis pass as written: checkRegularity(Mask) then generateACSRMetadata(Mask)
// (Listing 4; construction Sec. 5.1).  Each row's non-zero columns are
// split into the canonical greedy runs (reading R-4: the 2x2 solve on the first two unconsumed
// columns, extended while the next column passes P:219, restarted at the first failing
// column); a row that needs more than `max_runs` runs makes the mask NOT_REGULAR and the first
// such (row, column) in row-major order -- the column that would start run max_runs + 1 -- is
// reported.  max_runs = 1 is Def. 1's regularity.
//
// One warp per row, all arithmetic on 32-bit mask words, with one primitive, scan():
//   scan(from)               the first set column >= from;
//   scan(c0, lattice step)   the first column >= c0 whose bit differs from the run's lattice
//                            {c0 + t step}; every column of the lattice before it belongs to the
//                            run and the next run starts at the first set column from there.
// A run costs three scans; a row is read from HBM once (the rescans hit L1).  The mask is
// N^2 / 8 bytes (134 MB at N = 32768), so the kernel is an HBM-bound stream.  Its limit is
// memory-level parallelism, not volume: each scan iteration is a dependent load -> ballot, so a
// warp keeps 2 x 512 B in flight (two 16-byte loads per lane) and 64 warps per SM (8 per CTA,
// one row per warp, adjacent rows in flight together) cover HBM latency.
#include <cuda_runtime.h>

#include "kernels.h"
#include "splat_internal.h"

namespace splat {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// bits of word w that take part in a scan starting at column `from` (none outside [from, N))
__device__ __forceinline__ uint32_t valid_bits(int w, int W, int N, int from)
{
    if (w < (from >> 5) || w >= W) return 0u;
    uint32_t v = kFull;
    if (w == (from >> 5)) v &= kFull << (from & 31);
    if (w == W - 1 && (N & 31)) v &= (1u << (N & 31)) - 1u;
    return v;
}

// bits of word w on the lattice {c0 + t step : t >= 0}: the lattice hits the word's bit positions
// r, r + step, ... with r = (c0 - 32 w) mod step (or c0 - 32 w when the word starts before c0),
// i.e. the word is base << r, base = the bits 0, step, 2 step, ... of one word.
__device__ __forceinline__ uint32_t lattice_word(int w, int c0, int step, uint32_t base)
{
    const int lo = w * 32;
    if (lo <= c0) return c0 - lo < 32 ? base << (c0 - lo) : 0u;
    if (step == 1) return kFull;
    const int r = (step - (lo - c0) % step) % step;
    return r < 32 ? base << r : 0u;
}

__device__ __forceinline__ uint32_t lattice_base(int step)
{
    if (step == 1) return kFull;
    uint32_t e = 0u;
    for (int x = 0; x < 32; x += step) e |= 1u << x;
    return e;
}

template <int G>
__device__ __forceinline__ void load_words(const uint32_t *__restrict__ row, int w, int W, uint32_t (&v)[G])
{
    if (w < W) {
        if constexpr (G == 4) {
            const uint4 t = __ldg(reinterpret_cast<const uint4 *>(row + w));
            v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
#pragma unroll
            for (int g = 0; g < G; ++g) v[g] = __ldg(row + w + g);
        }
    } else {
#pragma unroll
        for (int g = 0; g < G; ++g) v[g] = 0u;
    }
}

// First column >= from (and < N) whose bit is set (step == 0) or differs from the lattice
// {c0 + t step} (step > 0); N if none.  The warp reads 64 G consecutive words per iteration, G
// per lane (16-byte loads when G == 4), both halves issued before the first ballot.  Only the
// lanes holding the first word (from >> 5) or the last one (W - 1) mask bits; the position is
// resolved by the first lane with a hit after the ballot.
template <int G>
__device__ __forceinline__ int scan(const uint32_t *__restrict__ row, int W, int N, int from, int c0, int step,
                                    int lane, int *next = nullptr)
{
    if (from >= N) return N;
    const int fw = from >> 5;
    const uint32_t base = step ? lattice_base(step) : 0u;
    for (int w0 = fw & ~(G - 1); w0 < W; w0 += 64 * G) {
        uint32_t v[2][G];
#pragma unroll
        for (int h = 0; h < 2; ++h) load_words<G>(row, w0 + (h * 32 + lane) * G, W, v[h]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int wb = w0 + (h * 32 + lane) * G;
            const bool edge = wb <= fw || wb + G >= W;
            uint32_t any = 0u;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                if (step) v[h][g] ^= lattice_word(wb + g, c0, step, base);
                if (edge) v[h][g] &= valid_bits(wb + g, W, N, from);
                any |= v[h][g];
            }
            const unsigned b = __ballot_sync(kFull, any != 0u);
            if (b) {
                int loc = -1, loc2 = -1;  // first hit; second hit in the same lane's words (or -1)
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint32_t x = v[h][g];
                    if (x && loc2 < 0) {
                        if (loc < 0) {
                            loc = (wb + g) * 32 + __ffs(x) - 1;
                            const uint32_t y = x & (x - 1u);
                            if (y) loc2 = (wb + g) * 32 + __ffs(y) - 1;
                        } else {
                            loc2 = (wb + g) * 32 + __ffs(x) - 1;
                        }
                    }
                }
                const int l = __ffs(b) - 1;
                if (next) *next = __shfl_sync(kFull, loc2, l);
                return __shfl_sync(kFull, loc, l);
            }
        }
    }
    return N;
}

template <int G>
__global__ void __launch_bounds__(256, 8) acsr_mask_kernel(const uint32_t *__restrict__ mask, int N, int W,
                                                        int max_runs, int4 *__restrict__ seg,
                                                        uint8_t *__restrict__ nseg, int64_t *__restrict__ row_ptr,
                                                        unsigned long long *__restrict__ bad)
{
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= N) return;
    const uint32_t *row = mask + (size_t)i * W;
    int4 *out = seg + (size_t)i * SPLAT_MAX_SEGS;
    int pos = 0, nr = 0, off = 0;
    while (true) {
        int c1 = -1;
        const int c0 = scan<G>(row, W, N, pos, 0, 0, lane, &c1);
        if (c0 >= N) break;
        if (nr == max_runs) {
            if (lane == 0) atomicMin(bad, ((unsigned long long)i << 32) | (unsigned)c0);
            break;
        }
        if (c1 < 0) c1 = scan<G>(row, W, N, c0 + 1, 0, 0, lane);   // not in the same lane's words
        int step = 1, cnt = 1, q = N;
        if (c1 < N) {
            step = c1 - c0;
            q = scan<G>(row, W, N, c0, c0, step, lane);
            cnt = (q - c0 + step - 1) / step;
        }
        if (lane == 0) out[nr] = make_int4(c0, step, cnt, off);
        off += cnt;
        ++nr;
        pos = q;
    }
    if (lane == 0) {
        for (int k = nr; k < SPLAT_MAX_SEGS; ++k) out[k] = make_int4(0, 0, 0, off);
        nseg[i] = (uint8_t)nr;
        row_ptr[i + 1] = off;
        if (i == 0) row_ptr[0] = 0;
    }
}

// Register-resident variant for rows of at most 128 JG words (N <= 4096 JG, JG <= 2; 16-byte aligned rows):
// the warp loads its whole row up front (JG 16-byte loads per lane, all in flight together) and
// every scan then runs on registers -- no dependent load per scan step, and no re-reads.
template <int JG>
__global__ void __launch_bounds__(256) acsr_mask_reg_kernel(const uint32_t *__restrict__ mask, int N, int W,
                                                            int max_runs, int4 *__restrict__ seg,
                                                            uint8_t *__restrict__ nseg,
                                                            int64_t *__restrict__ row_ptr,
                                                            unsigned long long *__restrict__ bad)
{
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= N) return;
    const uint4 *row4 = reinterpret_cast<const uint4 *>(mask + (size_t)i * W);
    uint32_t v[JG][4];
#pragma unroll
    for (int j = 0; j < JG; ++j) {
        const int q = j * 32 + lane;
        uint4 t = make_uint4(0u, 0u, 0u, 0u);
        if (4 * q < W) t = __ldg(row4 + q);
        v[j][0] = t.x; v[j][1] = t.y; v[j][2] = t.z; v[j][3] = t.w;
    }
    const uint32_t last_valid = (N & 31) ? (1u << (N & 31)) - 1u : kFull;
#pragma unroll
    for (int j = 0; j < JG; ++j)
#pragma unroll
        for (int g = 0; g < 4; ++g)
            if (128 * j + 4 * lane + g == W - 1) v[j][g] &= last_valid;
    // first column >= from that is set (step == 0) or off the lattice {c0 + t step}; N if none
    auto scan = [&](int from, int c0, int step, int *next) -> int {
        if (from >= N) return N;
        const int fw = from >> 5;
        const uint32_t base = step ? lattice_base(step) : 0u;
#pragma unroll
        for (int j = 0; j < JG; ++j) {
            if (128 * j + 127 < fw) continue;                 // warp-uniform: group before `from`
            uint32_t d[4], any = 0u;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const int w = 128 * j + 4 * lane + g;
                d[g] = v[j][g];
                if (step) d[g] ^= lattice_word(w, c0, step, base);
                if (w < fw || w >= W) d[g] = 0u;
                else if (w == fw) d[g] &= kFull << (from & 31);
                if (w == W - 1) d[g] &= last_valid;
                any |= d[g];
            }
            const unsigned b = __ballot_sync(kFull, any != 0u);
            if (b) {
                int loc = -1, loc2 = -1;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const uint32_t x = d[g];
                    const int w = 128 * j + 4 * lane + g;
                    if (x && loc2 < 0) {
                        if (loc < 0) {
                            loc = w * 32 + __ffs(x) - 1;
                            const uint32_t y = x & (x - 1u);
                            if (y) loc2 = w * 32 + __ffs(y) - 1;
                        } else {
                            loc2 = w * 32 + __ffs(x) - 1;
                        }
                    }
                }
                const int l = __ffs(b) - 1;
                if (next) *next = __shfl_sync(kFull, loc2, l);
                return __shfl_sync(kFull, loc, l);
            }
        }
        return N;
    };
    int4 *out = seg + (size_t)i * SPLAT_MAX_SEGS;
    int pos = 0, nr = 0, off = 0;
    while (true) {
        int c1 = -1;
        const int c0 = scan(pos, 0, 0, &c1);
        if (c0 >= N) break;
        if (nr == max_runs) {
            if (lane == 0) atomicMin(bad, ((unsigned long long)i << 32) | (unsigned)c0);
            break;
        }
        if (c1 < 0) c1 = scan(c0 + 1, 0, 0, nullptr);
        int step = 1, cnt = 1, q = N;
        if (c1 < N) {
            step = c1 - c0;
            q = scan(c0, c0, step, nullptr);
            cnt = (q - c0 + step - 1) / step;
        }
        if (lane == 0) out[nr] = make_int4(c0, step, cnt, off);
        off += cnt;
        ++nr;
        pos = q;
    }
    if (lane == 0) {
        for (int k = nr; k < SPLAT_MAX_SEGS; ++k) out[k] = make_int4(0, 0, 0, off);
        nseg[i] = (uint8_t)nr;
        row_ptr[i + 1] = off;
        if (i == 0) row_ptr[0] = 0;
    }
}

}  // namespace

cudaError_t launch_acsr_from_mask(const uint32_t *mask, int n, int max_runs, int4 *seg, uint8_t *nseg,
                                  int64_t *row_ptr, unsigned long long *bad, cudaStream_t st)
{
    const int W = (n + 31) / 32;
    cudaError_t e = cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    // 16-byte loads when every row starts 16-byte aligned; whole rows in registers up to 256 words
    // (wider register-resident rows cost occupancy: measured slower at 1024 words, 76 vs 51 us)
    const bool al = W % 4 == 0 && (reinterpret_cast<uintptr_t>(mask) & 15u) == 0;
    const int grid = (n + 7) / 8;
    if (al && W <= 128)
        acsr_mask_reg_kernel<1><<<grid, 256, 0, st>>>(mask, n, W, max_runs, seg, nseg, row_ptr, bad);
    else if (al && W <= 256)
        acsr_mask_reg_kernel<2><<<grid, 256, 0, st>>>(mask, n, W, max_runs, seg, nseg, row_ptr, bad);
    else if (al)
        acsr_mask_kernel<4><<<grid, 256, 0, st>>>(mask, n, W, max_runs, seg, nseg, row_ptr, bad);
    else
        acsr_mask_kernel<1><<<(n + 7) / 8, 256, 0, st>>>(mask, n, W, max_runs, seg, nseg, row_ptr, bad);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_acsr_scan(row_ptr, n, st);
}

}  // namespace splat

// Timing hook (not part of the public ABI): the ingest kernels alone, asynchronous on `stream`,
// into caller-owned device buffers (seg [n][4] int4, nseg [n], row_ptr [n+1], bad [1]).
extern "C" int splat_debug_mask_ingest(const uint32_t *mask, int n, int max_runs, void *seg, void *nseg,
                                       void *row_ptr, void *bad, void *stream)
{
    return (int)splat::launch_acsr_from_mask(mask, n, max_runs, static_cast<int4 *>(seg),
                                             static_cast<uint8_t *>(nseg), static_cast<int64_t *>(row_ptr),
                                             static_cast<unsigned long long *>(bad), (cudaStream_t)stream);
}
