// acsr.cu -- ACSR metadata build on the GPU.
//
// PAPER Sec. 5.1: per row the affine indices (a, b, nnzs) of its
// non-zero columns, O(rows) metadata; row_ptr locates each row in the
// row-compressed row-major value arrays (Fig. 5(b)).  The paper computes the
// indices on the host from an explicit mask (Listing 4).  Here the
// mask is a descriptor, so one thread per row evaluates the closed-form
// canonical runs (splat::row_segments), and a single-CTA scan produces
// row_ptr (int64).  N <= 2^24, so the metadata is at most ~1 GB and usually
// ~2 MB (Mistral N = 32768: 2.1 MB): the build is latency-bound.
#include <cuda_runtime.h>

#include "kernels.h"
#include "splat_internal.h"

namespace splat {

// One thread per row: runs -> seg[i][s] = (start, step, count, offset-in-row),
// nseg[i], and the row count into row_ptr[i+1] (scanned afterwards).
__global__ void acsr_rows_kernel(splat_pattern p, int4 *__restrict__ seg, uint8_t *__restrict__ nseg,
                                 int64_t *__restrict__ row_ptr)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.seq_len) return;
    Seg s[4];
    const int n = row_segments(p, i, s);
    int off = 0;
    int4 out[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k < n) {
            out[k] = make_int4(s[k].start, s[k].step, s[k].count, off);
            off += s[k].count;
        } else {
            out[k] = make_int4(0, 0, 0, off);
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) seg[(size_t)i * 4 + k] = out[k];
    nseg[i] = (uint8_t)n;
    row_ptr[i + 1] = off;
    if (i == 0) row_ptr[0] = 0;
}

// In-place inclusive scan of row_ptr[1..N] with one 1024-thread CTA, in tiles of 4096 counts
// staged through shared memory: coalesced global loads / stores (element base + 1024 k + t),
// thread t scans its 4 consecutive counts from SMEM, the 1024 thread totals are scanned with warp
// shuffles, and a running carry joins the tiles; the next tile's loads are issued before the
// current tile is scanned.  Exact int64 arithmetic.
__global__ void __launch_bounds__(1024) acsr_scan_kernel(int64_t *__restrict__ row_ptr, int n)
{
    constexpr int PER = 4, TILE = 1024 * PER;
    __shared__ int64_t buf[TILE];
    __shared__ int64_t warp_tot[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    int64_t *x = row_ptr + 1;   // x[0..n-1] = counts of rows 0..n-1
    int64_t carry = 0;
    int64_t nxt[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) nxt[k] = k * 1024 + t < n ? x[k * 1024 + t] : 0;
    for (int base = 0; base < n; base += TILE) {
#pragma unroll
        for (int k = 0; k < PER; ++k) buf[k * 1024 + t] = nxt[k];
        if (base + TILE < n) {
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int i = base + TILE + k * 1024 + t;
                nxt[k] = i < n ? x[i] : 0;
            }
        }
        __syncthreads();
        int64_t cur[PER], sum = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            sum += buf[PER * t + k];
            cur[k] = sum;
        }
        int64_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) warp_tot[w] = inc;
        __syncthreads();
        if (w == 0) {
            int64_t v = warp_tot[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += y;
            }
            warp_tot[lane] = v;   // inclusive over warps
        }
        __syncthreads();
        const int64_t prefix = carry + inc - sum + (w > 0 ? warp_tot[w - 1] : 0);
#pragma unroll
        for (int k = 0; k < PER; ++k) buf[PER * t + k] = prefix + cur[k];
        carry += warp_tot[31];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = base + k * 1024 + t;
            if (i < n) x[i] = buf[k * 1024 + t];
        }
        __syncthreads();      // buf and warp_tot are rewritten by the next tile
    }
}

cudaError_t launch_acsr_build(const splat_pattern &p, int4 *seg, uint8_t *nseg, int64_t *row_ptr,
                              cudaStream_t st)
{
    const int n = p.seq_len;
    acsr_rows_kernel<<<(n + 255) / 256, 256, 0, st>>>(p, seg, nseg, row_ptr);
    return launch_acsr_scan(row_ptr, n, st);
}

// Multi-CTA scan for n > 32 tiles: per-tile sums (one CTA per 8192 counts), an in-place scan of
// the sums by acsr_scan_kernel, then every tile scans itself from its offset.  The single-CTA
// kernel alone is latency-bound (~7 us per tile on B200: 28 us at N = 32768, ~14 ms at 2^24).
__global__ void __launch_bounds__(1024) acsr_tile_sum_kernel(const int64_t *__restrict__ row_ptr, int n,
                                                             int64_t *__restrict__ sums)
{
    __shared__ int64_t warp_tot[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t *x = row_ptr + 1;
    const long long base = (long long)blockIdx.x * 8192 + t * 8;
    int64_t sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (base + k < n) sum += x[base + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) warp_tot[w] = sum;
    __syncthreads();
    if (w == 0) {
        int64_t v = warp_tot[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sums[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(1024) acsr_tile_apply_kernel(int64_t *__restrict__ row_ptr, int n,
                                                               const int64_t *__restrict__ incl)
{
    __shared__ int64_t warp_tot[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    int64_t *x = row_ptr + 1;
    const long long base = (long long)blockIdx.x * 8192 + t * 8;
    int64_t cur[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        cur[k] = base + k < n ? x[base + k] : 0;
        sum += cur[k];
        cur[k] = sum;
    }
    int64_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    if (w == 0) {
        int64_t v = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        warp_tot[lane] = v;
    }
    __syncthreads();
    const int64_t prefix = (blockIdx.x > 0 ? incl[blockIdx.x - 1] : 0) + inc - sum + (w > 0 ? warp_tot[w - 1] : 0);
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (base + k < n) x[base + k] = prefix + cur[k];
}

cudaError_t launch_acsr_scan(int64_t *row_ptr, int n, cudaStream_t st)
{
    constexpr int TILE = 8192;   // multi-CTA tile (acsr_tile_*_kernel); the single CTA stages 4096
    // the multi-CTA path adds a stream-ordered allocation: it only pays beyond a few dozen tiles
    if (n <= 32 * TILE) {
        acsr_scan_kernel<<<1, 1024, 0, st>>>(row_ptr, n);
        return cudaGetLastError();
    }
    const int nb = (n + TILE - 1) / TILE;
    int64_t *sums = nullptr;
    cudaError_t e = dev_alloc_async(reinterpret_cast<void **>(&sums), sizeof(int64_t) * (size_t)nb, st);
    if (e != cudaSuccess) return e;
    acsr_tile_sum_kernel<<<nb, 1024, 0, st>>>(row_ptr, n, sums);
    acsr_scan_kernel<<<1, 1024, 0, st>>>(sums - 1, nb);     // inclusive scan of sums[0..nb-1]
    acsr_tile_apply_kernel<<<nb, 1024, 0, st>>>(row_ptr, n, sums);
    e = cudaGetLastError();
    cudaError_t e2 = cudaFreeAsync(sums, st);
    return e != cudaSuccess ? e : e2;
}

}  // namespace splat
