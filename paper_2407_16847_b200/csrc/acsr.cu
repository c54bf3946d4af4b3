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

// In-place inclusive scan of row_ptr[1..N] with one 1024-thread CTA: each
// thread scans a contiguous chunk, the chunk totals are scanned with warp
// shuffles, then each chunk adds its prefix.  Exact int64 arithmetic.
__global__ void __launch_bounds__(1024) acsr_scan_kernel(int64_t *__restrict__ row_ptr, int n)
{
    __shared__ int64_t warp_tot[32];
    const int t = threadIdx.x, nt = blockDim.x;
    const int chunk = (n + nt - 1) / nt;
    const int b = 1 + t * chunk, e = min(n + 1, b + chunk);
    int64_t sum = 0;
    for (int i = b; i < e; ++i) sum += row_ptr[i];
    // exclusive scan of per-thread sums
    int64_t x = sum;
    const int lane = t & 31, w = t >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t v = lane < (nt >> 5) ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        warp_tot[lane] = v;   // inclusive over warps
    }
    __syncthreads();
    int64_t prefix = x - sum + (w > 0 ? warp_tot[w - 1] : 0);
    for (int i = b; i < e; ++i) {
        prefix += row_ptr[i];
        row_ptr[i] = prefix;
    }
}

cudaError_t launch_acsr_build(const splat_pattern &p, int4 *seg, uint8_t *nseg, int64_t *row_ptr,
                              cudaStream_t st)
{
    const int n = p.seq_len;
    acsr_rows_kernel<<<(n + 255) / 256, 256, 0, st>>>(p, seg, nseg, row_ptr);
    acsr_scan_kernel<<<1, 1024, 0, st>>>(row_ptr, n);
    return cudaGetLastError();
}

}  // namespace splat
