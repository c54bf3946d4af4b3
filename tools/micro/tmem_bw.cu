// Microbenchmark (B200, sm_100a): tcgen05.ld read bandwidth of TMEM per SM in the softmax's access
// pattern -- each warp loads a 128-column fp32 row block of its lane quadrant with 4 x
// tcgen05.ld.32x32b.x32 and one wait, repeatedly -- for 4 / 8 / 12 / 16 warps per CTA (one CTA per
// SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tmem_bw.cu -o tmem_bw && ./tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

constexpr int kIters = 256;

__global__ void __launch_bounds__(512, 1) k(unsigned long long *out, int nw)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&slot, 512);
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem_raw)[i] = 0x3c003c00u;
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    if (warp < nw) {
        // warp w: lane quadrant w % 4, columns 128 (w / 4 % 3) .. + 127 (three 128-column blocks)
        const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16) + 128 * ((warp >> 2) % 3);
        float acc = 0.f;
        unsigned long long t0 = clock64();
        for (int i = 0; i < kIters; ++i) {
            float v[128];
            tmem_ld32(base, v);
            tmem_ld32(base + 32, v + 32);
            tmem_ld32(base + 64, v + 64);
            tmem_ld32(base + 96, v + 96);
            tmem_wait_ld();
            acc += v[0] + v[37] + v[64] + v[127];   // static indices: v stays in registers
        }
        unsigned long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + warp] = t1 - t0;
        if (acc == 1234.5f) out[0] = 0;
    }
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, 512);
}

int main()
{
    unsigned long long *d;
    cudaMalloc(&d, 1 << 20);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    for (int mma : {0}) {
        for (int nw : {1, 2, 4, 8, 12, 16}) {
            cudaMemset(d, 0, 1 << 20);
            k<<<148, 16 * 32, 66 * 1024>>>(d, nw);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            unsigned long long h[148 * 32];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double mx = 0, mean = 0;
            for (int w = 0; w < nw; ++w) { mx = h[w] > mx ? h[w] : mx; mean += h[w]; }
            mean /= nw;
            const double bytes = (double)nw * kIters * 128 * 128 * 4 / 4;   // per warp: 32 lanes x 128 cols x 4 B
            printf("mma=%d warps=%2d  cycles(max)=%8.0f  per-warp iter=%6.1f cyc  SM read BW=%6.1f B/cyc\n", mma, nw, mx,
                   mean / kIters, bytes / mx);
        }
    }
    return 0;
}
