// Microbenchmark (B200, sm_100a): tcgen05.mma throughput for the fused kernel's two shapes --
// SS (A, B from SMEM, K-major; the S = Q K^T MMA) and TS (A from TMEM; the O += P V MMA with
// an MN-major B) at M = 128, N in {64, 128, 256}, K = 16.  One CTA per SM, one issuing thread;
// cycles for n back-to-back MMAs from first issue to commit completion.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

__global__ void __launch_bounds__(128, 1) k(unsigned long long *out, int n, int N, int ts, int mn)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t *>(smem)[i] = 0x3c003c00u;
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t s = smem_u32(smem);
        const uint32_t id = idesc_bf16(128, N, mn != 0);
        unsigned long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
            if (ts)
                mma_bf16_ts(tm + 256, tm + (i & 7) * 8,
                            mn ? sdesc_sw128(s + 32768 + (i & 7) * 2048, 16384, 1024)
                               : sdesc_sw128(s + 32768 + (i & 3) * 32, 16, 1024), id, 1);
            else
                mma_bf16_ss(tm + 256, sdesc_sw128(s + (i & 3) * 32, 16, 1024),
                            mn ? sdesc_sw128(s + 32768 + (i & 7) * 2048, 16384, 1024)
                               : sdesc_sw128(s + 32768 + (i & 3) * 32, 16, 1024), id, 1);
        }
        unsigned long long t1 = clock64();
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t2 = clock64();
        out[blockIdx.x * 2 + 0] = t1 - t0;
        out[blockIdx.x * 2 + 1] = t2 - t0;
    }
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, 512);
}

int main()
{
    unsigned long long *d;
    cudaMalloc(&d, 1 << 20);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
    for (int ts : {0, 1})
        for (int mn : {0, 1})
            for (int N : {64, 128, 256}) {
                if (N == 256 && mn) continue;
                for (int n : {8, 64}) {
                    k<<<148, 128, 66 * 1024 + 1024>>>(d, n, N, ts, mn);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                    unsigned long long h[2];
                    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                    printf("%s B-%s M=128 N=%3d K=16 x%2d: issue %5llu cyc, done %6llu cyc = %.1f cyc/MMA (ideal %d)\n",
                           ts ? "TS" : "SS", mn ? "MN" : "K ", N, n, h[0], h[1], (double)h[1] / n, N / 2);
                }
            }
    return 0;
}
