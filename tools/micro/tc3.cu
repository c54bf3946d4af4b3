// Microbenchmark (B200): back-to-back tcgen05.mma throughput (x64, one thread issues), SS vs TS
// (A from TMEM), M = 128, N in {32, 64, 128}.  Cycles per K = 16 instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

__global__ void __launch_bounds__(128, 1) k(unsigned long long *out, int N, int ts)
{
    extern __shared__ __align__(1024) uint8_t smem[];
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
    if (warp == 0) {
        const uint32_t s = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
        const uint32_t tmu = __shfl_sync(0xffffffffu, tm, 0);
        const int Nu = __shfl_sync(0xffffffffu, N, 0), tsu = __shfl_sync(0xffffffffu, ts, 0);
        const uint32_t id = idesc_bf16(128, Nu, tsu != 0);
        const uint64_t da = sdesc_sw128(s, 16, 1024), db = sdesc_sw128(s + 32768, 16, 1024);
        const uint64_t dv = sdesc_sw128(s + 32768, 16384, 1024);
        unsigned long long t0 = clock64();
        if (tsu) {
            for (int i = 0; i < 64; ++i) {
                uint32_t pred;
                asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
                if (pred) mma_bf16_ts(tmu, tmu + 256 + (i & 3) * 8, dv + (uint64_t)((i & 3) * 128), id, 1);
                __syncwarp();
            }
        } else {
            for (int i = 0; i < 64; ++i) {
                uint32_t pred;
                asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
                if (pred) mma_bf16_ss(tmu, da + (uint64_t)((i & 3) * 2), db + (uint64_t)((i & 3) * 2), id, 1);
                __syncwarp();
            }
        }
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, 512);
}

int main()
{
    unsigned long long *d;
    cudaMalloc(&d, 1 << 20);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int ts : {0, 1})
        for (int N : {32, 64, 96, 128}) {
            k<<<148, 128, 65536>>>(d, N, ts);
            if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double a = 0; for (int i = 0; i < 148; ++i) a += h[i]; a /= 148;
            printf("%s M=128 N=%3d: %.1f cycles per K=16 MMA (64 back to back)\n", ts ? "TS" : "SS", N, a / 64);
        }
    return 0;
}
