// Microbenchmark (B200): back-to-back tcgen05.mma cost (cycles per K=16 instruction) by M, N and
// operand source (SS: A and B in SMEM; TS: A in TMEM).  One CTA per SM, one issuing warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

__global__ void __launch_bounds__(128, 1) k(unsigned long long *out, int nm, int M, int N, int ts)
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
        const uint32_t s = smem_u32(smem);
        const uint32_t id = idesc_bf16(M, N, ts != 0);
        const uint64_t da = sdesc_sw128(s, 16, 1024), db = sdesc_sw128(s + 32768, ts ? 16384 : 16, 1024);
        // warm
        for (int i = 0; i < 8; ++i) {
            if (elect_one()) {
                if (ts) mma_bf16_ts(tm, tm + 256 + (i & 3) * 8, db, id, 1);
                else mma_bf16_ss(tm, da + (uint64_t)((i & 3) * 2), db + (uint64_t)((i & 3) * 2), id, 1);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        unsigned long long t0 = clock64();
        for (int i = 0; i < nm; ++i) {
            if (elect_one()) {
                if (ts) mma_bf16_ts(tm, tm + 256 + (i & 3) * 8, db, id, 1);
                else mma_bf16_ss(tm, da + (uint64_t)((i & 3) * 2), db + (uint64_t)((i & 3) * 2), id, 1);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 1);
        unsigned long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, 512);
}

int main()
{
    unsigned long long *d;
    cudaMalloc(&d, 1 << 20);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    for (int ts : {0, 1})
        for (int M : {64, 128})
            for (int N : {16, 32, 64, 80, 128, 256}) {
                const int nm = 256;
                k<<<148, 128, 66 * 1024>>>(d, nm, M, N, ts);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("M=%d N=%d ts=%d err %s\n", M, N, ts, cudaGetErrorString(e)); return 1; }
                unsigned long long h[148];
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
                printf("%s M=%3d N=%3d K=16: %.1f cycles per MMA (%.0f FLOP/clk)\n", ts ? "TS" : "SS", M, N, avg / nm,
                       2.0 * M * N * 16 / (avg / nm));
            }
    return 0;
}
