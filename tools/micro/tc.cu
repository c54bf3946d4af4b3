// Microbenchmarks (B200, sm_100a): tcgen05.mma issue cost / throughput, commit->mbarrier
// latency, tcgen05.ld / st bandwidth and latency.  One CTA per SM, 128 threads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

__global__ void __launch_bounds__(128, 1) k_mma(unsigned long long *out, int n_mma, int N)
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
    if (warp == 0 && n_mma < 0) {
        // whole warp runs the loop (uniform control flow); one elected lane issues the MMA
        const int nm = -n_mma;
        const uint32_t s = smem_u32(smem);
        const uint32_t id = idesc_bf16(128, N, false);
        const uint64_t da = sdesc_sw128(s, 16, 1024), db = sdesc_sw128(s + 32768, 16, 1024);
        unsigned long long t0 = clock64();
        for (int i = 0; i < nm; ++i) {
            uint32_t pred;
            asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
            if (pred) mma_bf16_ss(tm, da + (uint64_t)((i & 3) * 2), db + (uint64_t)((i & 3) * 2), id, 1);
            __syncwarp();
        }
        unsigned long long t1 = clock64();
        if (threadIdx.x == 0) {
            mma_commit(&bar);
            mbar_wait(&bar, 0);
        }
        __syncwarp();
        unsigned long long t2 = clock64();
        if (threadIdx.x == 0) {
            mma_commit(&bar);
            mbar_wait(&bar, 1);
            unsigned long long t3 = clock64();
            out[blockIdx.x * 4 + 0] = t1 - t0;
            out[blockIdx.x * 4 + 1] = t2 - t0;
            out[blockIdx.x * 4 + 2] = t3 - t2;
        }
    } else if (threadIdx.x == 0 && n_mma > 0) {
        const uint32_t s = smem_u32(smem);
        const uint32_t id = idesc_bf16(128, N, false);
        unsigned long long t0 = clock64();
        for (int i = 0; i < n_mma; ++i)
            mma_bf16_ss(tm, sdesc_sw128(s + (i & 3) * 32, 16, 1024), sdesc_sw128(s + 32768 + (i & 3) * 32, 16, 1024), id, 1);
        unsigned long long t1 = clock64();
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t2 = clock64();
        // commit round trip with nothing outstanding
        mma_commit(&bar);
        mbar_wait(&bar, 1);
        unsigned long long t3 = clock64();
        out[blockIdx.x * 4 + 0] = t1 - t0;
        out[blockIdx.x * 4 + 1] = t2 - t0;
        out[blockIdx.x * 4 + 2] = t3 - t2;
    }
    __syncthreads();
    // tcgen05.ld bandwidth: 4 warps, each 64 x (ld.x32 + wait)
    float v[32];
    float acc = 0.f;
    unsigned long long t4 = clock64();
    for (int i = 0; i < 64; ++i) {
        tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + (i & 7) * 32, v);
        tmem_wait_ld();
        acc += v[i & 31];
    }
    unsigned long long t5 = clock64();
    for (int i = 0; i < 64; ++i) {
        tmem_st32(tm + ((uint32_t)(warp * 32) << 16) + (i & 7) * 32, v);
        tmem_wait_st();
    }
    unsigned long long t6 = clock64();
    // pipelined loads: 8 ld then one wait
    for (int i = 0; i < 8; ++i) {
        float w[32];
        tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + i * 32, w);
        acc += w[3];
    }
    tmem_wait_ld();
    unsigned long long t7 = clock64();
    if (threadIdx.x == 0) {
        out[blockIdx.x * 4 + 3] = ((t5 - t4) << 32) | (t6 - t5);
        out[gridDim.x * 4 + blockIdx.x] = t7 - t6;
    }
    if (acc == 123.f) out[0] = 0;
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, 512);
}

int main()
{
    unsigned long long *d;
    cudaMalloc(&d, 1 << 20);
    cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
    for (int N : {64, 128, 256}) {
        for (int n : {1, 4, 16, 64, -1, -4, -16, -64}) {
            k_mma<<<148, 128, 66 * 1024 + 1024>>>(d, n, N);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            unsigned long long h[4 * 148 + 148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            printf("M=128 N=%3d K=16 x%2d: issue %6llu cyc, issue+complete %6llu cyc (ideal %d), empty commit rt %llu; "
                   "ld.x32+wait %.1f cyc, st.x32+wait %.1f cyc, 8 ld pipelined %llu cyc\n",
                   N, n, h[0], h[1], (n < 0 ? -n : n) * N / 2, h[2], (h[3] >> 32) / 64.0, (h[3] & 0xffffffff) / 64.0, h[4 * 148]);
        }
    }
    return 0;
}
