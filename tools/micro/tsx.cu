// Microbenchmark (B200, sm_100a): tcgen05.mma throughput of the fused kernel's MMA shapes, issued the
// way the kernel issues them (whole warp converged, elect.sync, warp-uniform descriptors, groups of
// back-to-back MMAs), optionally while 8 other warps run tcgen05.ld / tcgen05.st on their own TMEM
// columns like the softmax warpgroups.
//   mode 0: S = Q K^T      SS, M = 128, N = 128, K-major A and B         (4 MMAs per group, K = 64)
//   mode 1: O += P V       TS, M = 128, N = 64,  A (P) in TMEM, B MN-major (8 MMAs per group, K = 128)
//   mode 2: O += P V       SS, M = 128, N = 64,  A (P) in SMEM K-major, B MN-major
//   mode 3: O += P V       TS, M = 128, N = 128 (d = 128)
//   mode 4: O^T += V^T P^T SS, M = 64?  (not valid for cta_group::1 kind::f16 at M=64 with N=128? skipped)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

__global__ void __launch_bounds__(384, 1) k(unsigned long long *out, int groups, int mode, int load)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw;
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    for (int i = threadIdx.x; i < 98304 / 4; i += 384) reinterpret_cast<uint32_t *>(smem)[i] = 0x3c003c00u;
    fence_proxy_async_smem();
    __syncthreads();
    if (warp == 1) {
        const uint32_t tmu = __shfl_sync(0xffffffffu, tm, 0);
        const uint32_t s = smem_u32(smem);
        constexpr uint32_t idS = idesc_bf16(128, 128, false), idO = idesc_bf16(128, 64, true);
        constexpr uint32_t idO2 = idesc_bf16(128, 128, true);
        unsigned long long w0 = clock64();
        while (clock64() - w0 < 20000) {}
        __syncwarp();
        unsigned long long t0 = clock64();
        for (int g = 0; g < groups; ++g) {
            if (elect_one()) {
                if (mode == 0) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_bf16_ss(tmu, sdesc_sw128(s + kk * 32, 16, 1024), sdesc_sw128(s + 32768 + kk * 32, 16, 1024),
                                    idS, 1u);
                } else if (mode == 1) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16_ts(tmu + 256, tmu + 384 + kk * 8, sdesc_sw128(s + 32768 + kk * 2048, 16384, 1024), idO, 1u);
                } else if (mode == 2) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16_ss(tmu + 256, sdesc_sw128(s + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                    sdesc_sw128(s + 65536 + kk * 2048, 16384, 1024), idO, 1u);
                } else {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16_ts(tmu + 256, tmu + 128 + kk * 8, sdesc_sw128(s + 32768 + kk * 2048, 16384, 1024), idO2, 1u);
                }
            }
            __syncwarp();
        }
        unsigned long long t1 = clock64();
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        unsigned long long t2 = clock64();
        if (lane == 0) {
            out[blockIdx.x * 2 + 0] = t1 - t0;
            out[blockIdx.x * 2 + 1] = t2 - t0;
            stop = 1;
        }
        __syncwarp();
    } else if (warp >= 4 && load) {
        const int quad = warp & 3, g = (warp - 4) >> 2;
        const uint32_t lo = (uint32_t)(quad * 32) << 16;
        // columns the MMA does not touch in modes 1-2 (S of an idle group); mode 0 / 3 share
        const uint32_t sb = tm + lo + 128 * g;
        float v[128];
        for (int x = 0; x < 128; ++x) v[x] = 0.f;
        int it = 0;
        while (!stop && it < 100000) {
            tmem_ld32(sb, v);
            tmem_ld32(sb + 32, v + 32);
            tmem_ld32(sb + 64, v + 64);
            tmem_ld32(sb + 96, v + 96);
            tmem_wait_ld();
            float acc = 0.f;
            for (int x = 0; x < 128; ++x) acc += v[x];
            v[0] = acc;
            tmem_st32(sb, v);
            tmem_st32(sb + 32, v + 32);
            tmem_wait_st();
            ++it;
        }
    }
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, 512);
}

int main()
{
    unsigned long long *d;
    cudaMalloc(&d, 1 << 20);
    const int sm = 98304;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    const char *names[] = {"SS QK^T  M128 N128 (x4/group)", "TS P.V   M128 N64  (x8/group)", "SS P.V   M128 N64  (x8/group)",
                           "TS P.V   M128 N128 (x8/group)"};
    const int per[] = {4, 8, 8, 8};
    const double flop[] = {2.0 * 128 * 128 * 16, 2.0 * 128 * 64 * 16, 2.0 * 128 * 64 * 16, 2.0 * 128 * 128 * 16};
    for (int mode = 0; mode < 4; ++mode)
        for (int load : {0, 1})
            for (int groups : {8, 64}) {
                k<<<148, 384, sm>>>(d, groups, mode, load);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                unsigned long long h[2];
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                const double n = (double)groups * per[mode];
                printf("%s load=%d n=%4d: issue %6llu done %7llu cyc = %6.1f cyc/MMA = %6.0f FLOP/clk/SM\n", names[mode], load,
                       (int)n, h[0], h[1], h[1] / n, flop[mode] * n / h[1]);
            }
    return 0;
}
