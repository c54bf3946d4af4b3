// Microbenchmark (B200, sm_100a): does TMEM load/store traffic from other warps slow tcgen05.mma?
// One CTA per SM, 384 threads.  Warp 1 issues n back-to-back MMAs of one shape (SS: S = Q K^T,
// M = N = 128; TS: O += P V, M = 128, N = 64, A from TMEM, B MN-major) and times issue -> commit
// completion.  With load = 1 the 8 warps 4..11 meanwhile loop tcgen05.ld (128 columns, 32x32b.x32)
// + wait + tcgen05.st (64 columns) on their own TMEM columns, like the fused kernel's softmax.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

__global__ void __launch_bounds__(384, 1) k(unsigned long long *out, int n, int ts, int load, int nst)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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
    for (int i = threadIdx.x; i < 65536 / 4; i += 384) reinterpret_cast<uint32_t *>(smem)[i] = 0x3c003c00u;
    fence_proxy_async_smem();
    __syncthreads();
    if (warp == 1) {
        if (lane == 0) {
            const uint32_t s = smem_u32(smem);
            const uint32_t idS = idesc_bf16(128, 128, false), idO = idesc_bf16(128, 64, true);
            // warm-up pause so the load warps are running
            unsigned long long w0 = clock64();
            while (clock64() - w0 < 20000) {}
            unsigned long long t0 = clock64();
            for (int i = 0; i < n; ++i) {
                if (ts)
                    mma_bf16_ts(tm + 256, tm + 384 + (i & 7) * 8, sdesc_sw128(s + 32768 + (i & 7) * 2048, 16384, 1024), idO, 1);
                else
                    mma_bf16_ss(tm + 0, sdesc_sw128(s + (i & 3) * 32, 16, 1024), sdesc_sw128(s + 32768 + (i & 3) * 32, 16, 1024), idS, 1);
            }
            unsigned long long t1 = clock64();
            mma_commit(&bar);
            mbar_wait(&bar, 0);
            unsigned long long t2 = clock64();
            out[blockIdx.x * 2 + 0] = t1 - t0;
            out[blockIdx.x * 2 + 1] = t2 - t0;
            stop = 1;
        }
        __syncwarp();
    } else if (warp >= 4 && load) {
        const int quad = warp & 3, g = (warp - 4) >> 2;
        const uint32_t lo = (uint32_t)(quad * 32) << 16;
        // group g: loads S columns [128 g, +128) (disjoint from the MMA's columns when ts), stores P
        const uint32_t sb = tm + lo + (ts ? 128 * g : 256 + 64 * g);
        float v[128];
        for (int x = 0; x < 128; ++x) v[x] = 0.f;
        int it = 0;
        while (!stop && it < 100000) {
            tmem_ld32(sb, v);
            tmem_ld32(sb + 32, v + 32);
            tmem_ld32(sb + 64, v + 64);
            tmem_ld32(sb + 96, v + 96);
            tmem_wait_ld();
            if (nst) {
                float acc = 0.f;
                for (int x = 0; x < 128; ++x) acc += v[x];
                v[0] = acc;
                tmem_st32(sb, v);
                tmem_st32(sb + 32, v + 32);
                tmem_wait_st();
            }
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
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
    for (int ts : {0, 1})
        for (int load : {0, 1})
            for (int nst : {0, 1}) {
                if (!load && nst) continue;
                for (int n : {64, 256}) {
                    k<<<148, 384, 66 * 1024 + 1024>>>(d, n, ts, load, nst);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                    unsigned long long h[2];
                    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                    printf("%s %s load=%d st=%d x%3d: issue %6llu done %7llu = %.1f cyc/MMA\n", ts ? "TS N=64 " : "SS N=128",
                           ts ? "(O+=PV)" : "(S=QK) ", load, nst, n, h[0], h[1], (double)h[1] / n);
                }
            }
    return 0;
}
