// Microbenchmark (B200): TMA 3-D box load latency (128 rows x 64 bf16 = 16 KB, 128B swizzle, the
// fused kernel's K/V tile) from L2-resident and from HBM-resident data, with `depth` loads in
// flight per CTA, 148 CTAs.  Prints median issue -> mbarrier-complete latency in cycles.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap tm, int nbh, int ntile, int depth,
                                           int iters, int stride_bh, unsigned long long *out)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[8];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    unsigned long long t_issue[8];
    unsigned long long tot = 0;
    int n = 0;
    uint32_t ph[8] = {0};
    int it = 0;
    for (int i = 0; i < depth && it < iters; ++i, ++it) {
        const int x = blockIdx.x * 7919 + it * 104729;
        t_issue[i] = clock64();
        mbar_expect_tx(&bar[i], 16384);
        tma_load_3d(smem + i * 16384, &tm, &bar[i], 0, (x % ntile) * 128, ((x / ntile) * stride_bh) % nbh);
    }
    for (int i = 0; it < iters + depth; ++it, i = (i + 1) % depth) {
        mbar_wait(&bar[i], ph[i]);
        ph[i] ^= 1;
        const unsigned long long t = clock64();
        tot += t - t_issue[i];
        ++n;
        if (it < iters) {
            const int x = blockIdx.x * 7919 + it * 104729;
            t_issue[i] = clock64();
            mbar_expect_tx(&bar[i], 16384);
            tma_load_3d(smem + i * 16384, &tm, &bar[i], 0, (x % ntile) * 128, ((x / ntile) * stride_bh) % nbh);
        }
    }
    out[blockIdx.x] = tot / n;
}

int main()
{
    const int N = 4096, d = 64;
    for (int nbh : {4, 1024}) {   // 4 heads = 4 MB (L2-resident); 1024 heads = 1 GB (HBM)
        size_t bytes = (size_t)nbh * N * d * 2;
        void *buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 0, bytes);
        CUtensorMap tm;
        make_map(&tm, buf, nbh, N, d);
        unsigned long long *out;
        cudaMalloc(&out, 148 * 8);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 1024);
        for (int grid : {16, 74, 148})
        for (int depth : {1, 2, 4, 8}) {
            k<<<grid, 32, 8 * 16384 + 1024>>>(tm, nbh, N / 128, depth, 200, 1, out);   // warm
            k<<<grid, 32, 8 * 16384 + 1024>>>(tm, nbh, N / 128, depth, 2000, 1, out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            std::vector<unsigned long long> h(grid);
            cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
            std::sort(h.begin(), h.end());
            printf("%s grid=%3d depth=%d: median per-load latency %llu cyc (min %llu max %llu); %.1f B/cyc/SM\n",
                   nbh == 4 ? "L2 " : "HBM", grid, depth, h[grid / 2], h[0], h[grid - 1], 16384.0 * depth / h[grid / 2]);
        }
        cudaFree(buf);
        cudaFree(out);
    }
    return 0;
}
