// Microbenchmark (B200): is per-SM TMA load throughput limited per issuing thread?  W warps per
// CTA each keep `depth` 16 KB box loads (3-D map, 128B swizzle) in flight; 148 CTAs, L2-resident.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ CUtensorMap tm, int depth, int iters,
                                            unsigned long long *out)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[8][4];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[w][i], 1); fence_mbar_init(); }
    __syncthreads();
    if ((threadIdx.x & 31) != 0) return;
    uint32_t ph[4] = {0};
    uint8_t *mys = smem;   // all warps share the destination buffers (bandwidth test only)
    const unsigned long long t0 = clock64();
    int it = 0;
    auto issue = [&](int i) {
        const int x = (blockIdx.x * 7919 + w * 313 + it * 104729) % 128;
        mbar_expect_tx(&bar[w][i], 16384);
        tma_load_3d(mys + i * 16384, &tm, &bar[w][i], 0, (x % 32) * 128, x / 32);
    };
    for (int i = 0; i < depth; ++i, ++it) issue(i);
    for (int i = 0; it < iters + depth; ++it, i = (i + 1) % depth) {
        mbar_wait(&bar[w][i], ph[i]);
        ph[i] ^= 1;
        if (it < iters) issue(i);
    }
    if (w == 0) out[blockIdx.x] = clock64() - t0;
}

int main()
{
    const int N = 4096, d = 64, nbh = 4;
    void *buf;
    cudaMalloc(&buf, (size_t)nbh * N * d * 2);
    cudaMemset(buf, 0, (size_t)nbh * N * d * 2);
    unsigned long long *out;
    cudaMalloc(&out, 148 * 8);
    CUtensorMap tm;
    make_map(&tm, buf, nbh, N, d);
    const int smem = 16384 * 4 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int warps : {1, 2, 4, 8})
        for (int depth : {1, 2, 4}) {
            const int iters = 1000;
            k<<<148, 32 * warps, smem>>>(tm, depth, 100, out);
            k<<<148, 32 * warps, smem>>>(tm, depth, iters, out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            std::vector<unsigned long long> h(148);
            cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
            std::sort(h.begin(), h.end());
            printf("warps=%d depth=%d: %.1f B/cyc/SM\n", warps, depth, (double)iters * warps * 16384 / h[74]);
        }
    return 0;
}
