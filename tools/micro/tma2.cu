// Microbenchmark (B200): per-SM TMA load throughput vs tensor-map shape (L2-resident source).
// Variants: 3-D [BH,N,64] box 64x128x1 (the fused kernel's), 2-D [BH*N,64] box 64x128 and
// 64x256, swizzle 128B vs none, L2 promotion 256B vs none.  148 CTAs, depth 4 loads in flight.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}

__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap tm, int dims, int rows_total, int box_rows,
                                           int depth, int iters, unsigned long long *out)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[8];
    if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
    __syncwarp();
    if (threadIdx.x != 0) return;
    const uint32_t bytes = box_rows * 128;
    uint32_t ph[8] = {0};
    const unsigned long long t0 = clock64();
    int it = 0;
    auto issue = [&](int i) {
        const int x = (blockIdx.x * 7919 + it * 104729) % (rows_total / box_rows);
        mbar_expect_tx(&bar[i], bytes);
        if (dims == 3) tma_load_3d(smem + i * 32768, &tm, &bar[i], 0, (x % 32) * 128, x / 32);
        else tma_load_2d(smem + i * 32768, &tm, &bar[i], 0, x * box_rows);
    };
    for (int i = 0; i < depth; ++i, ++it) issue(i);
    for (int i = 0; it < iters + depth; ++it, i = (i + 1) % depth) {
        mbar_wait(&bar[i], ph[i]);
        ph[i] ^= 1;
        if (it < iters) issue(i);
    }
    out[blockIdx.x] = clock64() - t0;
}

int main()
{
    const int N = 4096, d = 64, nbh = 4;
    size_t bytes = (size_t)nbh * N * d * 2;
    void *buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    unsigned long long *out;
    cudaMalloc(&out, 148 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32768 / 2 + 1024);
    EncodeTiledFn enc = get_encode();
    struct V { const char *name; int dims, box_rows; CUtensorMapSwizzle sw; CUtensorMapL2promotion l2; };
    V vs[] = {{"3d box64x128 sw128 L2_256", 3, 128, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B},
              {"3d box64x128 sw128 L2none", 3, 128, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE},
              {"2d box64x128 sw128 L2_256", 2, 128, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B},
              {"2d box64x256 sw128 L2_256", 2, 256, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B},
              {"2d box64x128 swNONE L2_256", 2, 128, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B},
              {"2d box64x64 sw128 L2_256", 2, 64, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B}};
    for (auto &v : vs) {
        CUtensorMap tm;
        CUresult r;
        if (v.dims == 3) {
            cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)N, (cuuint64_t)nbh};
            cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)N * d * 2};
            cuuint32_t box[3] = {64, (cuuint32_t)v.box_rows, 1}, es[3] = {1, 1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, v.sw, v.l2,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)N * nbh};
            cuuint64_t strides[1] = {(cuuint64_t)d * 2};
            cuuint32_t box[2] = {64, (cuuint32_t)v.box_rows}, es[2] = {1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, v.sw, v.l2,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", v.name, (int)r); continue; }
        for (int depth : {2, 4}) {
            const int iters = 2000;
            k<<<148, 32, 8 * 32768 / 2 + 1024>>>(tm, v.dims, N * nbh, v.box_rows, depth, 200, out);
            k<<<148, 32, 8 * 32768 / 2 + 1024>>>(tm, v.dims, N * nbh, v.box_rows, depth, iters, out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            std::vector<unsigned long long> h(148);
            cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
            std::sort(h.begin(), h.end());
            printf("%-28s depth=%d: %.1f B/cyc/SM\n", v.name, depth, (double)iters * v.box_rows * 128 / h[74]);
        }
    }
    return 0;
}
