// Microbenchmark (B200): mbarrier hand-off latency between two warps of a CTA (arrive -> try_wait
// wake-up), plain arrive vs tcgen05.commit (empty MMA group) on the return leg.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_16847_b200/csrc/sm100.cuh"
using namespace splat::sm100;

__global__ void __launch_bounds__(128, 1) k(int iters, int mode, unsigned long long *out)
{
    __shared__ uint64_t b1, b2;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { mbar_init(&b1, 1); mbar_init(&b2, 1); fence_mbar_init(); }
    if (warp == 1) tmem_alloc(&slot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (lane == 0) mbar_arrive(&b1);
            mbar_wait(&b2, i & 1);
        }
        if (lane == 0) out[blockIdx.x] = (clock64() - t0) / iters;
    } else if (warp == 1) {
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&b1, i & 1);
            if (mode == 0) {
                if (lane == 0) mbar_arrive(&b2);
            } else {
                if (elect_one()) mma_commit(&b2);
                __syncwarp();
            }
        }
    }
    __syncthreads();
    if (warp == 1) tmem_dealloc(slot, 32);
}

int main()
{
    unsigned long long *d;
    cudaMalloc(&d, 148 * 8);
    for (int mode : {0, 1}) {
        k<<<148, 128>>>(1000, mode, d);
        cudaDeviceSynchronize();
        unsigned long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("round trip (%s on return leg): %llu cycles\n", mode ? "tcgen05.commit" : "mbarrier.arrive", h);
    }
    return 0;
}
