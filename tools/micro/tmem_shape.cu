// Microbenchmark / probe (B200): the register layout of tcgen05.ld.16x64b and 16x256b.  Warp 0 writes
// lane l, column c = 1000 l + c with 32x32b.x16 (thread = lane), then reads lanes 0-15 (and 16-31)
// with the 16-lane shapes and prints which (lane, column) each thread's registers hold.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tmem_shape.cu -o tmem_shape && ./tmem_shape
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k(int *out)
{
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    if (warp == 0) {
        uint32_t v[16];
        for (int c = 0; c < 16; ++c) v[c] = 1000 * lane + c;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(tm), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                     "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
        uint32_t a[2], b[4];
        asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0,%1}, [%2];" : "=r"(a[0]), "=r"(a[1]) : "r"(tm));
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]) : "r"(tm));
        uint32_t c2[2];
        asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0,%1}, [%2];" : "=r"(c2[0]), "=r"(c2[1]) : "r"(tm + (16u << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        out[lane * 8 + 0] = a[0]; out[lane * 8 + 1] = a[1];
        for (int i = 0; i < 4; ++i) out[lane * 8 + 2 + i] = b[i];
        out[lane * 8 + 6] = c2[0]; out[lane * 8 + 7] = c2[1];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main()
{
    int *d, h[256];
    cudaMalloc(&d, sizeof(h));
    k<<<1, 128>>>(d);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("thread: 16x64b.x2 (r0 r1) | 16x256b.x1 (r0..r3) | 16x64b.x2 at lane 16 (r0 r1)   [value = 1000 lane + col]\n");
    for (int t = 0; t < 32; ++t)
        printf("%2d: %5d %5d | %5d %5d %5d %5d | %5d %5d\n", t, h[t * 8], h[t * 8 + 1], h[t * 8 + 2], h[t * 8 + 3],
               h[t * 8 + 4], h[t * 8 + 5], h[t * 8 + 6], h[t * 8 + 7]);
    return 0;
}
