// Microbenchmarks (B200): MUFU.EX2 throughput per SM, FFMA2 throughput.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ex2_tp(float *out, int iters, float seed)
{
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma_tp(float *out, int iters, float seed)
{
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 0.999f, 0.001f);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *out;
    cudaMalloc(&out, 1 << 26);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int warps = 1; warps <= 16; warps *= 2) {
        int iters = 20000;
        ex2_tp<<<sms, 32 * warps>>>(out, 10, 1.f);
        cudaEventRecord(a);
        ex2_tp<<<sms, 32 * warps>>>(out, iters, 1.f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = (double)sms * 32 * warps * iters * 8;
        printf("ex2  warps/SM=%2d: %.1f Gop/s = %.2f per clk per SM (clk %.0f MHz nominal)\n", warps, ops / ms / 1e6,
               ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
        ffma_tp<<<sms, 32 * warps>>>(out, 10, 1.f);
        cudaEventRecord(a);
        ffma_tp<<<sms, 32 * warps>>>(out, iters, 1.f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("ffma warps/SM=%2d: %.2f per clk per SM\n", warps, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    return 0;
}
