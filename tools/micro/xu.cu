// Microbenchmark (B200): which pipe F2FP (cvt.rn.bf16x2.f32) uses -- throughput alone and
// mixed with MUFU.EX2 -- plus FFMA2 / FADD2 throughput.  ops per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float *out, int iters, float seed)
{
    float a[8];
    uint32_t c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = seed + threadIdx.x * 1e-3f + i; c[i] = i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            if (MODE == 1) {   // F2FP only
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                c[i] ^= r;
                asm volatile("" : "+f"(a[i]) : "r"(c[i]));
            }
            if (MODE == 2) {   // 1 MUFU + 1 F2FP
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 3) & 7]));
                c[i] ^= r;
            }
            if (MODE == 3) {   // FFMA2
                uint64_t v;
                asm volatile("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(a[i]), "f"(a[i]));
                asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v));
                float lo, hi;
                asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
                a[i] = lo + hi;
            }
            if (MODE == 4) {   // FFMA2 chain (no unpack)
                uint64_t v = (uint64_t)c[i];
                asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v));
                asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v));
                c[i] = (uint32_t)v;
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i] + c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char *name, int per_iter, int sms, int warps)
{
    float *out;
    cudaMalloc(&out, 1 << 26);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int iters = 20000;
    k<MODE><<<sms, 32 * warps>>>(out, 10, 1.f);
    cudaEventRecord(a);
    k<MODE><<<sms, 32 * warps>>>(out, iters, 1.f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ops = (double)sms * 32 * warps * iters * 8 * per_iter;
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-22s warps=%2d  %.2f ops/clk/SM (at %d MHz nominal)\n", name, warps, ops / cyc / sms, clk / 1000);
    cudaFree(out);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {8, 16}) {
        run<0>("MUFU.EX2", 1, sms, w);
        run<1>("F2FP (pack)", 1, sms, w);
        run<2>("EX2+F2FP (pairs)", 1, sms, w);
        run<3>("FFMA2 (+mov)", 1, sms, w);
        run<4>("FFMA2 x2", 2, sms, w);
    }
    return 0;
}
