// softmax_math.cuh -- register-level softmax arithmetic shared by the fused kernels:
// 3-input max, packed fp32x2 FMA/add (FFMA2 / FADD2), exp2 on MUFU or emulated on the FMA pipe,
// bf16 packing and the per-chunk fast-index mask (reading A-7 of DESIGN.md).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

namespace splat {
namespace smx {

using sm100::ex2;
using sm100::pack_bf16;

__device__ __forceinline__ float fmax3(float a, float b, float c)
{
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

__device__ __forceinline__ uint64_t pack2(float lo, float hi)
{
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}

__device__ __forceinline__ void unpack2(uint64_t v, float &lo, float &hi)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c)
{
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b)
{
    uint64_t d;
    asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

__device__ __forceinline__ float max32(const float *v)
{
    float a0 = fmax3(v[0], v[1], v[2]), a1 = fmax3(v[3], v[4], v[5]);
    float a2 = fmax3(v[6], v[7], v[8]), a3 = fmax3(v[9], v[10], v[11]);
#pragma unroll
    for (int x = 12; x < 32; x += 8) {
        a0 = fmax3(a0, v[x + 0], v[x + 1]);
        a1 = fmax3(a1, v[x + 2], v[x + 3]);
        a2 = fmax3(a2, v[x + 4], v[x + 5]);
        a3 = fmax3(a3, v[x + 6], v[x + 7]);
    }
    return fmax3(fmax3(a0, a1, a2), a3, -INFINITY);
}

// Number of the 32 exponentials of a chunk evaluated on the FMA pipe instead of MUFU (the MUFU
// does 16 ex2/clk/SM against 8192 bf16 FLOP/clk on the tensor pipe: at d = 64 it is the
// co-bottleneck).  Multiple of 4.
#ifndef SPLAT_NEMU128
#define SPLAT_NEMU128 4       // d = 128 (MUFU has more slack against the tensor pipe there)
#endif
#ifndef SPLAT_NEMU
#define SPLAT_NEMU 12
#endif

__device__ __forceinline__ uint64_t fmax2_clamp(uint64_t z)
{
    float a, b;
    unpack2(z, a, b);
    return pack2(fmaxf(a, -126.f), fmaxf(b, -126.f));
}

// 2^x for a packed pair on the FMA pipe: x = j + f with j = rint(x) (1.5*2^23 magic-number
// rounding), f in [-1/2, 1/2]; 2^f by a degree-3 polynomial (max relative error 7.5e-5, far
// below bf16's 2^-9); the exponent j is added to the bits of 2^f.  x is clamped at -126 so
// masked (-inf) scores give 2^-126 (below any bf16 P that matters; -127 would wrap the
// exponent field of a p just under 1).
__device__ __forceinline__ void exp2_emu2(uint64_t z, float &ra, float &rb)
{
    const uint64_t zc = fmax2_clamp(z);
    const uint64_t t = fadd2(zc, pack2(12582912.f, 12582912.f));
    const uint64_t jf = fadd2(t, pack2(-12582912.f, -12582912.f));
    const uint64_t f = ffma2(jf, pack2(-1.f, -1.f), zc);
    uint64_t p = ffma2(pack2(0.0551716648f, 0.0551716648f), f, pack2(0.2426111251f, 0.2426111251f));
    p = ffma2(p, f, pack2(0.6932609677f, 0.6932609677f));
    p = ffma2(p, f, pack2(0.9999280572f, 0.9999280572f));
    float pa, pb, ta, tb;
    unpack2(p, pa, pb);
    unpack2(t, ta, tb);
    ra = __int_as_float(__float_as_int(pa) + (__float_as_int(ta) << 23));
    rb = __int_as_float(__float_as_int(pb) + (__float_as_int(tb) << 23));
}

// p = exp2(s*c - m) for 32 scores -> 16 packed bf16 pairs; row-sum partials in acc0/acc1.
template <int NEMU = SPLAT_NEMU>
__device__ __forceinline__ void exp32(const float *v, uint64_t cc, uint64_t mm, uint64_t &acc0, uint64_t &acc1,
                                      uint32_t *pw)
{
#pragma unroll
    for (int x = 0; x < 32; x += 4) {
        const uint64_t z0 = ffma2(pack2(v[x], v[x + 1]), cc, mm);
        const uint64_t z1 = ffma2(pack2(v[x + 2], v[x + 3]), cc, mm);
        float a, b, c, d;
        if (x < NEMU) {
            exp2_emu2(z0, a, b);
            exp2_emu2(z1, c, d);
        } else {
            unpack2(z0, a, b);
            unpack2(z1, c, d);
            a = ex2(a); b = ex2(b); c = ex2(c); d = ex2(d);
        }
#ifndef SPLAT_X_NOSUM
        acc0 = fadd2(acc0, pack2(a, b));
        acc1 = fadd2(acc1, pack2(c, d));
#endif
        pw[x / 2] = pack_bf16(a, b);
        pw[x / 2 + 1] = pack_bf16(c, d);
    }
}

__device__ __forceinline__ void apply_mask(float *v, uint32_t m)
{
#pragma unroll
    for (int x = 0; x < 32; ++x) v[x] = ((m >> x) & 1u) ? v[x] : -INFINITY;
}

}  // namespace smx
}  // namespace splat
