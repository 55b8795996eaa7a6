// common.cuh -- small shared helpers of libballcorr (device + host).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define BC_DEV __device__ __forceinline__

struct cf {
    float x, y;
};

// Complex arithmetic on sm_100's packed fp32x2 pipe (FADD2 / FMUL2 / FFMA2: one issue slot
// for both components; operand swaps, lane broadcasts and the negations below are encoded as
// instruction modifiers).  Per component the rounding is that of the scalar fadd / fmul / fma.
BC_DEV float2 f2(float x) { return make_float2(x, x); }
BC_DEV float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
BC_DEV float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
// a b = a.x (b.x, b.y) - a.y (b.y, -b.x)
BC_DEV float2 cmul(float2 a, float2 b) { return __ffma2_rn(f2(-a.y), make_float2(b.y, -b.x), __fmul2_rn(f2(a.x), b)); }
// a conj(b) = a.x (b.x, -b.y) + a.y (b.y, b.x)
BC_DEV float2 cmulc(float2 a, float2 b) { return __ffma2_rn(f2(a.x), make_float2(b.x, -b.y), __fmul2_rn(f2(a.y), make_float2(b.y, b.x))); }
BC_DEV float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
BC_DEV float2 cscale(float2 a, float s) { return __fmul2_rn(a, f2(s)); }
// a + b c (complex)
BC_DEV float2 cfma(float2 b, float2 c, float2 a) { return __ffma2_rn(f2(-b.y), make_float2(c.y, -c.x), __ffma2_rn(f2(b.x), c, a)); }

// e^{2 pi i num/den} for integers (argument reduced exactly before the float division)
BC_DEV float2 expi_frac(long long num, long long den)
{
    long long m = num % den;
    if (m < 0) m += den;
    float s, c;
    sincospif(2.0f * (float)m / (float)den, &s, &c);
    return make_float2(c, s);
}

// Order-preserving map float -> uint32 (monotone increasing).  -0 is canonicalised to +0.
BC_DEV uint32_t float_order_bits(float v)
{
    v = v + 0.0f;
    uint32_t u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
BC_DEV float float_from_order_bits(uint32_t o)
{
    uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(u);
}
