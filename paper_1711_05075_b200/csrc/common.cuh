// common.cuh -- small shared helpers of libballcorr (device + host).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define BC_DEV __device__ __forceinline__

struct cf {
    float x, y;
};

BC_DEV float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
BC_DEV float2 cmulc(float2 a, float2 b) { return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y); } // a * conj(b)
BC_DEV float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
BC_DEV float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
BC_DEV float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
BC_DEV float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

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
