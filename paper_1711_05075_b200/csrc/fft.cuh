// fft.cuh -- block-cooperative mixed-radix Stockham FFT in shared memory.
//
// The paper's FFT stages ("cuFFT(W)"; Appendix C,
// DFT as a Riemann sum, O(n log n)) are hand-written here so that they can be
// fused with the spreading, deconvolution, spectral product and reductions
// around them.  A block transforms NL lines of length L held in shared memory
// as buf[n * ld + line] (line fastest, ld >= NL for bank padding).
//
// Stage s with radix R (Govindaraju et al. Stockham autosort, natural order):
//   v[r] = a[j + r L/R] * w^{r (j mod Ns) L/(Ns R)},  V = DFT_R(v),
//   b[(j/Ns) Ns R + (j mod Ns) + r Ns] = V[r],  Ns *= R.
// Twiddles come from a per-block table tw[m] = exp(sign 2 pi i m / L).
#pragma once

#include "common.cuh"

#define BC_FFT_MAX_STAGES 12

struct FftPlan {
    int L;
    int nst;
    int radix[BC_FFT_MAX_STAGES];
};

// ---------------------------------------------------------------- small DFTs
BC_DEV float2 mul_i(float2 a, float sign) { return make_float2(-sign * a.y, sign * a.x); } // a * (sign i)

template <int R>
struct SmallDft;

template <>
struct SmallDft<2> {
    static BC_DEV void run(float2 *v, float) {
        float2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    }
};

template <>
struct SmallDft<3> {
    static BC_DEV void run(float2 *v, float sign) {
        const float s3 = 0.86602540378443864676f;
        float2 t1 = cadd(v[1], v[2]);
        float2 t2 = make_float2(v[0].x - 0.5f * t1.x, v[0].y - 0.5f * t1.y);
        float2 d = csub(v[1], v[2]);
        float2 t3 = mul_i(cscale(d, s3), sign);
        v[0] = cadd(v[0], t1);
        v[1] = cadd(t2, t3);
        v[2] = csub(t2, t3);
    }
};

template <>
struct SmallDft<4> {
    static BC_DEV void run(float2 *v, float sign) {
        float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
        float2 s13 = cadd(v[1], v[3]), d13 = mul_i(csub(v[1], v[3]), sign);
        v[0] = cadd(s02, s13);
        v[2] = csub(s02, s13);
        v[1] = cadd(d02, d13);
        v[3] = csub(d02, d13);
    }
};

template <>
struct SmallDft<5> {
    static BC_DEV void run(float2 *v, float sign) {
        // X_q = sum_r v_r w^{rq}, w = exp(sign 2 pi i / 5)
        const float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
        const float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
        float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
        float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
        float2 x0 = v[0];
        float2 r1 = make_float2(x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y);
        float2 r2 = make_float2(x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y);
        float2 i1 = mul_i(make_float2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y), sign);
        float2 i2 = mul_i(make_float2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y), sign);
        v[0] = make_float2(x0.x + a1.x + a2.x, x0.y + a1.y + a2.y);
        v[1] = cadd(r1, i1);
        v[4] = csub(r1, i1);
        v[2] = cadd(r2, i2);
        v[3] = csub(r2, i2);
    }
};

template <>
struct SmallDft<8> {
    static BC_DEV void run(float2 *v, float sign) {
        // radix-2 split into even/odd radix-4 DFTs
        float2 e[4] = {v[0], v[2], v[4], v[6]};
        float2 o[4] = {v[1], v[3], v[5], v[7]};
        SmallDft<4>::run(e, sign);
        SmallDft<4>::run(o, sign);
        const float r = 0.70710678118654752440f;
        // twiddles w8^q = exp(sign 2 pi i q / 8)
        float2 t1 = make_float2(r * (o[1].x - sign * o[1].y), r * (o[1].y + sign * o[1].x));
        float2 t2 = mul_i(o[2], sign);
        float2 t3 = make_float2(r * (-o[3].x - sign * o[3].y), r * (-o[3].y + sign * o[3].x));
        v[0] = cadd(e[0], o[0]);
        v[4] = csub(e[0], o[0]);
        v[1] = cadd(e[1], t1);
        v[5] = csub(e[1], t1);
        v[2] = cadd(e[2], t2);
        v[6] = csub(e[2], t2);
        v[3] = cadd(e[3], t3);
        v[7] = csub(e[3], t3);
    }
};

template <int R>
BC_DEV void fft_stage(const float2 *__restrict__ a, float2 *__restrict__ b, const float2 *__restrict__ tw,
                      int L, int Ns, int NL, int ld, float sign)
{
    const int LR = L / R;
    const int nitems = NL * LR;
    const int twstride = L / (Ns * R);
    for (int it = threadIdx.x; it < nitems; it += blockDim.x) {
        const int line = it % NL, j = it / NL;
        const int jm = j % Ns;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
            float2 x = a[(j + r * LR) * ld + line];
            v[r] = (r == 0) ? x : cmul(x, tw[r * jm * twstride]);
        }
        SmallDft<R>::run(v, sign);
        const int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
        for (int r = 0; r < R; r++) b[(idxD + r * Ns) * ld + line] = v[r];
    }
}

// Fill tw[m] = exp(sign 2 pi i m / L), m in [0, L).  Caller syncs.
BC_DEV void fft_twiddles(float2 *tw, int L, float sign)
{
    for (int m = threadIdx.x; m < L; m += blockDim.x) {
        float s, c;
        sincospif(2.0f * (float)m / (float)L, &s, &c);
        tw[m] = make_float2(c, sign * s);
    }
}

// Transform NL lines in `a` (scratch `b` of the same size).  Returns the buffer
// that holds the result.  Must be called by all threads of the block; the
// input must be complete (caller syncs before).  Ends with a __syncthreads.
BC_DEV float2 *block_fft(float2 *a, float2 *b, const float2 *tw, const FftPlan &pl, int NL, int ld, float sign)
{
    int Ns = 1;
    for (int s = 0; s < pl.nst; s++) {
        const int R = pl.radix[s];
        switch (R) {
        case 2: fft_stage<2>(a, b, tw, pl.L, Ns, NL, ld, sign); break;
        case 3: fft_stage<3>(a, b, tw, pl.L, Ns, NL, ld, sign); break;
        case 4: fft_stage<4>(a, b, tw, pl.L, Ns, NL, ld, sign); break;
        case 5: fft_stage<5>(a, b, tw, pl.L, Ns, NL, ld, sign); break;
        default: fft_stage<8>(a, b, tw, pl.L, Ns, NL, ld, sign); break;
        }
        __syncthreads();
        float2 *t = a;
        a = b;
        b = t;
        Ns *= R;
    }
    return a;
}
