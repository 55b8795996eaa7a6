// fft_ct.cuh -- compile-time-sized mixed-radix Stockham FFT over shared memory.
//
// Hand-written replacement of the paper's library FFT stages (PAPER.md L524-L526,
// "FFTW on the CPU and cuFFT(W) on the GPU"; Appendix C) so that every
// transform can be fused with the kernel arithmetic around it.
//
// A block transforms NL lines of length L; each line is owned by TPL consecutive
// threads.  Line l lives in shared memory at buf[l * LS + PAD(idx)], with
// PAD(idx) = idx + idx/16 and LS odd in float2 units (bank spreading).
// Stage with radix R (Stockham autosort, natural-order output):
//     v[r] = a[j + r L/R] * w_L^{r (j mod Ns) L/(Ns R)},  V = DFT_R(v),
//     b[(j / Ns) Ns R + (j mod Ns) + r Ns] = V[r],        Ns *= R.
// Sizes and radix schedules are compile-time, so all index arithmetic is
// strength-reduced; twiddles come from a per-block table tw[m] = exp(-2 pi i m / L).
#pragma once

#include "common.cuh"

namespace fct {

__host__ __device__ constexpr int pad(int idx) { return idx + (idx >> 4); }
__host__ __device__ constexpr int line_stride(int L) { return (pad(L - 1) + 1) | 1; }

// ---------------------------------------------------------------- schedules
template <int L> struct Sched;
#define BC_SCHED(L_, N_, A_, B_, C_, D_) \
    template <> struct Sched<L_> { static constexpr int n = N_; static constexpr int r[4] = {A_, B_, C_, D_}; };
BC_SCHED(16, 1, 16, 1, 1, 1)
BC_SCHED(20, 2, 4, 5, 1, 1)
BC_SCHED(24, 2, 8, 3, 1, 1)
BC_SCHED(32, 2, 16, 2, 1, 1)
BC_SCHED(36, 3, 4, 3, 3, 1)
BC_SCHED(40, 2, 8, 5, 1, 1)
BC_SCHED(48, 2, 16, 3, 1, 1)
BC_SCHED(64, 2, 16, 4, 1, 1)
BC_SCHED(72, 3, 8, 3, 3, 1)
BC_SCHED(80, 2, 16, 5, 1, 1)
BC_SCHED(96, 3, 16, 2, 3, 1)
BC_SCHED(128, 2, 16, 8, 1, 1)
BC_SCHED(144, 3, 16, 3, 3, 1)
BC_SCHED(160, 3, 16, 2, 5, 1)
BC_SCHED(192, 3, 16, 4, 3, 1)
BC_SCHED(240, 3, 16, 5, 3, 1)
BC_SCHED(256, 2, 16, 16, 1, 1)
BC_SCHED(288, 4, 16, 2, 3, 3)
BC_SCHED(320, 3, 16, 4, 5, 1)
BC_SCHED(384, 3, 16, 8, 3, 1)
BC_SCHED(480, 4, 16, 2, 5, 3)
BC_SCHED(512, 3, 8, 8, 8, 1)
BC_SCHED(576, 4, 16, 4, 3, 3)
BC_SCHED(640, 3, 16, 8, 5, 1)
BC_SCHED(768, 3, 16, 16, 3, 1)
BC_SCHED(960, 4, 16, 4, 5, 3)
BC_SCHED(1024, 3, 16, 16, 4, 1)
#undef BC_SCHED

// list used by the host dispatchers
#define BC_FOR_EACH_L(X) X(16) X(20) X(24) X(32) X(36) X(40) X(48) X(64) X(72) X(80) X(96) X(128) X(144) X(160) X(192) X(240) X(256) \
    X(288) X(320) X(384) X(480) X(512) X(576) X(640) X(768) X(960) X(1024)

template <int L, int S>
__host__ __device__ constexpr int ns_before()
{
    int ns = 1;
    for (int s = 0; s < S; s++) ns *= Sched<L>::r[s];
    return ns;
}

// ---------------------------------------------------------------- small DFTs (SIGN = -1 forward, +1 inverse)
template <int SIGN>
BC_DEV float2 mul_si(float2 a) { return SIGN < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x); }

template <int R, int SIGN> struct Dft;

template <int SIGN> struct Dft<2, SIGN> {
    static BC_DEV void run(float2 *v) {
        const float2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    }
};

template <int SIGN> struct Dft<3, SIGN> {
    static BC_DEV void run(float2 *v) {
        const float s3 = 0.86602540378443864676f;
        const float2 t1 = cadd(v[1], v[2]);
        const float2 t2 = make_float2(v[0].x - 0.5f * t1.x, v[0].y - 0.5f * t1.y);
        const float2 t3 = mul_si<SIGN>(cscale(csub(v[1], v[2]), s3));
        v[0] = cadd(v[0], t1);
        v[1] = cadd(t2, t3);
        v[2] = csub(t2, t3);
    }
};

template <int SIGN> struct Dft<4, SIGN> {
    static BC_DEV void run(float2 *v) {
        const float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
        const float2 s13 = cadd(v[1], v[3]), d13 = mul_si<SIGN>(csub(v[1], v[3]));
        v[0] = cadd(s02, s13);
        v[2] = csub(s02, s13);
        v[1] = cadd(d02, d13);
        v[3] = csub(d02, d13);
    }
};

template <int SIGN> struct Dft<5, SIGN> {
    static BC_DEV void run(float2 *v) {
        const float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
        const float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
        const float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
        const float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
        const float2 x0 = v[0];
        const float2 r1 = make_float2(x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y);
        const float2 r2 = make_float2(x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y);
        const float2 i1 = mul_si<SIGN>(make_float2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y));
        const float2 i2 = mul_si<SIGN>(make_float2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y));
        v[0] = make_float2(x0.x + a1.x + a2.x, x0.y + a1.y + a2.y);
        v[1] = cadd(r1, i1);
        v[4] = csub(r1, i1);
        v[2] = cadd(r2, i2);
        v[3] = csub(r2, i2);
    }
};

// w_n^m = exp(SIGN 2 pi i m / n) for the composite radices
template <int N, int SIGN>
BC_DEV float2 wconst(int m)
{
    // cos / sin of 2 pi m / 16 (N = 16) or 2 pi m / 8 (N = 8), m reduced mod N
    const float c16[16] = {1.0f, 0.92387953251128675613f, 0.70710678118654752440f, 0.38268343236508977173f,
                           0.0f, -0.38268343236508977173f, -0.70710678118654752440f, -0.92387953251128675613f,
                           -1.0f, -0.92387953251128675613f, -0.70710678118654752440f, -0.38268343236508977173f,
                           0.0f, 0.38268343236508977173f, 0.70710678118654752440f, 0.92387953251128675613f};
    const int mm = (m * (16 / N)) & 15;
    const float c = c16[mm], s = c16[(mm + 12) & 15];  // sin(x) = cos(x - pi/2)
    return make_float2(c, SIGN * s);
}

template <int SIGN> struct Dft<8, SIGN> {
    static BC_DEV void run(float2 *v) {
        float2 e[4] = {v[0], v[2], v[4], v[6]};
        float2 o[4] = {v[1], v[3], v[5], v[7]};
        Dft<4, SIGN>::run(e);
        Dft<4, SIGN>::run(o);
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const float2 t = q == 0 ? o[0] : cmul(o[q], wconst<8, SIGN>(q));
            v[q] = cadd(e[q], t);
            v[q + 4] = csub(e[q], t);
        }
    }
};

template <int SIGN> struct Dft<16, SIGN> {
    static BC_DEV void run(float2 *v) {
        // 16 = 4 x 4: inner DFT4 over n1 (stride 4), twiddle w16^{n2 k1}, outer DFT4 over n2
        float2 y[4][4];
#pragma unroll
        for (int n2 = 0; n2 < 4; n2++) {
            float2 t[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
            Dft<4, SIGN>::run(t);
#pragma unroll
            for (int k1 = 0; k1 < 4; k1++) y[n2][k1] = (n2 * k1 == 0) ? t[k1] : cmul(t[k1], wconst<16, SIGN>(n2 * k1));
        }
#pragma unroll
        for (int k1 = 0; k1 < 4; k1++) {
            float2 t[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
            Dft<4, SIGN>::run(t);
#pragma unroll
            for (int k2 = 0; k2 < 4; k2++) v[k1 + 4 * k2] = t[k2];
        }
    }
};

// ---------------------------------------------------------------- stages
// FIRST stage reads `src` (optionally multiplying input n by pre[n]); the rest ping-pong a/b.
template <int L, int TPL, int S, int SIGN>
BC_DEV void stage(const float2 *__restrict__ src, float2 *__restrict__ dst, const float2 *__restrict__ tw,
                  const float2 *__restrict__ pre, int tl)
{
    constexpr int R = Sched<L>::r[S];
    constexpr int Ns = ns_before<L, S>();
    constexpr int LR = L / R;
    constexpr int TWS = L / (Ns * R);
#pragma unroll
    for (int j0 = 0; j0 < LR; j0 += TPL) {
        const int j = j0 + tl;
        if ((LR % TPL) != 0 && j >= LR) break;
        const int jm = j % Ns;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
            float2 x = src[pad(j + r * LR)];
            if (S == 0 && pre) x = cmul(x, pre[j + r * LR]);
            if (Ns > 1 && r > 0) {
                const float2 w = tw[r * jm * TWS];
                x = SIGN < 0 ? cmul(x, w) : cmulc(x, w);
            }
            v[r] = x;
        }
        Dft<R, SIGN>::run(v);
        const int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
        for (int r = 0; r < R; r++) dst[pad(idxD + r * Ns)] = v[r];
    }
}

// Terminate when S == Sched<L>::n.  (specialisation through a dispatch helper)
template <int L, int TPL, int S, int SIGN, bool DONE = (S >= Sched<L>::n)>
struct Run;

template <int L, int TPL, int S, int SIGN>
struct Run<L, TPL, S, SIGN, true> {
    static BC_DEV float2 *go(const float2 *, float2 *, float2 *b, const float2 *, const float2 *, int) { return b; }
};

template <int L, int TPL, int S, int SIGN>
struct Run<L, TPL, S, SIGN, false> {
    static BC_DEV float2 *go(const float2 *src, float2 *a, float2 *b, const float2 *tw, const float2 *pre, int tl)
    {
        if (S == 0)
            stage<L, TPL, 0, SIGN>(src, a, tw, pre, tl);
        else
            stage<L, TPL, S, SIGN>(b, a, tw, nullptr, tl);
        __syncthreads();
        return Run<L, TPL, S + 1, SIGN>::go(src, b, a, tw, pre, tl);
    }
};

// Transform the calling thread-group's line.  `src` = input line (may alias b),
// a/b = scratch lines (a != src).  pre = optional per-input multiplier (global/L1).
// All threads of the block must call (block-wide barriers).  The returned
// pointer is the line buffer holding the natural-order result.
template <int L>
__host__ __device__ constexpr bool result_in_a() { return (Sched<L>::n % 2) == 1; }

// threads per line and lines per block used by the pass kernels (E = L / TPL = 16 inputs per thread)
template <int L>
__host__ __device__ constexpr int tpl_of() { return L <= 256 ? 16 : (L <= 512 ? 32 : 64); }

// src may alias b (stage 0 reads src, later stages never do).
template <int L, int TPL, int SIGN>
BC_DEV float2 *line_fft(const float2 *src, float2 *a, float2 *b, const float2 *tw, const float2 *pre, int tl)
{
    return Run<L, TPL, 0, SIGN>::go(src, a, b, tw, pre, tl);
}

}  // namespace fct
