// fft_ct.cuh -- compile-time mixed-radix FFT of lines held in registers.
//
// Hand-written replacement of the paper's library FFT stages (PAPER.md L524-L526,
// "FFTW on the CPU and cuFFT(W) on the GPU"; Appendix C) so that every
// transform fuses with the arithmetic around it.
//
// A line of length L is owned by TPL consecutive threads; thread tl holds the
// E = L / TPL elements x[m] = line[tl + TPL m] on entry and the outputs
// X[m] = DFT(line)[tl + TPL m] on exit.  Stockham stages (natural order):
//     v[r] = a[j + r L/R] * w_L^{r (j mod Ns) L/(Ns R)},  V = DFT_R(v),
//     b[(j / Ns) Ns R + (j mod Ns) + r Ns] = V[r],        Ns *= R.
// The first stage reads registers, the last writes registers; only the
// stages in between exchange through shared memory (line buffer with
// PAD(idx) = idx + idx/16).  Sizes, radices and thread counts are
// compile-time, so index arithmetic is strength-reduced; stage twiddles come
// from a per-block table tw[m] = exp(-2 pi i m / L), radix-internal twiddles
// are compile-time constants.
#pragma once

#include "common.cuh"

namespace fct {

__host__ __device__ constexpr int pad(int idx) { return idx + (idx >> 4); }
// line stride (float2 units) = 2 mod 16: a half-warp writing 8 lines x 2 consecutive
// elements during the strided-load transposes hits 16 distinct bank pairs
__host__ __device__ constexpr int line_stride(int L) { return ((pad(L - 1) + 1 + 13) & ~15) + 2; }

// ---------------------------------------------------------------- constexpr trigonometry
constexpr double kPiD = 3.14159265358979323846264338327950288;
__host__ __device__ constexpr double csin_red(double x)  // |x| <= pi/4
{
    double t = x, s = x;
    for (int n = 1; n < 14; n++) {
        t *= -x * x / ((2 * n) * (2 * n + 1));
        s += t;
    }
    return s;
}
__host__ __device__ constexpr double ccos_red(double x)
{
    double t = 1, s = 1;
    for (int n = 1; n < 14; n++) {
        t *= -x * x / ((2 * n - 1) * (2 * n));
        s += t;
    }
    return s;
}
// cos / sin of 2 pi m / n for integers (exact octant reduction)
__host__ __device__ constexpr double cos2pi(long long m, long long n)
{
    m %= n;
    if (m < 0) m += n;
    const long long o8 = (8 * m) / n;  // octant 0..7
    const double r = 2 * kPiD * ((double)(8 * m - o8 * n) / (8.0 * n));  // in [0, pi/4)
    switch (o8) {
    case 0: return ccos_red(r);
    case 1: return csin_red(kPiD / 4 - r);
    case 2: return -csin_red(r);
    case 3: return -ccos_red(kPiD / 4 - r);
    case 4: return -ccos_red(r);
    case 5: return -csin_red(kPiD / 4 - r);
    case 6: return csin_red(r);
    default: return ccos_red(kPiD / 4 - r);
    }
}
__host__ __device__ constexpr double sin2pi(long long m, long long n) { return cos2pi(4 * m - n, 4 * n); }

template <int N, int SIGN>
struct WTab {
    float re[N], im[N];
    __host__ __device__ constexpr WTab() : re(), im()
    {
        for (int m = 0; m < N; m++) {
            re[m] = (float)cos2pi(m, N);
            im[m] = (float)(SIGN * sin2pi(m, N));
        }
    }
};

// ---------------------------------------------------------------- small DFTs (SIGN = -1 forward, +1 inverse)
template <int SIGN>
BC_DEV float2 mul_si(float2 a) { return SIGN < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x); }

template <int R, int SIGN> struct Dft;

template <int SIGN> struct Dft<1, SIGN> {
    static BC_DEV void run(float2 *) {}
};

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
        const float2 t2 = __ffma2_rn(f2(-0.5f), t1, v[0]);
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
        const float2 r1 = __ffma2_rn(f2(c2), a2, __ffma2_rn(f2(c1), a1, x0));
        const float2 r2 = __ffma2_rn(f2(c1), a2, __ffma2_rn(f2(c2), a1, x0));
        const float2 i1 = mul_si<SIGN>(__ffma2_rn(f2(s2), b2, __fmul2_rn(f2(s1), b1)));
        const float2 i2 = mul_si<SIGN>(__ffma2_rn(f2(-s1), b2, __fmul2_rn(f2(s2), b1)));
        v[0] = cadd(cadd(x0, a1), a2);
        v[1] = cadd(r1, i1);
        v[4] = csub(r1, i1);
        v[2] = cadd(r2, i2);
        v[3] = csub(r2, i2);
    }
};

// Composite N = N1 N2 (Cooley-Tukey in registers): n = N2 n1 + n2, k = k1 + N1 k2.
template <int N1, int N2, int SIGN>
BC_DEV void dft_ct(float2 *v)
{
    constexpr int N = N1 * N2;
    constexpr WTab<N, SIGN> W{};
    float2 y[N2][N1];
#pragma unroll
    for (int n2 = 0; n2 < N2; n2++) {
        float2 t[N1];
#pragma unroll
        for (int n1 = 0; n1 < N1; n1++) t[n1] = v[N2 * n1 + n2];
        Dft<N1, SIGN>::run(t);
#pragma unroll
        for (int k1 = 0; k1 < N1; k1++) {
            // after unrolling m is a constant: multiples of a quarter turn are swaps / negations
            const int m = (n2 * k1) % N;
            float2 v;
            if (m == 0) v = t[k1];
            else if (4 * m == N) v = mul_si<SIGN>(t[k1]);
            else if (2 * m == N) v = make_float2(-t[k1].x, -t[k1].y);
            else if (4 * m == 3 * N) v = mul_si<-SIGN>(t[k1]);
            else v = cmul(t[k1], make_float2(W.re[m], W.im[m]));
            y[n2][k1] = v;
        }
    }
#pragma unroll
    for (int k1 = 0; k1 < N1; k1++) {
        float2 t[N2];
#pragma unroll
        for (int n2 = 0; n2 < N2; n2++) t[n2] = y[n2][k1];
        Dft<N2, SIGN>::run(t);
#pragma unroll
        for (int k2 = 0; k2 < N2; k2++) v[k1 + N1 * k2] = t[k2];
    }
}

template <int SIGN> struct Dft<6, SIGN> { static BC_DEV void run(float2 *v) { dft_ct<2, 3, SIGN>(v); } };
template <int SIGN> struct Dft<8, SIGN> { static BC_DEV void run(float2 *v) { dft_ct<2, 4, SIGN>(v); } };
template <int SIGN> struct Dft<10, SIGN> { static BC_DEV void run(float2 *v) { dft_ct<2, 5, SIGN>(v); } };
template <int SIGN> struct Dft<12, SIGN> { static BC_DEV void run(float2 *v) { dft_ct<4, 3, SIGN>(v); } };
template <int SIGN> struct Dft<16, SIGN> { static BC_DEV void run(float2 *v) { dft_ct<4, 4, SIGN>(v); } };

// ---------------------------------------------------------------- plans
// n stages with radices r[]; TPL threads per line (TPL divides L/r[0] and L/r[n-1]);
// NL lines per block.
template <int L> struct Plan;
#define BC_PLAN(L_, N_, A_, B_, C_, TPL_, NL_)                                                     \
    template <> struct Plan<L_> {                                                                  \
        static constexpr int n = N_;                                                               \
        static constexpr int r[3] = {A_, B_, C_};                                                  \
        static constexpr int TPL = TPL_;                                                           \
        static constexpr int NL = NL_;                                                             \
    };
//       L   n  radices      TPL NL
BC_PLAN(16, 2, 4, 4, 1, 4, 16)
BC_PLAN(20, 3, 2, 5, 2, 10, 16)
BC_PLAN(24, 3, 2, 3, 4, 6, 16)
BC_PLAN(32, 2, 8, 4, 1, 4, 16)
BC_PLAN(36, 2, 6, 6, 1, 6, 16)
BC_PLAN(40, 3, 2, 5, 4, 10, 16)
BC_PLAN(48, 2, 12, 4, 1, 4, 16)
BC_PLAN(64, 2, 8, 8, 1, 8, 16)
BC_PLAN(72, 2, 12, 6, 1, 6, 16)
BC_PLAN(80, 3, 4, 5, 4, 20, 8)
BC_PLAN(96, 3, 4, 6, 4, 24, 8)
BC_PLAN(128, 2, 16, 8, 1, 8, 16)
BC_PLAN(144, 2, 12, 12, 1, 12, 8)
BC_PLAN(160, 3, 8, 5, 4, 20, 8)
BC_PLAN(192, 3, 8, 3, 8, 24, 8)
BC_PLAN(240, 3, 12, 5, 4, 20, 8)
BC_PLAN(256, 2, 16, 16, 1, 16, 8)
BC_PLAN(288, 3, 12, 2, 12, 24, 8)
BC_PLAN(320, 3, 16, 5, 4, 20, 8)
BC_PLAN(384, 3, 4, 8, 12, 32, 8)
BC_PLAN(512, 3, 16, 2, 16, 32, 4)
BC_PLAN(576, 3, 12, 4, 12, 48, 4)
BC_PLAN(640, 3, 16, 5, 8, 40, 4)
BC_PLAN(768, 3, 16, 3, 16, 48, 4)
BC_PLAN(1024, 3, 16, 4, 16, 64, 2)
#undef BC_PLAN

#define BC_FOR_EACH_L(X) X(16) X(20) X(24) X(32) X(36) X(40) X(48) X(64) X(72) X(80) X(96) X(128) \
    X(144) X(160) X(192) X(240) X(256) X(288) X(320) X(384) X(512) X(576) X(640) X(768) X(1024)

template <int L, int S>
__host__ __device__ constexpr int ns_before()
{
    int ns = 1;
    for (int s = 0; s < S; s++) ns *= Plan<L>::r[s];
    return ns;
}

template <int L>
__host__ __device__ constexpr bool plan_ok()
{
    constexpr int n = Plan<L>::n;
    int p = 1;
    for (int s = 0; s < n; s++) p *= Plan<L>::r[s];
    return p == L && (L / Plan<L>::r[0]) % Plan<L>::TPL == 0 && (L / Plan<L>::r[n - 1]) % Plan<L>::TPL == 0 &&
           n >= 2;
}

// ---------------------------------------------------------------- twiddle table in shared memory
// Flat table tw[m] = exp(-2 pi i m / L) for plans with middle stages; for two-stage plans the
// last stage is the only user and reads w^{r j} with lanes at consecutive j, so the table is
// stored as tw[(r - 1) Ns + j] = w^{r j} (r in [1, R), j in [0, Ns)): conflict-free, where the
// flat table at lane stride r would serialise up to 8-way.
template <int L>
BC_DEV void load_twiddles(float2 *tw_s, const float2 *tw_g, int tid, int nt)
{
    if (Plan<L>::n == 2) {
        constexpr int R = Plan<L>::r[Plan<L>::n - 1], Ns = L / R;
        for (int e = tid; e < (R - 1) * Ns; e += nt) {
            const int r = e / Ns + 1, j = e % Ns;
            tw_s[e] = tw_g[(r * j) % L];
        }
    } else {
        for (int e = tid; e < L; e += nt) tw_s[e] = tw_g[e];
    }
}

// ---------------------------------------------------------------- stages
// middle stage S (0 < S < n-1): shared memory a -> b
template <int L, int S, int SIGN>
BC_DEV void mid_stage(const float2 *__restrict__ a, float2 *__restrict__ b, const float2 *__restrict__ tw, int tl)
{
    constexpr int TPL = Plan<L>::TPL;
    constexpr int R = Plan<L>::r[S];
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
            float2 x = a[pad(j + r * LR)];
            if (r > 0) {
                const float2 w = tw[r * jm * TWS];
                x = SIGN < 0 ? cmul(x, w) : cmulc(x, w);
            }
            v[r] = x;
        }
        Dft<R, SIGN>::run(v);
        const int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
        for (int r = 0; r < R; r++) b[pad(idxD + r * Ns)] = v[r];
    }
}

// Exchange barrier: block-wide, or warp-wide when every line lives inside one warp
// (WS: TPL divides 32, lines start at multiples of TPL) and only its own threads touch its
// buffers.
template <bool WS>
BC_DEV void line_sync()
{
    if (WS)
        __syncwarp();
    else
        __syncthreads();
}
template <int L>
__host__ __device__ constexpr bool warp_local() { return 32 % Plan<L>::TPL == 0; }

template <int L, int S, int SIGN, bool WS, bool DONE = (S >= Plan<L>::n - 1)>
struct Mid;
template <int L, int S, int SIGN, bool WS>
struct Mid<L, S, SIGN, WS, true> {
    static BC_DEV const float2 *go(const float2 *a, float2 *, const float2 *, int) { return a; }
};
template <int L, int S, int SIGN, bool WS>
struct Mid<L, S, SIGN, WS, false> {
    static BC_DEV const float2 *go(const float2 *a, float2 *b, const float2 *tw, int tl)
    {
        mid_stage<L, S, SIGN>(a, b, tw, tl);
        line_sync<WS>();
        return Mid<L, S + 1, SIGN, WS>::go(b, (float2 *)a, tw, tl);
    }
};

// Powers w[r] = u^r, r in [1, R), by a product tree of depth ceil(log2 R) (w[2^k] squares,
// w[h + k] = w[h] w[k]); relative error ~ r eps(u) + depth ulps (< 1e-6 for R = 16).
template <int R>
BC_DEV void twiddle_powers(float2 (&w)[R], float2 u)
{
    w[0] = make_float2(1.f, 0.f);
    if (R > 1) w[1] = u;
#pragma unroll
    for (int k = 2; k < R; k++) {
        int h = 1;
        while (2 * h <= k) h *= 2;  // highest power of two <= k (compile-time after unrolling)
        w[k] = (h == k) ? cmul(w[h / 2], w[h / 2]) : cmul(w[h], w[k - h]);
    }
}

// Two-stage plans whose last stage gives each thread one output group (Ns == TPL): thread
// j's last-stage twiddles are w^{r j} = u^r with u = w^j, so they are generated in registers
// (twiddle_powers) from one base instead of R - 1 shared-memory table loads -- these
// kernels are bound by L1 / shared-memory bandwidth, and sm_100's packed FFMA2 makes the
// 3-instruction complex products cheap.  A per-thread factor c^{r'} on stage input r'
// (a coset twiddle split as c^{tl} W^m) is absorbed by passing u = w^j c.
template <int L>
__host__ __device__ constexpr bool pow_plan() { return Plan<L>::n == 2 && L / Plan<L>::r[1] == Plan<L>::TPL; }

template <int L, int SIGN, bool WS = false>
BC_DEV void fft_regs_pow(float2 (&x)[L / Plan<L>::TPL], float2 *A, float2 u, int tl)
{
    static_assert(pow_plan<L>(), "fft_regs_pow needs a two-stage plan with Ns == TPL");
    static_assert(!WS || warp_local<L>(), "warp-synchronous FFT needs lines inside one warp");
    constexpr int R0 = Plan<L>::r[0], R = Plan<L>::r[1], TPL = Plan<L>::TPL;
    static_assert((L / R0) / TPL == 1, "one stage-0 group per thread");
    {
        float2 v[R0];
#pragma unroll
        for (int r = 0; r < R0; r++) v[r] = x[r];
        Dft<R0, SIGN>::run(v);
#pragma unroll
        for (int r = 0; r < R0; r++) A[pad(tl * R0 + r)] = v[r];
    }
    line_sync<WS>();
    {
        float2 w[R];
        twiddle_powers<R>(w, u);
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
            const float2 y = A[pad(tl + r * TPL)];
            v[r] = r ? cmul(y, w[r]) : y;
        }
        Dft<R, SIGN>::run(v);
#pragma unroll
        for (int r = 0; r < R; r++) x[r] = v[r];
    }
}

// Same two-stage transform with the last stage's twiddles read from a caller table
// tw2[(r - 1) TPL + tl] (r in [1, R)): lanes read consecutive entries (conflict-free).  Used
// where a coset twiddle is absorbed into per-coset tables (fold_fast_kernel).
template <int L, int SIGN, bool WS = false>
BC_DEV void fft_regs_tab(float2 (&x)[L / Plan<L>::TPL], float2 *A, const float2 *tw2, int tl)
{
    static_assert(pow_plan<L>(), "fft_regs_tab needs a two-stage plan with Ns == TPL");
    constexpr int R0 = Plan<L>::r[0], R = Plan<L>::r[1], TPL = Plan<L>::TPL;
    {
        float2 v[R0];
#pragma unroll
        for (int r = 0; r < R0; r++) v[r] = x[r];
        Dft<R0, SIGN>::run(v);
#pragma unroll
        for (int r = 0; r < R0; r++) A[pad(tl * R0 + r)] = v[r];
    }
    line_sync<WS>();
    {
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
            const float2 y = A[pad(tl + r * TPL)];
            v[r] = r ? cmul(y, tw2[(r - 1) * TPL + tl]) : y;
        }
        Dft<R, SIGN>::run(v);
#pragma unroll
        for (int r = 0; r < R; r++) x[r] = v[r];
    }
}

// ---------------------------------------------------------------- three-stage plans, conflict-free tables
// The flat table read as tw[r * jm * TWS] (mid stage) and tw[r * j] (last stage) puts lanes at
// stride r (or the Ns distinct jm rows at stride r TWS) and serialises up to 8-way (ncu on the
// L = 384 docking passes: 27 % of all shared wavefronts excessive).  T3 tables instead:
//   mid stage (S = 1, Ns = R0): twm[jm * (R1 + 1) + r] = w^{r jm L / (R0 R1)} -- a warp reads
//     R0 distinct rows, padded by one entry so they fall in different banks;
//   last stage (Ns = R0 R1): twl[(r - 1) Ns + j] = w^{r j} -- lanes read consecutive entries.
template <int L>
struct T3 {
    static_assert(Plan<L>::n == 3, "three-stage plans only");
    static constexpr int R0 = Plan<L>::r[0], R1 = Plan<L>::r[1], R2 = Plan<L>::r[2];
    static constexpr int NS2 = R0 * R1, MROW = R1 + 1;
    static constexpr int MSIZE = R0 * MROW, LSIZE = (R2 - 1) * NS2;
    static constexpr int SIZE = (MSIZE + LSIZE + 1) & ~1;  // even: 16-byte aligned buffers after it
    // the mid stage writes rows of R0 R1 outputs with lane groups R1 elements apart; 4 pad
    // slots per row put the warp's 32 stores on distinct bank pairs (the default pad, one slot
    // per 16, left up to 4 lanes on one pair).  A line's B buffer needs BLEN elements.
    static constexpr int ROW = R0 * R1;
    __host__ __device__ static constexpr int padB(int idx) { return idx + (idx / ROW) * 4; }
    static constexpr int BLEN = L + (L / ROW) * 4;
};

template <int L>
BC_DEV void load_twiddles_t3(float2 *t, const float2 *tw_g, int tid, int nt)
{
    using P = T3<L>;
    for (int e = tid; e < P::MSIZE + P::LSIZE; e += nt) {
        int idx;
        if (e < P::MSIZE) {
            const int jm = e / P::MROW, r = e % P::MROW;
            idx = r < P::R1 ? r * jm * (L / (P::R0 * P::R1)) : 0;
        } else {
            const int q = e - P::MSIZE;
            idx = ((q / P::NS2 + 1) * (q % P::NS2)) % L;
        }
        t[e] = tw_g[idx];
    }
}

// fft_regs for three-stage plans on the T3 tables (same data layout in and out).
template <int L, int SIGN, bool WS = false>
BC_DEV void fft_regs_t3(float2 (&x)[L / Plan<L>::TPL], float2 *A, float2 *B, const float2 *t3, int tl)
{
    static_assert(!WS || warp_local<L>(), "warp-synchronous FFT needs lines inside one warp");
    static_assert(plan_ok<L>(), "bad FFT plan");
    using P = T3<L>;
    constexpr int TPL = Plan<L>::TPL;
    {   // stage 0 (Ns = 1): registers -> A
        constexpr int R = P::R0, U = (L / R) / TPL;
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int j = tl + TPL * u;
            float2 v[R];
#pragma unroll
            for (int r = 0; r < R; r++) v[r] = x[u + U * r];
            Dft<R, SIGN>::run(v);
#pragma unroll
            for (int r = 0; r < R; r++) A[pad(j * R + r)] = v[r];
        }
    }
    line_sync<WS>();
    {   // mid stage (Ns = R0): A -> B
        constexpr int R = P::R1, Ns = P::R0, LR = L / R;
#pragma unroll
        for (int j0 = 0; j0 < LR; j0 += TPL) {
            const int j = j0 + tl;
            if ((LR % TPL) != 0 && j >= LR) break;
            const int jm = j % Ns;
            float2 v[R];
#pragma unroll
            for (int r = 0; r < R; r++) {
                float2 y = A[pad(j + r * LR)];
                if (r > 0) {
                    const float2 w = t3[jm * P::MROW + r];
                    y = SIGN < 0 ? cmul(y, w) : cmulc(y, w);
                }
                v[r] = y;
            }
            Dft<R, SIGN>::run(v);
            const int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
            for (int r = 0; r < R; r++) B[P::padB(idxD + r * Ns)] = v[r];
        }
    }
    line_sync<WS>();
    {   // last stage (Ns = R0 R1): B -> registers
        constexpr int R = P::R2, Ns = P::NS2, U = Ns / TPL;
        const float2 *twl = t3 + P::MSIZE;
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int j = tl + TPL * u;
            float2 v[R];
#pragma unroll
            for (int r = 0; r < R; r++) {
                float2 y = B[P::padB(j + r * Ns)];
                if (r > 0) {
                    const float2 w = twl[(r - 1) * Ns + j];
                    y = SIGN < 0 ? cmul(y, w) : cmulc(y, w);
                }
                v[r] = y;
            }
            Dft<R, SIGN>::run(v);
#pragma unroll
            for (int r = 0; r < R; r++) x[u + U * r] = v[r];
        }
    }
}

// FFT of the calling thread-group's line, registers in / registers out (see header).
// A and B are this line's shared-memory buffers (B used only when n >= 3).
// Contains barriers (block-wide, or warp-wide with WS = true, which requires
// warp_local<L>()): every thread of the block (warp) must call it.  The caller must
// barrier before writing A/B again (the last stage reads them); the twiddle table tw must
// be visible to the calling threads before the call.
template <int L, int SIGN, bool WS = false, bool POW = true>
BC_DEV void fft_regs(float2 (&x)[L / Plan<L>::TPL], float2 *A, float2 *B, const float2 *tw, int tl)
{
    static_assert(!WS || warp_local<L>(), "warp-synchronous FFT needs lines inside one warp");
    static_assert(plan_ok<L>(), "bad FFT plan");
    constexpr int TPL = Plan<L>::TPL;
    constexpr int n = Plan<L>::n;
    if constexpr (POW && L == 256 && pow_plan<L>()) {  // last-stage twiddles as powers of tw[tl] = w^{tl} (table row r = 1)
        const float2 w1 = tw[tl];
        fft_regs_pow<L, SIGN, WS>(x, A, SIGN < 0 ? w1 : cconj(w1), tl);
        return;
    }
    // stage 0 (Ns = 1, no twiddles): registers -> A
    {
        constexpr int R = Plan<L>::r[0];
        constexpr int U = (L / R) / TPL;
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int j = tl + TPL * u;
            float2 v[R];
#pragma unroll
            for (int r = 0; r < R; r++) v[r] = x[u + U * r];
            Dft<R, SIGN>::run(v);
#pragma unroll
            for (int r = 0; r < R; r++) A[pad(j * R + r)] = v[r];
        }
    }
    line_sync<WS>();
    const float2 *cur = Mid<L, 1, SIGN, WS>::go(A, B, tw, tl);
    // last stage (Ns = L / R): shared memory -> registers, output index j + r Ns
    {
        constexpr int R = Plan<L>::r[n - 1];
        constexpr int Ns = L / R;
        constexpr int U = Ns / TPL;
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int j = tl + TPL * u;
            float2 v[R];
#pragma unroll
            for (int r = 0; r < R; r++) {
                float2 y = cur[pad(j + r * Ns)];
                if (r > 0) {
                    const float2 w = n == 2 ? tw[(r - 1) * Ns + j] : tw[r * j];
                    y = SIGN < 0 ? cmul(y, w) : cmulc(y, w);
                }
                v[r] = y;
            }
            Dft<R, SIGN>::run(v);
#pragma unroll
            for (int r = 0; r < R; r++) x[u + U * r] = v[r];
        }
    }
}

}  // namespace fct
