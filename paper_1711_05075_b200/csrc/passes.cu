// passes.cu -- box-DFT passes, fused x-pass + spectral product + fold, inverse passes.
//
// Per rotation (eq_ccghat), after spreading the smoothed
// density of R B onto its box (spread.cu):
//   pass_contig  (z)  box [ix][iy][iz]  -> T1 [ix][iy][kz]
//   pass_strided (y)  T1               -> T2 [ix][ky][kz]
//   fold_x            T2 -> x-transform -> f_hat_A'(k) conj(f_hat_RB(k)) -> F[k mod Np]   (fused)
//   pass_strided (x, inverse) F -> X1 [mx][k'y][k'z]
//   pass_strided (y, inverse) X1 -> Y1 [mx][my][k'z]
//   last (z, inverse, C2R) Y1 -> f(t_m) or per-rotation min / max keys
// One axis of the box DFT is X(k) = mult(k) sum_{n<L} x_n exp(-2 pi i k n / G), G = c L,
// evaluated through c cosets k = c q + p of an L-point FFT of x_n exp(-2 pi i p n / G).
// Each block keeps its raw input lines in registers (L / TPL values per thread) and
// rewrites the coset-twiddled copy into shared memory before every coset FFT.
#include "kernels.cuh"
#include "fft_ct.cuh"

#include "ballcorr.h"

using namespace fct;

constexpr int BS = 128;  // threads per block of every FFT pass

template <int L>
__host__ __device__ constexpr int nl_of() { return BS / tpl_of<L>(); }
template <int L>
__host__ __device__ constexpr int epr_of() { return (L * nl_of<L>() + BS - 1) / BS; }  // inputs per thread

__device__ __forceinline__ int coset_kk(int q, int p, int c, int G, int klo, int signed_k)
{
    int k = c * q + p;
    if (signed_k && 2 * k > G) k -= G;
    return k - klo;
}

template <int L>
__device__ __forceinline__ void load_tw(float2 *tw, const float2 *g)
{
    for (int m = threadIdx.x; m < L; m += BS) tw[m] = g[m];
}

// ============================================================================ contiguous axis (forward z)

template <int L, bool REAL_IN>
__global__ void __launch_bounds__(BS) pass_contig_kernel(PassArgs a)
{
    constexpr int TPL = tpl_of<L>(), NL = nl_of<L>(), LS = line_stride(L), E = epr_of<L>();
    extern __shared__ float2 sm[];
    float2 *tw = sm;
    float2 *A = tw + L;
    float2 *B = A + NL * LS;
    float2 *OUT = B + NL * LS;
    const int line = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const int b = blockIdx.y;
    const long long gline = (long long)blockIdx.x * NL + line;
    const bool valid = gline < a.lines;

    load_tw<L>(tw, a.tw);
    float2 x[E];
#pragma unroll
    for (int m = 0; m < E; m++) {
        const int n = tl + TPL * m;
        x[m] = make_float2(0.f, 0.f);
        if (valid && n < L) {
            if (REAL_IN)
                x[m].x = ((const float *)a.in)[(long long)b * a.in_bstride + gline * L + n];
            else
                x[m] = ((const float2 *)a.in)[(long long)b * a.in_bstride + gline * L + n];
        }
    }
    for (int p = 0; p < a.c; p++) {
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int n = tl + TPL * m;
            if (n < L) A[line * LS + pad(n)] = p ? cmul(x[m], a.ctw[p * L + n]) : x[m];
        }
        __syncthreads();
        const float2 *res = line_fft<L, TPL, -1>(A + line * LS, B + line * LS, A + line * LS, tw, nullptr, tl);
        for (int q = tl; q < L; q += TPL) {
            const int kk = coset_kk(q, p, a.c, a.G, a.klo, a.signed_k);
            if (kk >= 0 && kk < a.nk) OUT[line * a.nk + kk] = cmul(res[pad(q)], a.mult[kk]);
        }
        __syncthreads();
    }
    const long long base = (long long)b * a.out_bstride + (long long)blockIdx.x * NL * a.nk;
    for (int e = threadIdx.x; e < NL * a.nk; e += BS) {
        const int l = e / a.nk;
        if ((long long)blockIdx.x * NL + l < a.lines) a.out[base + e] = OUT[e];
    }
}

// ============================================================================ strided axis (forward / inverse)

template <int L, int SIGN>
__global__ void __launch_bounds__(BS) pass_strided_kernel(PassArgs a)
{
    constexpr int TPL = tpl_of<L>(), NL = nl_of<L>(), LS = line_stride(L), E = epr_of<L>();
    extern __shared__ float2 sm[];
    float2 *tw = sm;
    float2 *A = tw + L;
    float2 *B = A + NL * LS;
    const int line = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const int b = blockIdx.y;
    const int itiles = (a.I + NL - 1) / NL;
    const int o = blockIdx.x / itiles;
    const int i0 = (blockIdx.x % itiles) * NL;
    const float2 *in = (const float2 *)a.in + (long long)b * a.in_bstride + (long long)o * L * a.I;
    float2 *out = a.out + (long long)b * a.out_bstride + (long long)o * a.nk * a.I;

    load_tw<L>(tw, a.tw);
    float2 x[E];
#pragma unroll
    for (int m = 0; m < E; m++) {
        const int e = threadIdx.x + BS * m;
        const int n = e / NL, i = e % NL;
        x[m] = (e < L * NL && i0 + i < a.I) ? in[(long long)n * a.I + i0 + i] : make_float2(0.f, 0.f);
    }
    float2 *resbuf = result_in_a<L>() ? B : A;  // stage 0 writes B (line_fft(A, B, A))
    for (int p = 0; p < a.c; p++) {
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int e = threadIdx.x + BS * m;
            const int n = e / NL, i = e % NL;
            if (e < L * NL) A[i * LS + pad(n)] = p ? cmul(x[m], a.ctw[p * L + n]) : x[m];
        }
        __syncthreads();
        line_fft<L, TPL, SIGN>(A + line * LS, B + line * LS, A + line * LS, tw, nullptr, tl);
        for (int e = threadIdx.x; e < L * NL; e += BS) {
            const int q = e / NL, i = e % NL;
            const int kk = coset_kk(q, p, a.c, a.G, a.klo, a.signed_k);
            if (kk >= 0 && kk < a.nk && i0 + i < a.I) {
                float2 v = resbuf[i * LS + pad(q)];
                if (a.mult) v = cmul(v, a.mult[kk]);
                out[(long long)kk * a.I + i0 + i] = v;
            }
        }
        __syncthreads();
    }
}

// ============================================================================ fused x-pass + product + fold

// Block: target row k'y = blockIdx.x / ztiles, targets k'z in [z0, z0 + 8), all k'x.
// For every alias group (ky, kz) of those targets, the x-transform of the T2 lines of
// R B gives f_hat_RB(kx, ky, kz) on the band; times f_hat_A'(k) (A's spectrum with the
// origin phase exp(2 pi i k.t0/P) folded in) and summed into F[k mod Np].
// DIRECT: every fold target of a coset is owned by one thread (Np / gcd(c, Np) is a
// multiple of TPL and G is a multiple of Np), so products accumulate straight into acc; otherwise they are
// staged per line in Pb[kx] and gathered.
template <int L, bool CPLX, bool DIRECT>
__global__ void __launch_bounds__(8 * tpl_of<L>()) fold_x_kernel(FoldXArgs a)
{
    constexpr int NL = 8;
    constexpr int TPL = tpl_of<L>();
    constexpr int NT = NL * TPL;
    constexpr int LS = line_stride(L);
    constexpr int E = (L * NL + NT - 1) / NT;
    extern __shared__ float2 sm[];
    float2 *tw = sm;
    float2 *A = tw + L;
    float2 *B = A + NL * LS;
    float2 *acc = B + NL * LS;           // [NL][Np]
    float2 *Pb = acc + NL * a.Np;        // [NL][M] (gather path only)
    const int line = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const int b = blockIdx.y;
    const int K = a.K, M = a.M, Np = a.Np, Kz = a.Kz;
    const int ztiles = (a.Fz + NL - 1) / NL;
    const int kyp = blockIdx.x / ztiles;
    const int z0 = (blockIdx.x % ztiles) * NL;
    const float2 *T2 = a.T2 + (long long)b * a.t2_bstride;
    float2 *resbuf = result_in_a<L>() ? B : A;

    for (int m = threadIdx.x; m < L; m += NT) tw[m] = a.tw[m];
    for (int e = threadIdx.x; e < NL * Np; e += NT) acc[e] = make_float2(0.f, 0.f);

    const int span = K / Np + 2;
    for (int pass = 0; pass < (CPLX ? 1 : 2); pass++) {
        const int s = pass ? -1 : 1;   // conj pass: target (-k) mod Np
        const int zlo = CPLX ? -K : (pass ? 1 : 0);
        for (int nz = -span; nz <= span; nz++) {
            bool any = false;
            for (int i = 0; i < NL; i++) {
                const int kz = s * (z0 + i) + nz * Np;
                any |= (z0 + i < a.Fz) && kz >= zlo && kz <= K;
            }
            if (!any) continue;
            for (int ny = -span; ny <= span; ny++) {
                const int ky = s * kyp + ny * Np;
                if (ky < -K || ky > K) continue;
                // source lines of R B: (ky, kz) for real weights, (-ky, -kz) for complex (f_hat_RB(-k))
                const int kys = CPLX ? -ky : ky;
                float2 x[E];
#pragma unroll
                for (int m = 0; m < E; m++) {
                    const int e = threadIdx.x + NT * m;
                    const int n = e / NL, i = e % NL;
                    const int kz = s * (z0 + i) + nz * Np;
                    x[m] = make_float2(0.f, 0.f);
                    if (e < L * NL && (z0 + i < a.Fz) && kz >= zlo && kz <= K) {
                        const int kzs = CPLX ? (-kz + K) : kz;
                        x[m] = T2[((long long)n * M + (kys + K)) * Kz + kzs];
                    }
                }
                for (int p = 0; p < a.c; p++) {
#pragma unroll
                    for (int m = 0; m < E; m++) {
                        const int e = threadIdx.x + NT * m;
                        const int n = e / NL, i = e % NL;
                        if (e < L * NL) A[i * LS + pad(n)] = p ? cmul(x[m], a.ctw[p * L + n]) : x[m];
                    }
                    __syncthreads();
                    line_fft<L, TPL, -1>(A + line * LS, B + line * LS, A + line * LS, tw, nullptr, tl);
                    for (int e = threadIdx.x; e < L * NL; e += NT) {
                        const int q = e / NL, i = e % NL;
                        int kx = a.c * q + p;
                        if (2 * kx > a.G) kx -= a.G;
                        if (kx < -K || kx > K) continue;
                        const int kz = s * (z0 + i) + nz * Np;
                        const bool ok = (z0 + i < a.Fz) && kz >= zlo && kz <= K;
                        float2 P = make_float2(0.f, 0.f);
                        int kxa = kx;
                        if (ok) {
                            const float2 bv = cmul(resbuf[i * LS + pad(q)], a.mult[kx + K]);
                            if (!CPLX) {
                                const float2 av = a.Ahat[((long long)(kx + K) * M + (ky + K)) * Kz + kz];
                                P = cmulc(av, bv);   // f_hat_A'(k) conj(f_hat_RB(k))
                            } else {
                                // bv = f_hat_RB(kx, -ky, -kz) = f_hat_RB(-k') at k' = (-kx, ky, kz)
                                kxa = -kx;
                                const float2 av = a.Ahat[((long long)(kxa + K) * M + (ky + K)) * Kz + (kz + K)];
                                P = cmul(av, bv);    // weights not conjugated (reading C-3)
                            }
                        }
                        if (DIRECT) {
                            if (ok) {
                                int t = (s > 0 ? kxa : -kxa) % Np;
                                if (t < 0) t += Np;
                                acc[i * Np + t] = cadd(acc[i * Np + t], s > 0 ? P : cconj(P));
                            }
                        } else {
                            Pb[i * M + kxa + K] = P;
                        }
                    }
                    __syncthreads();
                }
                if (!DIRECT) {
                    for (int e = threadIdx.x; e < NL * Np; e += NT) {
                        const int i = e % NL, t = e / NL;
                        const int base = s > 0 ? t : (Np - t) % Np;
                        int kx = base - ((base + K) / Np) * Np;   // smallest alias >= -K
                        float2 sum = make_float2(0.f, 0.f);
                        for (; kx <= K; kx += Np) sum = cadd(sum, Pb[i * M + kx + K]);
                        acc[i * Np + t] = cadd(acc[i * Np + t], s > 0 ? sum : cconj(sum));
                    }
                    __syncthreads();
                }
            }
        }
    }
    float2 *F = a.F + (long long)b * a.f_bstride;
    for (int e = threadIdx.x; e < NL * Np; e += NT) {
        const int i = e % NL, t = e / NL;
        if (z0 + i < a.Fz) F[((long long)t * Np + kyp) * a.Fz + z0 + i] = acc[i * Np + t];
    }
}

// ============================================================================ last inverse pass + epilogue

__device__ __forceinline__ unsigned long long key_min(float v, unsigned idx)
{
    return ((unsigned long long)float_order_bits(v) << 32) | idx;
}
__device__ __forceinline__ unsigned long long key_max(float v, unsigned idx)
{
    return ((unsigned long long)float_order_bits(v) << 32) | (0xffffffffu - idx);
}

template <int L, bool HERM>
__global__ void __launch_bounds__(BS) last_kernel(LastArgs a)
{
    constexpr int TPL = tpl_of<L>(), NL = nl_of<L>(), LS = line_stride(L);
    extern __shared__ float2 sm[];
    float2 *tw = sm;
    float2 *A = tw + L;
    float2 *B = A + NL * LS;
    const int line = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const int b = blockIdx.y;
    const long long lines = (long long)a.N * a.N;
    const long long gline = (long long)blockIdx.x * NL + line;
    const bool valid = gline < lines;

    load_tw<L>(tw, a.tw);
    {
        const float2 *row = a.in + (long long)b * a.in_bstride + gline * a.Fz;
        float2 *dst = A + line * LS;
        for (int n = tl; n < L; n += TPL) {
            float2 v = make_float2(0.f, 0.f);
            if (valid) {
                if (!HERM || n < a.Fz)
                    v = row[n];
                else
                    v = cconj(row[L - n]);
            }
            dst[pad(n)] = v;
        }
    }
    __syncthreads();
    const float2 *res = line_fft<L, TPL, +1>(A + line * LS, B + line * LS, A + line * LS, tw, nullptr, tl);

    unsigned long long kmin = ~0ull, kmax = 0ull;
    if (valid) {
        for (int m = tl; m < a.N; m += TPL) {
            const float2 v = cscale(res[pad(m)], a.scale);
            const long long gidx = gline * a.N + m;
            if (a.out_kind == BC_OUT_F_FULL) {
                if (HERM)
                    ((float *)a.out_full)[(long long)b * a.full_bstride + gidx] = v.x;
                else
                    ((float2 *)a.out_full)[(long long)b * a.full_bstride + gidx] = v;
            } else {
                const unsigned gi = (unsigned)gidx;
                const unsigned long long k1 = key_min(v.x, gi), k2 = key_max(v.x, gi);
                kmin = k1 < kmin ? k1 : kmin;
                kmax = k2 > kmax ? k2 : kmax;
            }
        }
    }
    if (a.out_kind != BC_OUT_F_FULL) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o1 = __shfl_xor_sync(0xffffffffu, kmin, off);
            const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, kmax, off);
            kmin = o1 < kmin ? o1 : kmin;
            kmax = o2 > kmax ? o2 : kmax;
        }
        if ((threadIdx.x & 31) == 0) {
            if (kmin != ~0ull) atomicMin(&a.keys[2 * b + 0], kmin);
            if (kmax != 0ull) atomicMax(&a.keys[2 * b + 1], kmax);
        }
    }
}

// ============================================================================ host dispatch

template <int L>
static size_t fft_smem(size_t extra_f2)
{
    return sizeof(float2) * ((size_t)L + 2 * (size_t)nl_of<L>() * line_stride(L) + extra_f2);
}

template <typename KernelT>
static void set_smem(KernelT k, size_t bytes)
{
    if (bytes > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

bool fft_size_supported(int L)
{
    switch (L) {
#define X(L_) case L_:
        BC_FOR_EACH_L(X)
#undef X
        return true;
    default: return false;
    }
}

static int gcd_int(int a, int b) { return b ? gcd_int(b, a % b) : a; }

void launch_pass_contig(const PassArgs &a, int batch, cudaStream_t s)
{
    switch (a.L) {
#define X(L_)                                                                                 \
    case L_: {                                                                                \
        constexpr int NL = nl_of<L_>();                                                       \
        const size_t sm = fft_smem<L_>((size_t)NL * a.nk);                                    \
        dim3 grid((unsigned)((a.lines + NL - 1) / NL), batch);                                \
        if (a.in_real) {                                                                      \
            set_smem(pass_contig_kernel<L_, true>, sm);                                       \
            pass_contig_kernel<L_, true><<<grid, BS, sm, s>>>(a);                             \
        } else {                                                                              \
            set_smem(pass_contig_kernel<L_, false>, sm);                                      \
            pass_contig_kernel<L_, false><<<grid, BS, sm, s>>>(a);                            \
        }                                                                                     \
        break;                                                                                \
    }
        BC_FOR_EACH_L(X)
#undef X
    default: break;
    }
}

void launch_pass_strided(const PassArgs &a, int sign, int batch, cudaStream_t s)
{
    switch (a.L) {
#define X(L_)                                                                                 \
    case L_: {                                                                                \
        constexpr int NL = nl_of<L_>();                                                       \
        const size_t sm = fft_smem<L_>(0);                                                    \
        const int itiles = (a.I + NL - 1) / NL;                                               \
        dim3 grid((unsigned)(a.O * itiles), batch);                                           \
        if (sign < 0) {                                                                       \
            set_smem(pass_strided_kernel<L_, -1>, sm);                                        \
            pass_strided_kernel<L_, -1><<<grid, BS, sm, s>>>(a);                              \
        } else {                                                                              \
            set_smem(pass_strided_kernel<L_, 1>, sm);                                         \
            pass_strided_kernel<L_, 1><<<grid, BS, sm, s>>>(a);                               \
        }                                                                                     \
        break;                                                                                \
    }
        BC_FOR_EACH_L(X)
#undef X
    default: break;
    }
}

template <int L, bool CPLX, bool DIRECT>
static void fold_launch(const FoldXArgs &a, dim3 grid, cudaStream_t s)
{
    const size_t sm = sizeof(float2) * ((size_t)L + 2 * 8 * (size_t)line_stride(L) + 8 * (size_t)a.Np +
                                        (DIRECT ? 0 : 8 * (size_t)a.M));
    set_smem(fold_x_kernel<L, CPLX, DIRECT>, sm);
    fold_x_kernel<L, CPLX, DIRECT><<<grid, 8 * tpl_of<L>(), sm, s>>>(a);
}

void launch_fold_x(const FoldXArgs &a, int batch, cudaStream_t s)
{
    const int ztiles = (a.Fz + 7) / 8;
    dim3 grid((unsigned)(a.Np * ztiles), batch);
    switch (a.L) {
#define X(L_)                                                                                   \
    case L_: {                                                                                  \
        const bool direct = ((a.Np / gcd_int(a.c, a.Np)) % tpl_of<L_>()) == 0 && (a.G % a.Np) == 0;                 \
        if (a.complex_w) {                                                                      \
            if (direct) fold_launch<L_, true, true>(a, grid, s);                                \
            else fold_launch<L_, true, false>(a, grid, s);                                      \
        } else {                                                                                \
            if (direct) fold_launch<L_, false, true>(a, grid, s);                               \
            else fold_launch<L_, false, false>(a, grid, s);                                     \
        }                                                                                       \
        break;                                                                                  \
    }
        BC_FOR_EACH_L(X)
#undef X
    default: break;
    }
}

void launch_last(const LastArgs &a, int batch, cudaStream_t s)
{
    switch (a.Np) {
#define X(L_)                                                                                 \
    case L_: {                                                                                \
        constexpr int NL = nl_of<L_>();                                                       \
        const size_t sm = fft_smem<L_>(0);                                                    \
        const long long lines = (long long)a.N * a.N;                                         \
        dim3 grid((unsigned)((lines + NL - 1) / NL), batch);                                  \
        if (a.hermitian) {                                                                    \
            set_smem(last_kernel<L_, true>, sm);                                              \
            last_kernel<L_, true><<<grid, BS, sm, s>>>(a);                                    \
        } else {                                                                              \
            set_smem(last_kernel<L_, false>, sm);                                             \
            last_kernel<L_, false><<<grid, BS, sm, s>>>(a);                                   \
        }                                                                                     \
        break;                                                                                \
    }
        BC_FOR_EACH_L(X)
#undef X
    default: break;
    }
}

// ============================================================================ reduction keys

__global__ void keys_init_kernel(unsigned long long *keys, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = (i & 1) ? 0ull : ~0ull;
}

void launch_keys_init(unsigned long long *keys, int n, cudaStream_t s)
{
    keys_init_kernel<<<(n + 255) / 256, 256, 0, s>>>(keys, n);
}

__global__ void keys_finalize_kernel(const unsigned long long *keys, int batch, int kind, bc_extremum *out)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= batch) return;
    const unsigned long long kmin = keys[2 * r], kmax = keys[2 * r + 1];
    bc_extremum emin, emax;
    emin.val = (double)float_from_order_bits((uint32_t)(kmin >> 32));
    emin.idx = (int64_t)(kmin & 0xffffffffull);
    emax.val = (double)float_from_order_bits((uint32_t)(kmax >> 32));
    emax.idx = (int64_t)(0xffffffffull - (kmax & 0xffffffffull));
    if (kind == BC_OUT_MIN_ARGMIN)
        out[r] = emin;
    else if (kind == BC_OUT_MINMAX) {
        out[2 * r] = emin;
        out[2 * r + 1] = emax;
    } else
        out[r] = emax;
}

void launch_keys_finalize(const unsigned long long *keys, int batch, int out_kind, void *out, cudaStream_t s)
{
    keys_finalize_kernel<<<(batch + 127) / 128, 128, 0, s>>>(keys, batch, out_kind, (bc_extremum *)out);
}
