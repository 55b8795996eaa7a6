// passes.cu -- box-DFT passes, fused x-pass + spectral product + fold, inverse passes.
//
// Per rotation (eq_ccghat), after spreading the smoothed
// density of R B onto its box (spread.cu):
//   pass (z, contig)   box [ix][iy][iz]  -> T1 [ix][iy][kz]
//   pass (y, strided)  T1               -> T2 [ix][ky][kz]
//   fold_x             T2 -> x-transform -> f_hat_A'(k) conj(f_hat_RB(k)) -> F[k mod Np]   (fused)
//   pass (x, inverse)  F  -> X1 [mx][k'y][k'z]
//   pass (y, inverse)  X1 -> Y1 [mx][my][k'z]
//   last (z, inverse, C2R) Y1 -> f(t_m) or per-rotation min / max keys
// For A (once): z, y, then an x pass writing A' = A_hat * origin phase as [ky][kz][kx].
// One axis of the box DFT is X(k) = mult(k) sum_{n<L} x_n exp(-2 pi i k n / G), G = c L,
// evaluated through c cosets k = c q + p of an L-point FFT of x_n exp(-2 pi i p n / G).
// Lines live in registers (fft_ct.cuh); strided loads / stores are transposed through
// shared memory so that global accesses stay coalesced.
#include "kernels.cuh"
#include "fft_ct.cuh"

#include "ballcorr.h"

using namespace fct;

__device__ __forceinline__ int coset_kk(int q, int p, int c, int G, int klo, int signed_k)
{
    int k = c * q + p;
    if (signed_k && 2 * k > G) k -= G;
    return k - klo;
}

// ============================================================================ generic axis pass
// IN_MODE: 0 contiguous real rows, 1 contiguous complex rows, 2 strided in[b][O][L][I].
// OUT_MODE: 0 rows out[b][row][nk] (row = line index), 1 strided out[b][O][nk][I].
template <int L, int SIGN, int IN_MODE, int OUT_MODE>
__global__ void __launch_bounds__(Plan<L>::TPL * Plan<L>::NL, 512 / (Plan<L>::TPL * Plan<L>::NL)) pass_kernel(PassArgs a)
{
    constexpr int TPL = Plan<L>::TPL, NL = Plan<L>::NL, NT = TPL * NL;
    constexpr int LS = line_stride(L), E = L / TPL;
    extern __shared__ float2 sm[];
    float2 *tw = sm;
    float2 *A = tw + L;
    float2 *B = A + NL * LS;
    float2 *OUT = B + NL * LS;
    const int line = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const int b = blockIdx.y;

    long long row0;  // global row (line) index of this block's first line
    int o = 0, i0 = 0;
    if (IN_MODE == 2) {
        const int itiles = (a.I + NL - 1) / NL;
        o = blockIdx.x / itiles;
        i0 = (blockIdx.x % itiles) * NL;
        row0 = (long long)o * a.I + i0;
    } else {
        row0 = (long long)blockIdx.x * NL;
    }
    const long long nrows = IN_MODE == 2 ? (long long)a.O * a.I : a.lines;
    const bool valid = IN_MODE == 2 ? (i0 + line < a.I) : (row0 + line < nrows);

    for (int m = threadIdx.x; m < L; m += NT) tw[m] = a.tw[m];
    float2 x[E];
    if (IN_MODE == 2) {
        const float2 *in = (const float2 *)a.in + (long long)b * a.in_bstride + (long long)o * L * a.I;
        // all loads first (E independent loads in flight per thread), then the transpose
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int e = threadIdx.x + NT * m;
            const int n = e / NL, i = e % NL;
            x[m] = (i0 + i < a.I) ? in[(long long)n * a.I + i0 + i] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int e = threadIdx.x + NT * m;
            A[(e % NL) * LS + pad(e / NL)] = x[m];
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < E; m++) x[m] = A[line * LS + pad(tl + TPL * m)];
        __syncthreads();
    } else {
        const long long g = (long long)b * a.in_bstride + (row0 + line) * L;
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int n = tl + TPL * m;
            x[m] = make_float2(0.f, 0.f);
            if (valid) {
                if (IN_MODE == 0)
                    x[m].x = ((const float *)a.in)[g + n];
                else
                    x[m] = ((const float2 *)a.in)[g + n];
            }
        }
    }

    float2 *outs = a.out + (long long)b * a.out_bstride;
    for (int p = 0; p < a.c; p++) {
        float2 y[E];
#pragma unroll
        for (int m = 0; m < E; m++) y[m] = p ? cmul(x[m], a.ctw[p * L + tl + TPL * m]) : x[m];
        fft_regs<L, SIGN>(y, A + line * LS, B + line * LS, tw, tl);
        if (OUT_MODE == 0) {
#pragma unroll
            for (int m = 0; m < E; m++) {
                const int kk = coset_kk(tl + TPL * m, p, a.c, a.G, a.klo, a.signed_k);
                if (kk >= 0 && kk < a.nk) OUT[line * a.nk + kk] = a.mult ? cmul(y[m], a.mult[kk]) : y[m];
            }
            __syncthreads();
        } else {
            __syncthreads();
#pragma unroll
            for (int m = 0; m < E; m++) A[line * LS + pad(tl + TPL * m)] = y[m];
            __syncthreads();
            float2 *out = outs + (long long)o * a.nk * a.I;
            for (int e = threadIdx.x; e < L * NL; e += NT) {
                const int q = e / NL, i = e % NL;
                const int kk = coset_kk(q, p, a.c, a.G, a.klo, a.signed_k);
                if (kk >= 0 && kk < a.nk && i0 + i < a.I) {
                    const float2 v = A[i * LS + pad(q)];
                    out[(long long)kk * a.I + i0 + i] = a.mult ? cmul(v, a.mult[kk]) : v;
                }
            }
            __syncthreads();
        }
    }
    if (OUT_MODE == 0) {
        for (int e = threadIdx.x; e < NL * a.nk; e += NT) {
            const int l = e / a.nk;
            const bool ok = IN_MODE == 2 ? (i0 + l < a.I) : (row0 + l < nrows);
            if (ok) outs[(row0 + l) * a.nk + (e % a.nk)] = OUT[e];
        }
    }
}

// ============================================================================ fused x-pass + product + fold

// Block: target row k'y = blockIdx.x / ztiles, targets k'z in [z0, z0 + 8), all k'x.
// For every alias group (ky, kz) of those targets, the x-transform of the T2 lines of
// R B gives f_hat_RB(kx, ky, kz) on the band; times f_hat_A'(k) (A's spectrum with the
// origin phase exp(2 pi i k.t0/P) folded in, layout [ky][kz][kx]) and summed into
// F[k mod Np].  DIRECT: the fold targets of a thread's outputs are owned by that thread
// (Np / gcd(c, Np) a multiple of TPL and G a multiple of Np), so products accumulate
// straight into acc; otherwise they are staged in Pb[line][kx] and gathered.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int L, bool CPLX, bool DIRECT>
__global__ void __launch_bounds__(8 * Plan<L>::TPL, 512 / (8 * Plan<L>::TPL) > 0 ? 512 / (8 * Plan<L>::TPL) : 1) fold_x_kernel(FoldXArgs a)
{
    constexpr int NL = 8;
    constexpr int TPL = Plan<L>::TPL, NT = NL * TPL;
    constexpr int LS = line_stride(L), E = L / TPL;
    constexpr bool USE_B = Plan<L>::n >= 3;
    extern __shared__ float2 sm[];
    const int K = a.K, M = a.M, Np = a.Np, Kz = a.Kz;
    const int SEG = cm_max_seg(L, a.c, a.G, K);
    const int AS = Np + (Np >> 3) + 1;          // acc row stride; element t at t + t/8 (bank spread)
    float2 *tw = sm;
    float2 *A = tw + L;
    float2 *B = A + NL * LS;
    float2 *acc = B + (USE_B ? NL * LS : 0);    // [NL][AS]
    float2 *ctw = acc + NL * AS;                // [c][L] coset twiddles
    float2 *As = ctw + a.c * L;                 // [2][NL][SEG] A'' segments (cp.async double buffer)
    int *tab = (int *)(As + 2 * NL * SEG);      // [c][L]: segment position | target << 16, or -1
    int2 *segs = (int2 *)(tab + a.c * L);       // [c] (offset, entries)
    float2 *Pb = (float2 *)(segs + 8);          // [NL][M] (gather path only)
    const int line = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const int b = blockIdx.y;
    const int ztiles = (a.Fz + NL - 1) / NL;
    const int kyp = blockIdx.x / ztiles;
    const int z0 = (blockIdx.x % ztiles) * NL;
    const float2 *T2 = a.T2 + (long long)b * a.t2_bstride;

    for (int m = threadIdx.x; m < L; m += NT) tw[m] = a.tw[m];
    for (int e = threadIdx.x; e < NL * AS; e += NT) acc[e] = make_float2(0.f, 0.f);
    for (int e = threadIdx.x; e < a.c * L; e += NT) {
        ctw[e] = a.ctw[e];
        tab[e] = a.xtab[e];
    }
    if (threadIdx.x < a.c) segs[threadIdx.x] = a.segs[threadIdx.x];
    __syncthreads();

    const int span = K / Np + 2;
    for (int pass = 0; pass < (CPLX ? 1 : 2); pass++) {
        const int s = pass ? -1 : 1;  // conj pass: target (-k) mod Np
        const int zlo = CPLX ? -K : (pass ? 1 : 0);
        for (int nz = -span; nz <= span; nz++) {
            bool any = false;
            for (int i = 0; i < NL; i++) {
                const int kz = s * (z0 + i) + nz * Np;
                any |= (z0 + i < a.Fz) && kz >= zlo && kz <= K;
            }
            if (!any) continue;
            const int my_kz = s * (z0 + line) + nz * Np;
            const bool my_ok = (z0 + line < a.Fz) && my_kz >= zlo && my_kz <= K;
            for (int ny = -span; ny <= span; ny++) {
                const int ky = s * kyp + ny * Np;
                if (ky < -K || ky > K) continue;
                // A'' rows of this group: [ky][kz(i)]; coset p's segment is contiguous
                // this thread group copies its own line's row segment (16-byte chunks)
                const float2 *arow_g = a.Ahat + ((long long)(ky + K) * Kz + (CPLX ? my_kz + K : my_kz)) * a.MS;
                auto prefetch = [&](int p, int buf) {
                    const int2 sg = segs[p];
                    if (my_ok)
                        for (int ch = tl; 2 * ch < sg.y; ch += TPL)
                            cp_async16(As + (buf * NL + line) * SEG + 2 * ch, arow_g + sg.x + 2 * ch);
                    cp_async_commit();
                };
                prefetch(0, 0);
                // source lines of R B: (ky, kz) for real weights, (-ky, -kz) for complex (f_hat_RB(-k))
                const int kys = CPLX ? -ky : ky;
                float2 x[E];
#pragma unroll
                for (int m = 0; m < E; m++) {
                    const int e = threadIdx.x + NT * m;
                    const int n = e / NL, i = e % NL;
                    const int kz = s * (z0 + i) + nz * Np;
                    float2 v = make_float2(0.f, 0.f);
                    if ((z0 + i < a.Fz) && kz >= zlo && kz <= K)
                        v = T2[((long long)n * M + (kys + K)) * Kz + (CPLX ? (-kz + K) : kz)];
                    x[m] = v;
                }
                __syncthreads();
#pragma unroll
                for (int m = 0; m < E; m++) {
                    const int e = threadIdx.x + NT * m;
                    A[(e % NL) * LS + pad(e / NL)] = x[m];
                }
                __syncthreads();
#pragma unroll
                for (int m = 0; m < E; m++) x[m] = A[line * LS + pad(tl + TPL * m)];
                __syncthreads();
                for (int p = 0; p < a.c; p++) {
                    if (p + 1 < a.c) prefetch(p + 1, (p + 1) & 1);
                    float2 y[E];
#pragma unroll
                    for (int m = 0; m < E; m++) y[m] = p ? cmul(x[m], ctw[p * L + tl + TPL * m]) : x[m];
                    fft_regs<L, -1>(y, A + line * LS, B + line * LS, tw, tl);
                    if (p + 1 < a.c) cp_async_wait<1>(); else cp_async_wait<0>();
                    __syncthreads();
                    const float2 *arow = As + ((p & 1) * NL + line) * SEG;
                    if (my_ok) {
#pragma unroll
                        for (int m = 0; m < E; m++) {
                            const int t = tab[p * L + tl + TPL * m];
                            if (t < 0) continue;
                            const float2 av = arow[t & 0xffff];
                            // real: f_hat_A'(k) conj(f_hat_RB(k)); complex: f_hat_A'(k') f_hat_RB(-k'),
                            // k' = (-kx, ky, kz), weights not conjugated (reading C-3)
                            const float2 P = CPLX ? cmul(av, y[m]) : cmulc(av, y[m]);
                            if (DIRECT) {
                                int tt = t >> 16;                        // (kx' mod Np), kx' = +-kx
                                if (s < 0 && tt) tt = Np - tt;           // conj pass: (-kx) mod Np
                                tt += tt >> 3;
                                acc[line * AS + tt] = cadd(acc[line * AS + tt], s > 0 ? P : cconj(P));
                            } else {
                                int kx = a.c * (tl + TPL * m) + p;
                                if (2 * kx > a.G) kx -= a.G;
                                Pb[line * M + (CPLX ? -kx : kx) + K] = P;
                            }
                        }
                    } else if (!DIRECT) {
#pragma unroll
                        for (int m = 0; m < E; m++) {
                            int kx = a.c * (tl + TPL * m) + p;
                            if (2 * kx > a.G) kx -= a.G;
                            if (kx >= -K && kx <= K) Pb[line * M + kx + K] = make_float2(0.f, 0.f);
                        }
                    }
                    __syncthreads();
                }
                if (!DIRECT) {
                    for (int e = threadIdx.x; e < NL * Np; e += NT) {
                        const int i = e / Np, t = e % Np;
                        const int base = s > 0 ? t : (Np - t) % Np;
                        int kx = base - ((base + K) / Np) * Np;  // smallest alias >= -K
                        float2 sum = make_float2(0.f, 0.f);
                        for (; kx <= K; kx += Np) sum = cadd(sum, Pb[i * M + kx + K]);
                        acc[i * AS + t + (t >> 3)] = cadd(acc[i * AS + t + (t >> 3)], s > 0 ? sum : cconj(sum));
                    }
                }
            }
        }
    }
    __syncthreads();
    float2 *F = a.F + (long long)b * a.f_bstride;
    for (int e = threadIdx.x; e < NL * Np; e += NT) {
        const int i = e % NL, t = e / NL;
        if (z0 + i < a.Fz) F[((long long)t * Np + kyp) * a.Fz + z0 + i] = acc[i * AS + t + (t >> 3)];
    }
}

// ============================================================================ band permutation
// out[row][cm(s k)] = in[row][k + K], k in [-K, K]: A's spectrum into the coset-major x order
// of B's plan (s = -1 for complex weights, where the fold reads A'(-k) against RB's line).
// B's x multipliers (natural order, index k + K) are folded in: real weights store
// A'(k) conj(mult(k)) at cm(k); complex weights store A'(k) mult(-k) at cm(-k).
__global__ void permute_cm_kernel(const float2 *__restrict__ in, const float2 *__restrict__ mult,
                                  float2 *__restrict__ out, long long rows, int K, int L, int c, int G, int neg, int MS,
                                  int Kz, double R2)
{
    const int M = 2 * K + 1;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * M) return;
    const long long row = e / M;
    const int k = (int)(e % M) - K;
    float2 v = neg ? cmul(in[e], mult[-k + K]) : cmulc(in[e], mult[k + K]);
    if (R2 > 0) {  // spherical band: zero the modes with |k| > band_radius
        const long long ky = row / Kz - K, kz = (row % Kz) - (Kz == M ? K : 0);
        if ((double)(k * (long long)k + ky * ky + kz * kz) > R2) v = make_float2(0.f, 0.f);
    }
    out[row * MS + cm_of_k(neg ? -k : k, L, c, G, K)] = v;
}

void launch_permute_cm(const float2 *in, const float2 *mult, float2 *out, long long rows, int K, int L, int c, int G,
                       int neg, int MS, int Kz, double band_radius, cudaStream_t s)
{
    const long long n = rows * (2LL * K + 1);
    cudaMemsetAsync(out, 0, sizeof(float2) * rows * MS, s);
    permute_cm_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, mult, out, rows, K, L, c, G, neg, MS, Kz,
                                                                 band_radius > 0 ? band_radius * band_radius : 0.0);
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
__global__ void __launch_bounds__(Plan<L>::TPL * Plan<L>::NL, 512 / (Plan<L>::TPL * Plan<L>::NL)) last_kernel(LastArgs a)
{
    constexpr int TPL = Plan<L>::TPL, NL = Plan<L>::NL, NT = TPL * NL;
    constexpr int LS = line_stride(L), E = L / TPL;
    extern __shared__ float2 sm[];
    float2 *tw = sm;
    float2 *A = tw + L;
    float2 *B = A + NL * LS;
    const int line = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const int b = blockIdx.y;
    const long long lines = (long long)a.N * a.N;
    const long long gline = (long long)blockIdx.x * NL + line;
    const bool valid = gline < lines;

    for (int m = threadIdx.x; m < L; m += NT) tw[m] = a.tw[m];
    const float2 *row = a.in + (long long)b * a.in_bstride + gline * a.Fz;
    float2 x[E];
#pragma unroll
    for (int m = 0; m < E; m++) {
        const int n = tl + TPL * m;
        float2 v = make_float2(0.f, 0.f);
        if (valid) {
            if (!HERM || n < a.Fz)
                v = row[n];
            else
                v = cconj(row[L - n]);
        }
        x[m] = v;
    }
    fft_regs<L, +1>(x, A + line * LS, B + line * LS, tw, tl);

    unsigned long long kmin = ~0ull, kmax = 0ull;
    if (valid) {
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int q = tl + TPL * m;
            if (q >= a.N) continue;
            const float2 v = cscale(x[m], a.scale);
            const long long gidx = gline * a.N + q;
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
    return sizeof(float2) * ((size_t)L + 2 * (size_t)Plan<L>::NL * line_stride(L) + extra_f2);
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

template <int L, int SIGN, int IN_MODE, int OUT_MODE>
static void pass_launch(const PassArgs &a, int batch, cudaStream_t s)
{
    constexpr int NL = Plan<L>::NL;
    const size_t sm = fft_smem<L>(OUT_MODE == 0 ? (size_t)NL * a.nk : 0);
    const long long blocks = IN_MODE == 2 ? (long long)a.O * ((a.I + NL - 1) / NL) : (a.lines + NL - 1) / NL;
    set_smem(pass_kernel<L, SIGN, IN_MODE, OUT_MODE>, sm);
    pass_kernel<L, SIGN, IN_MODE, OUT_MODE><<<dim3((unsigned)blocks, batch), Plan<L>::TPL * NL, sm, s>>>(a);
}

// kind: 0 forward contiguous (z), 1 forward strided -> strided (y), 2 forward strided -> rows (x of A),
//       3 inverse strided -> strided
void launch_pass(const PassArgs &a, int kind, int batch, cudaStream_t s)
{
    switch (a.L) {
#define X(L_)                                                                         \
    case L_:                                                                          \
        if (kind == 0) {                                                              \
            if (a.in_real) pass_launch<L_, -1, 0, 0>(a, batch, s);                    \
            else pass_launch<L_, -1, 1, 0>(a, batch, s);                              \
        } else if (kind == 1) pass_launch<L_, -1, 2, 1>(a, batch, s);                 \
        else if (kind == 2) pass_launch<L_, -1, 2, 0>(a, batch, s);                   \
        else pass_launch<L_, 1, 2, 1>(a, batch, s);                                   \
        break;
        BC_FOR_EACH_L(X)
#undef X
    default: break;
    }
}

template <int L, bool CPLX, bool DIRECT>
static void fold_launch(const FoldXArgs &a, dim3 grid, cudaStream_t s)
{
    const size_t sm = sizeof(float2) * ((size_t)L + (Plan<L>::n >= 3 ? 2 : 1) * 8 * (size_t)line_stride(L) +
                                        8 * (size_t)(a.Np + (a.Np >> 3) + 1) + (size_t)a.c * L +
                                        16 * (size_t)cm_max_seg(L, a.c, a.G, a.K) + (DIRECT ? 0 : 8 * (size_t)a.M)) +
                      sizeof(int) * (size_t)a.c * L + sizeof(int2) * 8;
    set_smem(fold_x_kernel<L, CPLX, DIRECT>, sm);
    fold_x_kernel<L, CPLX, DIRECT><<<grid, 8 * Plan<L>::TPL, sm, s>>>(a);
}

void launch_fold_x(const FoldXArgs &a, int batch, cudaStream_t s)
{
    const int ztiles = (a.Fz + 7) / 8;
    dim3 grid((unsigned)(a.Np * ztiles), batch);
    switch (a.L) {
#define X(L_)                                                                                   \
    case L_: {                                                                                  \
        const bool direct = ((a.Np / gcd_int(a.c, a.Np)) % Plan<L_>::TPL) == 0 && (a.G % a.Np) == 0; \
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
        constexpr int NL = Plan<L_>::NL;                                                      \
        const size_t sm = fft_smem<L_>(0);                                                    \
        const long long lines = (long long)a.N * a.N;                                         \
        dim3 grid((unsigned)((lines + NL - 1) / NL), batch);                                  \
        if (a.hermitian) {                                                                    \
            set_smem(last_kernel<L_, true>, sm);                                              \
            last_kernel<L_, true><<<grid, Plan<L_>::TPL * NL, sm, s>>>(a);                    \
        } else {                                                                              \
            set_smem(last_kernel<L_, false>, sm);                                             \
            last_kernel<L_, false><<<grid, Plan<L_>::TPL * NL, sm, s>>>(a);                   \
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
