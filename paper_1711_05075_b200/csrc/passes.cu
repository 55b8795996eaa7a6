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
#include <algorithm>

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
// SIGN > 0 (the inverse passes): one coset, no multipliers, outputs q < nk (every inverse
// launch sets c = 1, klo = 0, unsigned k) -- compile-time here.
template <int L, int SIGN, int IN_MODE, int OUT_MODE>
__global__ void __launch_bounds__(Plan<L>::TPL * Plan<L>::NL, 512 / (Plan<L>::TPL * Plan<L>::NL)) pass_kernel(PassArgs a)
{
    constexpr bool INV = SIGN > 0;
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

    load_twiddles<L>(tw, a.tw, threadIdx.x, NT);
    __syncthreads();  // the table is read across warps (warp-synchronous FFTs do not order it)
    float2 x[E];
    if (IN_MODE == 2) {
        const int pin = a.pitch_in ? a.pitch_in : a.I;
        const float2 *in = (const float2 *)a.in + (long long)b * a.in_bstride + (long long)o * L * pin;
        int ylo = 0, yhi = L - 1;
        if (!INV && a.ylive) {  // live rows of this x plane (block-uniform)
            const float dxl = (float)o - a.zcx;
            const float h2 = a.live_r2 - dxl * dxl;
            ylo = 0;
            yhi = -1;
            if (h2 > 0.f) {
                const float hh = sqrtf(h2);
                ylo = max(0, (int)ceilf(a.zcy - hh));
                yhi = min(L - 1, (int)floorf(a.zcy + hh));
            }
            if (ylo > yhi) {  // plane outside the support cylinder: its band rows are zero
                const int pout = a.pitch_out ? a.pitch_out : a.I;
                float2 *out = a.out + (long long)b * a.out_bstride + (long long)o * a.nk * pout;
                for (int e = threadIdx.x; e < a.nk * NL; e += NT) {
                    const int q = e / NL, i = e % NL;
                    if (i0 + i < a.I) out[(long long)q * pout + i0 + i] = make_float2(0.f, 0.f);
                }
                return;
            }
        }
        // all loads first (E independent loads in flight per thread), then the transpose
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int e = threadIdx.x + NT * m;
            const int n = e / NL, i = e % NL;
            x[m] = (i0 + i < a.I && n >= ylo && n <= yhi) ? in[(long long)n * pin + i0 + i] : make_float2(0.f, 0.f);
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
        bool live = valid;
        if (IN_MODE != 2 && a.zskip) {
            // the tile of this row (spread_z's zero-tile test): unwritten tiles read as zero
            auto zero_tile = [&](long long row) {
                const int X0 = (int)(row / L) & ~3, Y0 = (int)(row % L) & ~3;
                const float dx = fmaxf(fmaxf((float)X0 - a.zcx, a.zcx - (float)(X0 + 3)), 0.f);
                const float dy = fmaxf(fmaxf((float)Y0 - a.zcy, a.zcy - (float)(Y0 + 3)), 0.f);
                return dx * dx + dy * dy > a.zero_r2;
            };
            live = valid && !zero_tile(row0 + line);
            // whole block zero (NL consecutive rows of one x lie in NL / 4 tiles): zero rows out
            if (zero_tile(row0) && zero_tile(row0 + NL - 1) && (NL <= 8 || __syncthreads_and(!live))) {
                if (a.zskip == 2) return;  // the consumer (ylive) never reads these rows
                float2 *outs = a.out + (long long)b * a.out_bstride;
                for (int e = threadIdx.x; e < NL * a.nk; e += NT) {
                    const long long r = row0 + e / a.nk;
                    if (r < nrows) outs[r * a.nk + (e % a.nk)] = make_float2(0.f, 0.f);
                }
                return;
            }
        }
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int n = tl + TPL * m;
            x[m] = make_float2(0.f, 0.f);
            if (live) {
                if (IN_MODE == 0)
                    x[m].x = ((const float *)a.in)[g + n];
                else
                    x[m] = ((const float2 *)a.in)[g + n];
            }
        }
    }

    float2 *outs = a.out + (long long)b * a.out_bstride;
    const int ncos = INV ? 1 : a.c;
    for (int p = 0; p < ncos; p++) {
        float2 y[E];
#pragma unroll
        for (int m = 0; m < E; m++) y[m] = p ? cmul(x[m], a.ctw[p * L + tl + TPL * m]) : x[m];
        fft_regs<L, SIGN, warp_local<L>()>(y, A + line * LS, B + line * LS, tw, tl);
        if (OUT_MODE == 0) {
#pragma unroll
            for (int m = 0; m < E; m++) {
                const int kk = INV ? tl + TPL * m : coset_kk(tl + TPL * m, p, a.c, a.G, a.klo, a.signed_k);
                if (kk >= 0 && kk < a.nk) OUT[line * a.nk + kk] = (!INV && a.mult) ? cmul(y[m], a.mult[kk]) : y[m];
            }
            __syncthreads();
        } else {
            __syncthreads();
#pragma unroll
            for (int m = 0; m < E; m++) A[line * LS + pad(tl + TPL * m)] = y[m];
            __syncthreads();
            const int pout = a.pitch_out ? a.pitch_out : a.I;
            float2 *out = outs + (long long)o * a.nk * pout;
            if (INV) {  // rows q < nk of this block's NL columns: no per-element coset arithmetic
                const int i = threadIdx.x % NL;
                float2 *oc = out + i0 + i;
                if (i0 + i < a.I)
                    for (int q = threadIdx.x / NL; q < a.nk; q += NT / NL) oc[(long long)q * pout] = A[i * LS + pad(q)];
            } else
            for (int e = threadIdx.x; e < L * NL; e += NT) {
                const int q = e / NL, i = e % NL;
                const int kk = coset_kk(q, p, a.c, a.G, a.klo, a.signed_k);
                if (kk >= 0 && kk < a.nk && i0 + i < a.I) {
                    const float2 v = A[i * LS + pad(q)];
                    out[(long long)kk * pout + i0 + i] = a.mult ? cmul(v, a.mult[kk]) : v;
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

// Blocks are ordered rotation-fastest (blockIdx.x = target block * nb + rotation), so the
// nb blocks that read the same A'' rows run together and share them through L2.
// NP > 0: the inverse x-FFT (length NP, same threads per line as L) is fused: the block
// transforms its accumulated k'x lines and writes X1[mx][k'y][k'z] (mx < N) instead of F.
template <int L, int NP, bool CPLX, bool DIRECT>
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
    const int b = blockIdx.x % a.nb;
    const int tb = blockIdx.x / a.nb;
    const int ztiles = (a.Fz + NL - 1) / NL;
    const int kyp = tb / ztiles;
    const int z0 = (tb % ztiles) * NL;
    const float2 *T2 = a.T2 + (long long)b * a.t2_bstride;

    load_twiddles<L>(tw, a.tw, threadIdx.x, NT);
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
    if constexpr (NP > 0) {
        // inverse x: line i = k'z, F[k'x] -> X1[mx][k'y][k'z] for mx < N
        static_assert(Plan<NP>::TPL == TPL && Plan<NP>::n == 2 && NP <= L, "fused inverse plan");
        constexpr int EI = NP / TPL;
        float2 v[EI];
#pragma unroll
        for (int m = 0; m < EI; m++) {
            const int t = tl + TPL * m;
            v[m] = acc[line * AS + t + (t >> 3)];
        }
        load_twiddles<NP>(tw, a.tw_inv, threadIdx.x, NT);
        __syncthreads();
        fft_regs<NP, +1>(v, A + line * LS, B + line * LS, tw, tl);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < EI; m++) A[line * LS + pad(tl + TPL * m)] = v[m];
        __syncthreads();
        float2 *X1 = a.F + (long long)b * a.f_bstride;
        const long long rs = (long long)Np * a.Fz;
        for (int e = threadIdx.x; e < NL * a.N; e += NT) {
            const int i = e % NL, q = e / NL;
            if (z0 + i < a.Fz) X1[(long long)q * rs + (long long)kyp * a.Fz + z0 + i] = A[i * LS + pad(q)];
        }
    } else {
        float2 *F = a.F + (long long)b * a.f_bstride;
        for (int e = threadIdx.x; e < NL * Np; e += NT) {
            const int i = e % NL, t = e / NL;
            if (z0 + i < a.Fz) F[((long long)t * Np + kyp) * a.Fz + z0 + i] = acc[i * AS + t + (t >> 3)];
        }
    }
}

// ============================================================================ band permutation
// out[row][cm(s k)] = in[row][k + K], k in [-K, K]: A's spectrum into the coset-major x order
// of B's plan (s = -1 for complex weights, where the fold reads A'(-k) against RB's line).
// B's x multipliers (natural order, index k + K) are folded in: real weights store
// A'(k) conj(mult(k)) at cm(k); complex weights store A'(k) mult(-k) at cm(-k).
// dec != nullptr: B's radial window deconvolution 1 / phi_hat(|k|) (indexed by |k|^2) is folded in.
// mult_y != nullptr: B's y and z multipliers too -- real weights as conj(mult(ky)) conj(mult(kz))
// (the fold's product A'' conj(B) per mode); complex weights (docking plan, whose fold takes
// A''(ky, kz) times B's line at (-ky, -kz)) as mult(-ky) mult(-kz) -- and the passes skip them.
__global__ void permute_cm_kernel(const float2 *__restrict__ in, const float2 *__restrict__ mult,
                                  float2 *__restrict__ out, long long rows, int K, int L, int c, int G, int neg, int MS,
                                  int Kz, double R2, const float *__restrict__ dec,
                                  const float2 *__restrict__ mult_y, const float2 *__restrict__ mult_z)
{
    const int M = 2 * K + 1;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * M) return;
    const long long row = e / M;
    const int k = (int)(e % M) - K;
    float2 v = neg ? cmul(in[e], mult[-k + K]) : cmulc(in[e], mult[k + K]);
    const long long ky = row / Kz - K, kz = (row % Kz) - (Kz == M ? K : 0);
    const long long k2 = k * (long long)k + ky * ky + kz * kz;
    if (dec) v = cscale(v, dec[k2]);
    if (mult_y)  // the y / z passes skip theirs (real: conj at k; complex, docking fold: at -k)
        v = neg ? cmul(cmul(v, mult_y[-ky + K]), mult_z[-kz + K]) : cmulc(cmulc(v, mult_y[ky + K]), mult_z[kz]);
    if (R2 > 0 && (double)k2 > R2) v = make_float2(0.f, 0.f);  // spherical band: |k| <= band_radius
    out[row * MS + cm_of_k(neg ? -k : k, L, c, G, K)] = v;
}

void launch_permute_cm(const float2 *in, const float2 *mult, float2 *out, long long rows, int K, int L, int c, int G,
                       int neg, int MS, int Kz, double band_radius, const float *dec, cudaStream_t s,
                       const float2 *mult_y, const float2 *mult_z)
{
    const long long n = rows * (2LL * K + 1);
    cudaMemsetAsync(out, 0, sizeof(float2) * rows * MS, s);
    permute_cm_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, mult, out, rows, K, L, c, G, neg, MS, Kz,
                                                                 band_radius > 0 ? band_radius * band_radius : 0.0, dec,
                                                                 mult_y, mult_z);
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

// HERM (real weights, C2R): the lines are taken in pairs (l, l+1) and transformed as one
// complex line Z = A + i B of their Hermitian-expanded spectra, so Re z = a and Im z = b
// (the imaginary parts of the DC and Nyquist modes are dropped, as a C2R transform does).
// The block walks tiles of NL units (line pairs, or single lines for C2C) grid-stride and
// reduces its keys in registers / shared memory before one atomic per kind.
template <int L, bool HERM>
__global__ void __launch_bounds__(Plan<L>::TPL * Plan<L>::NL, 512 / (Plan<L>::TPL * Plan<L>::NL)) last_kernel(LastArgs a)
{
    constexpr int TPL = Plan<L>::TPL, NL = Plan<L>::NL, NT = TPL * NL;
    constexpr int LS = line_stride(L), E = L / TPL;
    extern __shared__ float2 sm[];
    float2 *tw = sm;
    float2 *A = tw + L;
    float2 *B = A + NL * LS;
    __shared__ unsigned long long red[2][NT / 32];
    const int line = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const int b = blockIdx.y;
    const long long lines = (long long)a.N * a.N;
    const long long units = HERM ? (lines + 1) / 2 : lines;
    const long long ntiles = (units + NL - 1) / NL;
    const bool reduce = a.out_kind != BC_OUT_F_FULL;

    load_twiddles<L>(tw, a.tw, threadIdx.x, NT);
    __syncthreads();
    constexpr bool WS = warp_local<L>();
    // running extrema of this thread: values in fp32 with their linear index; a thread visits
    // its outputs in increasing index order, so strict comparisons keep the lowest index on
    // ties, as the 64-bit keys (built once at the end) do across threads
    float vmin = INFINITY, vmax = -INFINITY;
    unsigned imin = 0xffffffffu, imax = 0xffffffffu;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long u = tile * NL + line;
        const bool valid = u < units;
        const long long l0 = HERM ? 2 * u : u;
        const bool has1 = HERM && valid && (l0 + 1 < lines);
        const int pitch = a.pitch ? a.pitch : a.Fz;
        const float2 *row = a.in + (long long)b * a.in_bstride + l0 * pitch;
        float2 x[E];
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int n = tl + TPL * m;
            float2 v = make_float2(0.f, 0.f);
            if (valid) {
                if (!HERM) {
                    v = row[n];
                } else {
                    const bool lo = n < a.Fz;
                    const int src = lo ? n : L - n;
                    float2 va = row[src];
                    float2 vb = has1 ? row[pitch + src] : make_float2(0.f, 0.f);
                    if (n == 0 || 2 * n == L) {
                        va.y = 0.f;
                        vb.y = 0.f;
                    } else if (!lo) {
                        va.y = -va.y;
                        vb.y = -vb.y;
                    }
                    v = make_float2(va.x - vb.y, va.y + vb.x);  // A + i B
                }
            }
            x[m] = v;
        }
        fft_regs<L, +1, WS>(x, A + line * LS, B + line * LS, tw, tl);

        if (valid) {
#pragma unroll
            for (int m = 0; m < E; m++) {
                const int q = tl + TPL * m;
                if (q >= a.N) continue;
                const float2 v = cscale(x[m], a.scale);
                const long long gidx = l0 * a.N + q;
                if (!reduce) {
                    if (HERM) {
                        float *o = (float *)a.out_full + (long long)b * a.full_bstride + gidx;
                        o[0] = v.x;
                        if (has1) o[a.N] = v.y;
                    } else {
                        ((float2 *)a.out_full)[(long long)b * a.full_bstride + gidx] = v;
                    }
                } else {
                    const unsigned gi = (unsigned)gidx;
                    if (v.x < vmin) { vmin = v.x; imin = gi; }
                    if (v.x > vmax) { vmax = v.x; imax = gi; }
                }
            }
            if (HERM && has1 && reduce) {  // line l0 + 1: indices above all of line l0's
#pragma unroll
                for (int m = 0; m < E; m++) {
                    const int q = tl + TPL * m;
                    if (q >= a.N) continue;
                    const float vy = x[m].y * a.scale;
                    const unsigned gi = (unsigned)((l0 + 1) * a.N + q);
                    if (vy < vmin) { vmin = vy; imin = gi; }
                    if (vy > vmax) { vmax = vy; imax = gi; }
                }
            }
        }
        line_sync<WS>();  // the next tile's first FFT stage rewrites this line's A
    }
    unsigned long long kmin = imin != 0xffffffffu ? key_min(vmin, imin) : ~0ull;
    unsigned long long kmax = imax != 0xffffffffu ? key_max(vmax, imax) : 0ull;
    if (reduce) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o1 = __shfl_xor_sync(0xffffffffu, kmin, off);
            const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, kmax, off);
            kmin = o1 < kmin ? o1 : kmin;
            kmax = o2 > kmax ? o2 : kmax;
        }
        if ((threadIdx.x & 31) == 0) {
            red[0][threadIdx.x >> 5] = kmin;
            red[1][threadIdx.x >> 5] = kmax;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < NT / 32; w++) {
                kmin = red[0][w] < kmin ? red[0][w] : kmin;
                kmax = red[1][w] > kmax ? red[1][w] : kmax;
            }
            if (kmin != ~0ull) atomicMin(&a.keys[2 * b + 0], kmin);
            if (kmax != 0ull) atomicMax(&a.keys[2 * b + 1], kmax);
        }
    }
}

// ---------------------------------------------------------------- TMA-fed variant (real weights)
// Same arithmetic as last_kernel<L, true>; the 2 NL rows of a tile are contiguous in Y1, so
// one thread arms an mbarrier with the byte count and issues a 1D bulk copy
// (cp.async.bulk ... mbarrier::complete_tx) of the NEXT tile into the other half of a
// double buffer while the block transforms the current one from shared memory.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int L, bool NFULL>  // NFULL: N = L output rows (compile-time loop bounds)
__global__ void __launch_bounds__(Plan<L>::TPL * Plan<L>::NL, 512 / (Plan<L>::TPL * Plan<L>::NL)) last_tma_kernel(LastArgs a)
{
    constexpr int TPL = Plan<L>::TPL, NL = Plan<L>::NL, NT = TPL * NL;
    constexpr int LS = line_stride(L), E = L / TPL;
    constexpr bool WS = warp_local<L>();
    extern __shared__ __align__(16) float2 sm[];
    constexpr int Fz = L / 2 + 1;  // Hermitian rows (launch_last takes this kernel only then)
    const int Pz = a.pitch ? a.pitch : a.Fz;  // row pitch
    float2 *stage = sm;                          // [2][2 NL][Pz]
    float2 *tw = stage + 2 * 2 * NL * Pz;
    float2 *A = tw + L;
    float2 *B = A + NL * LS;
    __shared__ unsigned long long bar[2];
    __shared__ unsigned long long red[2][NT / 32];
    const int line = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const int b = blockIdx.y;
    const int Nn = NFULL ? L : a.N;  // output rows
    const long long lines = (long long)Nn * Nn;
    const long long ntiles = (lines + 2 * NL - 1) / (2 * NL);
    const bool reduce = a.out_kind != BC_OUT_F_FULL;
    const float2 *in = a.in + (long long)b * a.in_bstride;

    auto issue = [&](long long tile, int s) {  // one thread: arm + copy tile -> stage s
        const long long l0 = tile * 2 * NL;
        const long long nl = lines - l0 < 2 * NL ? lines - l0 : 2 * NL;
        const unsigned bytes = (unsigned)(nl * Pz * sizeof(float2));
        mbar_expect_tx(&bar[s], bytes);
        bulk_g2s(stage + (size_t)s * 2 * NL * Pz, in + l0 * Pz, bytes, &bar[s]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    load_twiddles<L>(tw, a.tw, threadIdx.x, NT);
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < ntiles) issue(blockIdx.x, 0);

    float vmin = INFINITY, vmax = -INFINITY;
    unsigned imin = 0xffffffffu, imax = 0xffffffffu;
    int it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
        const int s = it & 1;
        if (threadIdx.x == 0 && tile + gridDim.x < ntiles) issue(tile + gridDim.x, s ^ 1);
        mbar_wait(&bar[s], (it >> 1) & 1);
        const float2 *st = stage + (size_t)s * 2 * NL * Pz;
        const long long l0 = tile * 2 * NL + 2 * line;
        const bool valid = l0 < lines;
        const bool has1 = l0 + 1 < lines;
        const float2 *ra = st + (2 * line) * Pz, *rb = ra + Pz;
        float2 x[E];
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int n = tl + TPL * m;
            float2 v = make_float2(0.f, 0.f);
            if (valid) {
                const bool lo = n < Fz;
                const int src = lo ? n : L - n;
                float2 va = ra[src];
                float2 vb = has1 ? rb[src] : make_float2(0.f, 0.f);
                if (n == 0 || 2 * n == L) {
                    va.y = 0.f;
                    vb.y = 0.f;
                } else if (!lo) {
                    va.y = -va.y;
                    vb.y = -vb.y;
                }
                v = make_float2(va.x - vb.y, va.y + vb.x);  // A + i B
            }
            x[m] = v;
        }
        fft_regs<L, +1, WS>(x, A + line * LS, B + line * LS, tw, tl);
        if (valid) {
#pragma unroll
            for (int m = 0; m < E; m++) {
                const int q = tl + TPL * m;
                if (!NFULL && q >= Nn) continue;
                const float2 v = cscale(x[m], a.scale);
                const long long gidx = l0 * Nn + q;
                if (!reduce) {
                    float *o = (float *)a.out_full + (long long)b * a.full_bstride + gidx;
                    o[0] = v.x;
                    if (has1) o[Nn] = v.y;
                } else {
                    const unsigned gi = (unsigned)gidx;
                    if (v.x < vmin) { vmin = v.x; imin = gi; }
                    if (v.x > vmax) { vmax = v.x; imax = gi; }
                }
            }
            if (has1 && reduce) {
#pragma unroll
                for (int m = 0; m < E; m++) {
                    const int q = tl + TPL * m;
                    if (!NFULL && q >= Nn) continue;
                    const float vy = x[m].y * a.scale;
                    const unsigned gi = (unsigned)((l0 + 1) * Nn + q);
                    if (vy < vmin) { vmin = vy; imin = gi; }
                    if (vy > vmax) { vmax = vy; imax = gi; }
                }
            }
        }
        __syncthreads();  // stage s fully read (it is refilled next iteration); FFT buffers free
    }
    unsigned long long kmin = imin != 0xffffffffu ? key_min(vmin, imin) : ~0ull;
    unsigned long long kmax = imax != 0xffffffffu ? key_max(vmax, imax) : 0ull;
    if (reduce) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o1 = __shfl_xor_sync(0xffffffffu, kmin, off);
            const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, kmax, off);
            kmin = o1 < kmin ? o1 : kmin;
            kmax = o2 > kmax ? o2 : kmax;
        }
        if ((threadIdx.x & 31) == 0) {
            red[0][threadIdx.x >> 5] = kmin;
            red[1][threadIdx.x >> 5] = kmax;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < NT / 32; w++) {
                kmin = red[0][w] < kmin ? red[0][w] : kmin;
                kmax = red[1][w] > kmax ? red[1][w] : kmax;
            }
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

template <int L, int NP, bool CPLX, bool DIRECT>
static void fold_launch(const FoldXArgs &a, dim3 grid, cudaStream_t s)
{
    const size_t sm = sizeof(float2) * ((size_t)L + (Plan<L>::n >= 3 ? 2 : 1) * 8 * (size_t)line_stride(L) +
                                        8 * (size_t)(a.Np + (a.Np >> 3) + 1) + (size_t)a.c * L +
                                        16 * (size_t)cm_max_seg(L, a.c, a.G, a.K) + (DIRECT ? 0 : 8 * (size_t)a.M)) +
                      sizeof(int) * (size_t)a.c * L + sizeof(int2) * 8;
    set_smem(fold_x_kernel<L, NP, CPLX, DIRECT>, sm);
    fold_x_kernel<L, NP, CPLX, DIRECT><<<grid, 8 * Plan<L>::TPL, sm, s>>>(a);
}

bool fold_fuses_inverse(int L, int Np) { return L == 256 && Np == 256; }

void launch_fold_x(const FoldXArgs &a_in, int batch, cudaStream_t s)
{
    FoldXArgs a = a_in;
    a.nb = batch;
    const int ztiles = (a.Fz + 7) / 8;
    dim3 grid((unsigned)(a.Np * ztiles * batch), 1);
    if (a.fuse_inv && fold_fuses_inverse(a.L, a.Np)) {
        const bool direct = ((a.Np / gcd_int(a.c, a.Np)) % Plan<256>::TPL) == 0 && (a.G % a.Np) == 0;
        if (a.complex_w) {
            if (direct) fold_launch<256, 256, true, true>(a, grid, s);
            else fold_launch<256, 256, true, false>(a, grid, s);
        } else {
            if (direct) fold_launch<256, 256, false, true>(a, grid, s);
            else fold_launch<256, 256, false, false>(a, grid, s);
        }
        return;
    }
    switch (a.L) {
#define X(L_)                                                                                   \
    case L_: {                                                                                  \
        const bool direct = ((a.Np / gcd_int(a.c, a.Np)) % Plan<L_>::TPL) == 0 && (a.G % a.Np) == 0; \
        if (a.complex_w) {                                                                      \
            if (direct) fold_launch<L_, 0, true, true>(a, grid, s);                             \
            else fold_launch<L_, 0, true, false>(a, grid, s);                                   \
        } else {                                                                                \
            if (direct) fold_launch<L_, 0, false, true>(a, grid, s);                            \
            else fold_launch<L_, 0, false, false>(a, grid, s);                                  \
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
    // TMA-fed C2R path: the tile rows must be 16-byte aligned (the stage offsets and
    // the row blocks are multiples of 2 NL rows; Fz * 8 bytes per row)
    // every row (not only every full tile): a ragged last tile of an odd number of rows must
    // still copy a multiple of 16 bytes (cp.async.bulk size rule and the expect_tx count)
    if (a.hermitian && a.Np == 256 && ((uintptr_t)a.in % 16) == 0 && (a.in_bstride * 8) % 16 == 0 &&
        ((a.pitch ? a.pitch : a.Fz) * 8) % 16 == 0) {
        constexpr int NL = Plan<256>::NL;
        const size_t sm = sizeof(float2) * (2 * 2 * NL * (size_t)(a.pitch ? a.pitch : a.Fz) + 256 +
                                            (Plan<256>::n >= 3 ? 2 : 1) * (size_t)NL * line_stride(256));
        const long long lines = (long long)a.N * a.N;
        const long long tiles = (lines + 2 * NL - 1) / (2 * NL);
        const long long cap = std::max(1LL, 4LL * 148 * 4 / std::max(batch, 1));
        if (a.N == 256) {
            set_smem(last_tma_kernel<256, true>, sm);
            last_tma_kernel<256, true><<<dim3((unsigned)std::min(tiles, cap), batch), Plan<256>::TPL * NL, sm, s>>>(a);
        } else {
            set_smem(last_tma_kernel<256, false>, sm);
            last_tma_kernel<256, false><<<dim3((unsigned)std::min(tiles, cap), batch), Plan<256>::TPL * NL, sm, s>>>(a);
        }
        return;
    }
    switch (a.Np) {
#define X(L_)                                                                                 \
    case L_: {                                                                                \
        constexpr int NL = Plan<L_>::NL;                                                      \
        const size_t sm = fft_smem<L_>(0);                                                    \
        const long long lines = (long long)a.N * a.N;                                         \
        const long long units = a.hermitian ? (lines + 1) / 2 : lines;                        \
        const long long tiles = (units + NL - 1) / NL;                                        \
        const long long cap = std::max(1LL, 4LL * 148 * 4 / std::max(batch, 1));             \
        dim3 grid((unsigned)std::min(tiles, cap), batch);                                     \
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

__global__ void keys_finalize_kernel(const unsigned long long *keys, int batch, int kind, bc_extremum *out,
                                     ResultPeers peers)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= batch) return;
    const unsigned long long kmin = keys[2 * r], kmax = keys[2 * r + 1];
    bc_extremum emin, emax;
    emin.val = (double)float_from_order_bits((uint32_t)(kmin >> 32));
    emin.idx = (int64_t)(kmin & 0xffffffffull);
    emax.val = (double)float_from_order_bits((uint32_t)(kmax >> 32));
    emax.idx = (int64_t)(0xffffffffull - (kmax & 0xffffffffull));
    const int per = kind == BC_OUT_MINMAX ? 2 : 1;
    const bc_extremum e0 = kind == BC_OUT_MAX_ARGMAX || kind == BC_OUT_MAX_REAL ? emax : emin;
    out[per * r] = e0;
    if (per == 2) out[2 * r + 1] = emax;
    // fused result exchange (collectives.cu): the same records into every peer's buffer at the
    // rotation's global index -- NVLink stores instead of an all-gather after the step
    for (int p = 0; p < peers.n; p++) {
        bc_extremum *o = (bc_extremum *)peers.buf[p] + per * (peers.base + r);
        o[0] = e0;
        if (per == 2) o[1] = emax;
    }
    if (peers.n) __threadfence_system();
}

void launch_keys_finalize(const unsigned long long *keys, int batch, int out_kind, void *out, const ResultPeers &peers,
                          cudaStream_t s)
{
    keys_finalize_kernel<<<(batch + 127) / 128, 128, 0, s>>>(keys, batch, out_kind, (bc_extremum *)out, peers);
}
