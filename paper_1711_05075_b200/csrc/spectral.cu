// spectral.cu -- the Fourier-route kernels of libballcorr (sm_100a).
//
// Per rotation (eq_ccghat):
//   spread      rho_s = (sum_j v_j 1_{B(R b_j, s_j)}) * G_tau on a fine box  (eq_rhoAtrans, eq_ballconv)
//   axis z,y,x  box DFT on the band, times hf exp(-2 pi i k o / G) exp(+2 pi^2 tau^2 k^2 / P^2)
//               => f_hat_RB(k / P) = sum_j v_j beta_hat(s_j, |k|/P) exp(-2 pi i k.R b_j / P)  (eq_fballhat)
//   fold        F[k mod Np] += f_hat_A(k/P) f_hat_RB(-k/P) exp(2 pi i k.t0 / P)         (eq_ccghat)
//   inverse     f(t0 + m h) = (1/P^3) sum_k' F[k'] exp(2 pi i k'.m / Np), m in [0, N)^3  (L829-L833)
//   reduce      per-rotation min / max (argmin / argmax, lowest index on ties)
#include "kernels.cuh"

#include "ballcorr.h"

#define SP_T 16
#define MAXPER 16

// ============================================================================ spreading

// (1_{B(0,s)} * G_tau)(d) with G_tau the unit-mass isotropic 3D Gaussian of sd tau:
//   1/2 [erf((s-d)/(sqrt2 tau)) + erf((s+d)/(sqrt2 tau))]
//     - tau / (d sqrt(2 pi)) [exp(-(s-d)^2 / 2tau^2) - exp(-(s+d)^2 / 2tau^2)]
// evaluated without cancellation (erfc in the tail, sinh(x)/x series near d = 0).
__device__ __forceinline__ float smoothed_ball(float s, float d, float tau)
{
    const float inv_sqrt2 = 0.70710678118654752440f;
    const float inv_sqrt2pi = 0.39894228040143267794f;
    const float it = 1.0f / tau;
    const float a = (s - d) * it * inv_sqrt2, b = (s + d) * it * inv_sqrt2;
    const float t1 = (a >= 0.0f) ? 0.5f * (erff(a) + erff(b)) : 0.5f * (erfcf(-a) - erfcf(b));
    const float x = s * d * it * it;
    float t2;
    if (x < 1.0f) {
        const float x2 = x * x;
        const float shc = 1.0f + x2 * (1.0f / 6.0f + x2 * (1.0f / 120.0f + x2 * (1.0f / 5040.0f)));
        t2 = 2.0f * s * it * inv_sqrt2pi * expf(-0.5f * (s * s + d * d) * it * it) * shc;
    } else {
        const float em = expf(-0.5f * (s - d) * (s - d) * it * it);
        const float ep = expf(-0.5f * (s + d) * (s + d) * it * it);
        t2 = tau / d * inv_sqrt2pi * (em - ep);
    }
    return t1 - t2;
}

template <bool CPLX>
__global__ void __launch_bounds__(256) spread_kernel(SpreadArgs a)
{
    __shared__ float4 sb[256];
    __shared__ float4 sw[256];
    __shared__ int wcount[8];

    const int b = blockIdx.y;
    const int tile = blockIdx.x;
    const int tpa = a.tiles_per_axis;
    const int tz = tile % tpa, ty = (tile / tpa) % tpa, tx = tile / (tpa * tpa);
    const int X0 = tx * SP_T, Y0 = ty * SP_T, Z0 = tz * SP_T;
    const int x = X0 + (threadIdx.x >> 4), y = Y0 + (threadIdx.x & 15);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

    float R[9];
    if (a.rot) {
#pragma unroll
        for (int q = 0; q < 9; q++) R[q] = a.rot[9 * b + q];
    }

    float accr[SP_T], acci[SP_T];
#pragma unroll
    for (int z = 0; z < SP_T; z++) {
        accr[z] = 0.f;
        acci[z] = 0.f;
    }

    int c0 = 0, ncand = a.n_balls;
    if (a.csr_off) {
        c0 = a.csr_off[tile];
        ncand = a.csr_off[tile + 1] - c0;
    }
    const float fx0 = (float)X0, fy0 = (float)Y0, fz0 = (float)Z0, fe = (float)(SP_T - 1);

    for (int base = 0; base < ncand; base += 256) {
        const int q = base + threadIdx.x;
        bool ok = false;
        float4 u = make_float4(0, 0, 0, 0), wv = make_float4(0, 0, 0, 0);
        if (q < ncand) {
            const int j = a.csr_idx ? a.csr_idx[c0 + q] : q;
            const float4 bl = a.balls[j];
            float cx = bl.x, cy = bl.y, cz = bl.z;
            if (a.rot) {  // eq_Mink0 (L235): a rigid motion relocates the centre only
                cx = R[0] * bl.x + R[1] * bl.y + R[2] * bl.z;
                cy = R[3] * bl.x + R[4] * bl.y + R[5] * bl.z;
                cz = R[6] * bl.x + R[7] * bl.y + R[8] * bl.z;
            }
            u.x = cx * a.inv_hf - (float)a.ox;
            u.y = cy * a.inv_hf - (float)a.oy;
            u.z = cz * a.inv_hf - (float)a.oz;
            u.w = (bl.w + a.cut) * a.inv_hf;
            const float dx = fmaxf(fmaxf(fx0 - u.x, u.x - (fx0 + fe)), 0.f);
            const float dy = fmaxf(fmaxf(fy0 - u.y, u.y - (fy0 + fe)), 0.f);
            const float dz = fmaxf(fmaxf(fz0 - u.z, u.z - (fz0 + fe)), 0.f);
            ok = dx * dx + dy * dy + dz * dz < u.w * u.w;
            if (ok) {
                wv.x = bl.w;
                wv.y = a.w_re ? a.w_re[j] : 1.f;
                wv.z = (CPLX && a.w_im) ? a.w_im[j] : 0.f;
            }
        }
        // order-preserving compaction (deterministic summation order)
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) wcount[wid] = __popc(m);
        __syncthreads();
        int off = 0, total = 0;
#pragma unroll
        for (int w = 0; w < 8; w++) {
            const int cw = wcount[w];
            off += (w < wid) ? cw : 0;
            total += cw;
        }
        if (ok) {
            const int pos = off + __popc(m & ((1u << lane) - 1u));
            sb[pos] = u;
            sw[pos] = wv;
        }
        __syncthreads();
        for (int e = 0; e < total; e++) {
            const float4 ue = sb[e];
            const float dx = (float)x - ue.x, dy = (float)y - ue.y;
            const float dxy2 = dx * dx + dy * dy;
            const float rc2 = ue.w * ue.w;
            if (dxy2 < rc2) {
                const float4 we = sw[e];
#pragma unroll
                for (int z = 0; z < SP_T; z++) {
                    const float dz = (fz0 + (float)z) - ue.z;
                    const float d2 = dxy2 + dz * dz;
                    if (d2 < rc2) {
                        const float g = smoothed_ball(we.x, sqrtf(d2) * a.hf, a.tau);
                        accr[z] += we.y * g;
                        if (CPLX) acci[z] += we.z * g;
                    }
                }
            }
        }
        __syncthreads();
    }

    const int L = a.L;
    if (x < L && y < L) {
        const long long rowoff = (long long)b * a.out_batch_stride + ((long long)x * L + y) * L;
        if (CPLX) {
            float2 *o = (float2 *)a.out + rowoff;
#pragma unroll
            for (int z = 0; z < SP_T; z++)
                if (Z0 + z < L) o[Z0 + z] = make_float2(accr[z], acci[z]);
        } else {
            float *o = (float *)a.out + rowoff;
#pragma unroll
            for (int z = 0; z < SP_T; z++)
                if (Z0 + z < L) o[Z0 + z] = accr[z];
        }
    }
}

void launch_spread(const SpreadArgs &a, int batch, cudaStream_t s)
{
    const int tpa = a.tiles_per_axis;
    dim3 grid(tpa * tpa * tpa, batch);
    if (a.complex_w)
        spread_kernel<true><<<grid, 256, 0, s>>>(a);
    else
        spread_kernel<false><<<grid, 256, 0, s>>>(a);
}

// ============================================================================ axis transforms

__device__ __forceinline__ int coset_k(const AxisArgs &a, int q, int p)
{
    const int G = a.c * a.L;
    int k = a.c * q + p;
    if (a.signed_k && 2 * k > G) k -= G;
    return k - a.klo;
}

__device__ __forceinline__ float2 coset_twiddle(int p, int n, int G, float sign)
{
    float2 e = expi_frac((long long)p * n, G);
    e.y *= sign;
    return e;
}

// Lines contiguous in memory: in[b][line][L] -> out[b][line][nk].
__global__ void __launch_bounds__(256) axis_contig_kernel(AxisArgs a, int lines, int TL)
{
    extern __shared__ float2 sm[];
    const int L = a.L, ld = TL + 1, G = a.c * L;
    float2 *bufA = sm;
    float2 *bufB = bufA + L * ld;
    float2 *tw = bufB + L * ld;
    float2 *stage = tw + L;
    const int b = blockIdx.y;
    const long long line0 = (long long)blockIdx.x * TL;
    const int tid = threadIdx.x;

    fft_twiddles(tw, L, a.sign);

    float2 x[MAXPER];
    const int total = TL * L;
#pragma unroll
    for (int m = 0; m < MAXPER; m++) {
        const int e = tid + 256 * m;
        x[m] = make_float2(0.f, 0.f);
        if (e < total) {
            const int line = e / L, n = e % L;
            if (line0 + line < lines) {
                const long long gi = (long long)b * a.in_bstride + (line0 + line) * L + n;
                if (a.in_real)
                    x[m].x = ((const float *)a.in)[gi];
                else
                    x[m] = ((const float2 *)a.in)[gi];
            }
        }
    }
    for (int p = 0; p < a.c; p++) {
#pragma unroll
        for (int m = 0; m < MAXPER; m++) {
            const int e = tid + 256 * m;
            if (e < total) {
                const int line = e / L, n = e % L;
                bufA[n * ld + line] = (p == 0) ? x[m] : cmul(x[m], coset_twiddle(p, n, G, a.sign));
            }
        }
        __syncthreads();
        const float2 *res = block_fft(bufA, bufB, tw, a.plan, TL, ld, a.sign);
        for (int it = tid; it < total; it += 256) {
            const int line = it / L, q = it % L;
            const int kk = coset_k(a, q, p);
            if (kk >= 0 && kk < a.nk) {
                float2 v = res[q * ld + line];
                if (a.mult) v = cmul(v, a.mult[kk]);
                stage[line * a.nk + kk] = v;
            }
        }
        __syncthreads();
    }
    const int tot_out = TL * a.nk;
    for (int it = tid; it < tot_out; it += 256) {
        const int line = it / a.nk, kk = it % a.nk;
        if (line0 + line < lines)
            a.out[(long long)b * a.out_bstride + (line0 + line) * a.nk + kk] = stage[it];
    }
}

// Lines strided: in[b][O][L][I] -> out[b][O][nk][I]; a block owns TI consecutive i.
__global__ void __launch_bounds__(256) axis_strided_kernel(AxisArgs a, int TI)
{
    extern __shared__ float2 sm[];
    const int L = a.L, ld = TI + 1, G = a.c * L;
    float2 *bufA = sm;
    float2 *bufB = bufA + L * ld;
    float2 *tw = bufB + L * ld;
    const int b = blockIdx.y;
    const int itiles = (a.I + TI - 1) / TI;
    const int o = blockIdx.x / itiles;
    const int i0 = (blockIdx.x % itiles) * TI;
    const int tid = threadIdx.x;
    const float2 *in = (const float2 *)a.in + (long long)b * a.in_bstride + (long long)o * L * a.I;
    float2 *out = a.out + (long long)b * a.out_bstride + (long long)o * a.nk * a.I;

    fft_twiddles(tw, L, a.sign);

    float2 x[MAXPER];
    const int total = TI * L;
#pragma unroll
    for (int m = 0; m < MAXPER; m++) {
        const int e = tid + 256 * m;
        x[m] = make_float2(0.f, 0.f);
        if (e < total) {
            const int n = e / TI, i = e % TI;
            if (i0 + i < a.I) x[m] = in[(long long)n * a.I + i0 + i];
        }
    }
    for (int p = 0; p < a.c; p++) {
#pragma unroll
        for (int m = 0; m < MAXPER; m++) {
            const int e = tid + 256 * m;
            if (e < total) {
                const int n = e / TI, i = e % TI;
                bufA[n * ld + i] = (p == 0) ? x[m] : cmul(x[m], coset_twiddle(p, n, G, a.sign));
            }
        }
        __syncthreads();
        const float2 *res = block_fft(bufA, bufB, tw, a.plan, TI, ld, a.sign);
        for (int it = tid; it < total; it += 256) {
            const int q = it / TI, i = it % TI;
            const int kk = coset_k(a, q, p);
            if (kk >= 0 && kk < a.nk && i0 + i < a.I) {
                float2 v = res[q * ld + i];
                if (a.mult) v = cmul(v, a.mult[kk]);
                out[(long long)kk * a.I + i0 + i] = v;
            }
        }
        __syncthreads();
    }
}

static int pick_tl(int L) { return L <= 512 ? 8 : 4; }

void launch_axis_contig(const AxisArgs &a, int lines, int batch, cudaStream_t s)
{
    const int TL = pick_tl(a.L);
    const size_t smem = sizeof(float2) * ((size_t)2 * a.L * (TL + 1) + a.L + (size_t)TL * a.nk);
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(axis_contig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = 200 * 1024;
    }
    dim3 grid((lines + TL - 1) / TL, batch);
    axis_contig_kernel<<<grid, 256, smem, s>>>(a, lines, TL);
}

void launch_axis_strided(const AxisArgs &a, int batch, cudaStream_t s)
{
    const int TI = pick_tl(a.L);
    const size_t smem = sizeof(float2) * ((size_t)2 * a.L * (TI + 1) + a.L);
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(axis_strided_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = 200 * 1024;
    }
    const int itiles = (a.I + TI - 1) / TI;
    dim3 grid(a.O * itiles, batch);
    axis_strided_kernel<<<grid, 256, smem, s>>>(a, TI);
}

// ============================================================================ product + fold

// first n with base + n*Np >= lo
__device__ __forceinline__ int first_alias(int base, int lo, int Np)
{
    int d = lo - base;
    return d <= 0 ? -((-d) / Np) : (d + Np - 1) / Np;
}

__global__ void __launch_bounds__(256) fold_kernel(FoldArgs a)
{
    const int b = blockIdx.y;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long ntarget = (long long)a.Np * a.Np * a.Fz;
    if (t >= ntarget) return;
    const int kzp = (int)(t % a.Fz);
    const int kyp = (int)((t / a.Fz) % a.Np);
    const int kxp = (int)(t / ((long long)a.Fz * a.Np));
    const int K = a.K, M = 2 * K + 1, Np = a.Np;
    const float2 *Bh = a.Bhat + (long long)b * a.b_bstride;
    float2 acc = make_float2(0.f, 0.f);

    if (!a.complex_w) {
        // stored kz in [0, K]; a mode with kz < 0 is the conjugate of the stored -k
        for (int pass = 0; pass < 2; pass++) {
            const int bx = pass ? -kxp : kxp, by = pass ? -kyp : kyp, bz = pass ? -kzp : kzp;
            const int zlo = pass ? 1 : 0;
            float2 part = make_float2(0.f, 0.f);
            for (int kz = bz + first_alias(bz, zlo, Np) * Np; kz <= K; kz += Np)
                for (int ky = by + first_alias(by, -K, Np) * Np; ky <= K; ky += Np)
                    for (int kx = bx + first_alias(bx, -K, Np) * Np; kx <= K; kx += Np) {
                        const long long idx = ((long long)(kx + K) * M + (ky + K)) * a.Kz + kz;
                        float2 P = cmulc(a.Ahat[idx], Bh[idx]);  // A conj(B) = f_hat_A(k) f_hat_B(-k)
                        P = cmul(P, cmul(cmul(a.phx[kx + K], a.phy[ky + K]), a.phz[kz + K]));
                        part = cadd(part, P);
                    }
            acc = cadd(acc, pass ? cconj(part) : part);
        }
    } else {
        for (int kz = kzp + first_alias(kzp, -K, Np) * Np; kz <= K; kz += Np)
            for (int ky = kyp + first_alias(kyp, -K, Np) * Np; ky <= K; ky += Np)
                for (int kx = kxp + first_alias(kxp, -K, Np) * Np; kx <= K; kx += Np) {
                    const long long idx = ((long long)(kx + K) * M + (ky + K)) * a.Kz + (kz + K);
                    const long long nidx = ((long long)(-kx + K) * M + (-ky + K)) * a.Kz + (-kz + K);
                    float2 P = cmul(a.Ahat[idx], Bh[nidx]);  // f_hat_A(k) f_hat_B(-k), weights not conjugated (C-3)
                    P = cmul(P, cmul(cmul(a.phx[kx + K], a.phy[ky + K]), a.phz[kz + K]));
                    acc = cadd(acc, P);
                }
    }
    a.F[(long long)b * a.f_bstride + t] = acc;
}

void launch_fold(const FoldArgs &a, int batch, cudaStream_t s)
{
    const long long n = (long long)a.Np * a.Np * a.Fz;
    dim3 grid((unsigned)((n + 255) / 256), batch);
    fold_kernel<<<grid, 256, 0, s>>>(a);
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

__global__ void __launch_bounds__(256) last_kernel(LastArgs a, int TL)
{
    extern __shared__ float2 sm[];
    const int L = a.Np, ld = TL + 1;
    float2 *bufA = sm;
    float2 *bufB = bufA + L * ld;
    float2 *tw = bufB + L * ld;
    const int b = blockIdx.y;
    const long long lines = (long long)a.N * a.N;
    const long long line0 = (long long)blockIdx.x * TL;
    const int tid = threadIdx.x;
    const float2 *in = a.in + (long long)b * a.in_bstride;

    fft_twiddles(tw, L, 1.0f);
    // load (and Hermitian-expand) TL lines into bufA[n*ld + line]
    for (int e = tid; e < TL * L; e += 256) {
        const int line = e / L, n = e % L;
        float2 v = make_float2(0.f, 0.f);
        if (line0 + line < lines) {
            const float2 *row = in + (line0 + line) * a.Fz;
            if (!a.hermitian)
                v = row[n];
            else if (n < a.Fz)
                v = row[n];
            else
                v = cconj(row[L - n]);
        }
        bufA[n * ld + line] = v;
    }
    __syncthreads();
    const float2 *res = block_fft(bufA, bufB, tw, a.plan, TL, ld, 1.0f);

    unsigned long long kmin = ~0ull, kmax = 0ull;
    const int tot = TL * a.N;
    for (int it = tid; it < tot; it += 256) {
        const int line = it / a.N, m = it % a.N;
        if (line0 + line >= lines) continue;
        const float2 v = cscale(res[m * ld + line], a.scale);
        const long long gidx = (line0 + line) * a.N + m;
        if (a.out_kind == BC_OUT_F_FULL) {
            if (a.hermitian)
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
    if (a.out_kind != BC_OUT_F_FULL) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o1 = __shfl_xor_sync(0xffffffffu, kmin, off);
            const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, kmax, off);
            kmin = o1 < kmin ? o1 : kmin;
            kmax = o2 > kmax ? o2 : kmax;
        }
        if ((tid & 31) == 0) {
            if (kmin != ~0ull) atomicMin(&a.keys[2 * b + 0], kmin);
            if (kmax != 0ull) atomicMax(&a.keys[2 * b + 1], kmax);
        }
    }
}

void launch_last(const LastArgs &a, int batch, cudaStream_t s)
{
    const int TL = pick_tl(a.Np);
    const size_t smem = sizeof(float2) * ((size_t)2 * a.Np * (TL + 1) + a.Np);
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(last_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = 200 * 1024;
    }
    const long long lines = (long long)a.N * a.N;
    dim3 grid((unsigned)((lines + TL - 1) / TL), batch);
    last_kernel<<<grid, 256, smem, s>>>(a, TL);
}

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
