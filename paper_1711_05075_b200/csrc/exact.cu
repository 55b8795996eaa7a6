// exact.cu -- the combinatorial (pair-lens) route of libballcorr.
//
// PAPER.md L343-L360 (eq_ORP, eq_convgP): the translational obstacle of two
// ball sets is the union of obstacle balls centred at a_i - R b_j with radius
// r_i + s_j, and g = rho_{P_O} * f_{B_O} with primitive kernel
// f_{B_O} = f_{B_1} * f_{B_2}.  For indicator primitives that kernel is the
// two-ball intersection volume V(r, s, d), so
//     f_R(t_m) = sum_ij w_i v_j V(r_i, s_j, |a_i - R b_j - t_m|).
// Each (i, j) pair spreads V onto the grid points inside its obstacle ball;
// accumulation is fp64.  This is the paper's "pairwise Minkowski sum" GPU
// kernel (L515-L520), here with exact lens weights.
#include "kernels.cuh"

#include "ballcorr.h"

template <typename T>
__device__ __forceinline__ T lens_volume_dev(T r, T s, T d)
{
    const T pi = (T)3.14159265358979323846;
    if (d >= r + s) return (T)0;
    const T m = r < s ? r : s;
    const T rs = r - s;
    if (d <= (rs < 0 ? -rs : rs)) return (T)4 / (T)3 * pi * m * m * m;
    const T e = r + s - d;
    return pi * e * e * (d * d + (T)2 * d * (r + s) - (T)3 * rs * rs) / ((T)12 * d);
}

template <typename T, bool CPLX>
__global__ void __launch_bounds__(256) exact_kernel(ExactArgs a)
{
    const int b = blockIdx.y;
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= (long long)a.nA * a.nB) return;
    const int i = (int)(p / a.nB), j = (int)(p % a.nB);
    const double *R = a.rot + 9 * b;
    const double4 ai = a.A[i], bj = a.B[j];
    // obstacle knot a_i - R b_j (eq_ORP), radius r_i + s_j
    const double cx = ai.x - (R[0] * bj.x + R[1] * bj.y + R[2] * bj.z);
    const double cy = ai.y - (R[3] * bj.x + R[4] * bj.y + R[5] * bj.z);
    const double cz = ai.z - (R[6] * bj.x + R[7] * bj.y + R[8] * bj.z);
    const double rs = ai.w + bj.w;
    const int N = a.N;
    const double ih = 1.0 / a.h;
    int x0 = (int)ceil((cx - rs - a.t0x) * ih), x1 = (int)floor((cx + rs - a.t0x) * ih);
    int y0 = (int)ceil((cy - rs - a.t0y) * ih), y1 = (int)floor((cy + rs - a.t0y) * ih);
    int z0 = (int)ceil((cz - rs - a.t0z) * ih), z1 = (int)floor((cz + rs - a.t0z) * ih);
    x0 = max(x0, 0); y0 = max(y0, 0); z0 = max(z0, 0);
    x1 = min(x1, N - 1); y1 = min(y1, N - 1); z1 = min(z1, N - 1);
    if (x0 > x1 || y0 > y1 || z0 > z1) return;
    const double2 wa = a.wA[i], wb = a.wB[j];
    const double wr = wa.x * wb.x - wa.y * wb.y, wi = wa.x * wb.y + wa.y * wb.x;
    double *acc = a.acc + (long long)b * a.acc_bstride;
    const long long N3 = (long long)N * N * N;
    const T r = (T)ai.w, s = (T)bj.w;
    for (int mx = x0; mx <= x1; mx++) {
        const T dx = (T)(cx - (a.t0x + mx * a.h));
        for (int my = y0; my <= y1; my++) {
            const T dy = (T)(cy - (a.t0y + my * a.h));
            for (int mz = z0; mz <= z1; mz++) {
                const T dz = (T)(cz - (a.t0z + mz * a.h));
                const T d = sqrt(dx * dx + dy * dy + dz * dz);
                const T v = lens_volume_dev<T>(r, s, d);
                if (v == (T)0) continue;
                const long long idx = ((long long)mx * N + my) * N + mz;
                atomicAdd(acc + idx, wr * (double)v);
                if (CPLX) atomicAdd(acc + N3 + idx, wi * (double)v);
            }
        }
    }
}

void launch_exact(const ExactArgs &a, int batch, cudaStream_t s)
{
    const long long np = (long long)a.nA * a.nB;
    dim3 grid((unsigned)((np + 255) / 256), batch);
    if (a.fp64) {
        if (a.complex_w) exact_kernel<double, true><<<grid, 256, 0, s>>>(a);
        else exact_kernel<double, false><<<grid, 256, 0, s>>>(a);
    } else {
        if (a.complex_w) exact_kernel<float, true><<<grid, 256, 0, s>>>(a);
        else exact_kernel<float, false><<<grid, 256, 0, s>>>(a);
    }
}

// ---------------------------------------------------------------- outputs of exact mode

__global__ void exact_full_kernel(ExactOutArgs a)
{
    const int b = blockIdx.y;
    const long long N3 = (long long)a.N * a.N * a.N;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N3) return;
    const double *acc = a.acc + (long long)b * a.acc_bstride;
    const double re = acc[i], im = a.complex_w ? acc[N3 + i] : 0.0;
    if (a.fp64) {
        double *o = (double *)a.out;
        if (a.complex_w) {
            o[2 * (b * N3 + i)] = re;
            o[2 * (b * N3 + i) + 1] = im;
        } else
            o[b * N3 + i] = re;
    } else {
        float *o = (float *)a.out;
        if (a.complex_w) {
            o[2 * (b * N3 + i)] = (float)re;
            o[2 * (b * N3 + i) + 1] = (float)im;
        } else
            o[b * N3 + i] = (float)re;
    }
}

struct ValIdx {
    double v;
    long long i;
};
__device__ __forceinline__ bool better_min(ValIdx a, ValIdx b) { return a.v < b.v || (a.v == b.v && a.i < b.i); }
__device__ __forceinline__ bool better_max(ValIdx a, ValIdx b) { return a.v > b.v || (a.v == b.v && a.i < b.i); }

__device__ __forceinline__ ValIdx shfl_vi(ValIdx x, int off)
{
    ValIdx y;
    y.v = __shfl_xor_sync(0xffffffffu, x.v, off);
    y.i = __shfl_xor_sync(0xffffffffu, x.i, off);
    return y;
}

// Block-reduce to (min, max) of Re f; partial[b][blk] written.  Deterministic.
__global__ void __launch_bounds__(256) exact_reduce1(ExactOutArgs a, int nblk)
{
    __shared__ ValIdx smin[8], smax[8];
    const int b = blockIdx.y;
    const long long N3 = (long long)a.N * a.N * a.N;
    const double *acc = a.acc + (long long)b * a.acc_bstride;
    ValIdx mn = {1e300, 0x7fffffffffffffffll}, mx = {-1e300, 0x7fffffffffffffffll};
    for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < N3; i += (long long)nblk * 256) {
        const ValIdx c = {acc[i] + 0.0, i};
        if (better_min(c, mn)) mn = c;
        if (better_max(c, mx)) mx = c;
    }
    for (int off = 16; off > 0; off >>= 1) {
        ValIdx o = shfl_vi(mn, off);
        if (better_min(o, mn)) mn = o;
        o = shfl_vi(mx, off);
        if (better_max(o, mx)) mx = o;
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        smin[w] = mn;
        smax[w] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ValIdx bmin = smin[0], bmax = smax[0];
        for (int q = 1; q < 8; q++) {
            if (better_min(smin[q], bmin)) bmin = smin[q];
            if (better_max(smax[q], bmax)) bmax = smax[q];
        }
        const long long o = (long long)b * nblk + blockIdx.x;
        a.partials[2 * o] = bmin.v;
        a.partial_idx[2 * o] = bmin.i;
        a.partials[2 * o + 1] = bmax.v;
        a.partial_idx[2 * o + 1] = bmax.i;
    }
}

__global__ void exact_reduce2(ExactOutArgs a, int nblk)
{
    const int b = blockIdx.x;
    if (threadIdx.x != 0) return;
    ValIdx mn = {1e300, 0x7fffffffffffffffll}, mx = {-1e300, 0x7fffffffffffffffll};
    for (int q = 0; q < nblk; q++) {
        const long long o = (long long)b * nblk + q;
        const ValIdx c1 = {a.partials[2 * o], a.partial_idx[2 * o]};
        const ValIdx c2 = {a.partials[2 * o + 1], a.partial_idx[2 * o + 1]};
        if (better_min(c1, mn)) mn = c1;
        if (better_max(c2, mx)) mx = c2;
    }
    bc_extremum *out = (bc_extremum *)a.out;
    bc_extremum emin = {mn.v, (int64_t)mn.i}, emax = {mx.v, (int64_t)mx.i};
    if (a.out_kind == BC_OUT_MIN_ARGMIN)
        out[b] = emin;
    else if (a.out_kind == BC_OUT_MINMAX) {
        out[2 * b] = emin;
        out[2 * b + 1] = emax;
    } else
        out[b] = emax;
}

void launch_exact_out(const ExactOutArgs &a, int batch, cudaStream_t s, int *launches)
{
    const long long N3 = (long long)a.N * a.N * a.N;
    if (a.out_kind == BC_OUT_F_FULL) {
        dim3 grid((unsigned)((N3 + 255) / 256), batch);
        exact_full_kernel<<<grid, 256, 0, s>>>(a);
        *launches += 1;
        return;
    }
    const int nblk = 64;
    exact_reduce1<<<dim3(nblk, batch), 256, 0, s>>>(a, nblk);
    exact_reduce2<<<batch, 32, 0, s>>>(a, nblk);
    *launches += 2;
}
