// exact.cu -- the combinatorial (pair-lens) route of libballcorr.
//
// PAPER.md L343-L360 (eq_ORP, eq_convgP): the translational obstacle of two
// ball sets is the union of obstacle balls centred at a_i - R b_j with radius
// r_i + s_j, and g = rho_{P_O} * f_{B_O} with primitive kernel
// f_{B_O} = f_{B_1} * f_{B_2}.  For indicator primitives that kernel is the
// two-ball intersection volume V(r, s, d), so
//     f_R(t_m) = sum_ij w_i v_j V(r_i, s_j, |a_i - R b_j - t_m|).
// Each (i, j) pair (one warp, lanes over its footprint) spreads V onto the grid points
// inside its obstacle ball (fixed-point integer sums: see below).  This is the paper's "pairwise
// Minkowski sum" GPU kernel (L515-L520), here with exact lens weights.
#include <algorithm>

#include "kernels.cuh"

#include "ballcorr.h"

template <typename T>
__device__ __forceinline__ T lens_div(T a, T b) { return a / b; }
template <>
__device__ __forceinline__ float lens_div<float>(float a, float b) { return __fdividef(a, b); }

template <typename T>
__device__ __forceinline__ T lens_volume_dev(T r, T s, T d)
{
    const T pi = (T)3.14159265358979323846;
    if (d >= r + s) return (T)0;
    const T m = r < s ? r : s;
    const T rs = r - s;
    if (d <= (rs < 0 ? -rs : rs)) return (T)4 / (T)3 * pi * m * m * m;
    const T e = r + s - d;
    return lens_div<T>(pi * e * e * (d * d + (T)2 * d * (r + s) - (T)3 * rs * rs), (T)12 * d);
}

// ---------------------------------------------------------------- accumulation
//
// The per-point sums are fixed-point integers: each term w_i v_j V x qscale rounded to int64,
// qscale = 2^61 / (a bound on |f|, set by the host).  Integer addition is associative, so the
// sums are bitwise independent of the order in which warps add their terms (64-bit integer
// reductions, RED.E.ADD.64 -- no floating-point atomics), of the batching and of the launch:
// deterministic.  The quantisation (<= 2^-62 of the bound per term) sits far below fp64's 1e-9
// parity bar.
struct KnotBox {
    double cx, cy, cz, rs;
    int lo[3], hi[3];  // grid point range (inclusive), empty if lo > hi on an axis
};

__device__ __forceinline__ KnotBox knot_box(const ExactArgs &a, int b, int i, int j)
{
    const double *R = a.rot + 9 * b;
    const double4 ai = a.A[i], bj = a.B[j];
    KnotBox kb;
    // obstacle knot a_i - R b_j (eq_ORP), radius r_i + s_j
    kb.cx = ai.x - (R[0] * bj.x + R[1] * bj.y + R[2] * bj.z);
    kb.cy = ai.y - (R[3] * bj.x + R[4] * bj.y + R[5] * bj.z);
    kb.cz = ai.z - (R[6] * bj.x + R[7] * bj.y + R[8] * bj.z);
    kb.rs = ai.w + bj.w;
    const double ih = a.inv_h;
    const double c[3] = {kb.cx - a.t0x, kb.cy - a.t0y, kb.cz - a.t0z};
#pragma unroll
    for (int d = 0; d < 3; d++) {
        kb.lo[d] = max((int)ceil((c[d] - kb.rs) * ih), 0);
        kb.hi[d] = min((int)floor((c[d] + kb.rs) * ih), a.N - 1);
    }
    return kb;
}

__device__ __forceinline__ long long to_fixed(double x) { return __double2ll_rn(x); }
__device__ __forceinline__ long long to_fixed(float x) { return __float2ll_rn(x); }

// Warp per obstacle knot: lanes own (y, z) columns of the knot's footprint box, walk x, and add their
// fixed-point terms to the output accumulator with 64-bit integer reductions (RED.E.ADD.64:
// associative, so the result does not depend on which warp adds first -- deterministic).
template <typename T, bool CPLX>
__global__ void __launch_bounds__(256) exact_scatter_kernel(ExactArgs a)
{
    // grid (ceil(nB / 8), A chunk, rotation): warp w of the block = knot (i, j), no division
    const int b = blockIdx.z;
    const int i = a.i0 + blockIdx.y, j = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= a.nB) return;
    const KnotBox kb = knot_box(a, b, i, j);
    const int nx = kb.hi[0] - kb.lo[0] + 1, ny = kb.hi[1] - kb.lo[1] + 1, nz = kb.hi[2] - kb.lo[2] + 1;
    if (nx <= 0 || ny <= 0 || nz <= 0) return;
    const double ih = a.inv_h;
    // centre relative to the box's first point and radii, grid units
    const T cx = (T)((kb.cx - a.t0x) * ih - kb.lo[0]), cy = (T)((kb.cy - a.t0y) * ih - kb.lo[1]),
            cz = (T)((kb.cz - a.t0z) * ih - kb.lo[2]);
    const double rr = a.A[i].w * ih, ss = a.B[j].w * ih;
    const T r = (T)rr, s = (T)ss, rho2 = (T)((rr + ss) * (rr + ss));
    const double2 wa = a.wA[i], wb = a.wB[j];
    const double h3q = a.h * a.h * a.h * a.qscale;  // V in grid units x h^3 x fixed-point scale
    const T wr = (T)((wa.x * wb.x - wa.y * wb.y) * h3q), wi = (T)((wa.x * wb.y + wa.y * wb.x) * h3q);
    const long long N = a.N, N3 = N * N * N;
    unsigned long long *acc = (unsigned long long *)a.iacc + (long long)b * a.acc_bstride;
    // lanes own (y, z) columns of the footprint box (one division per column) and walk x
    const int nyz = ny * nz;
    for (int q = lane; q < nyz; q += 32) {
        const int iy = q / nz, iz = q - (q / nz) * nz;
        const T dy = cy - (T)iy, dz = cz - (T)iz;
        const T dyz2 = dy * dy + dz * dz;
        if (dyz2 >= rho2) continue;
        const long long row = ((long long)kb.lo[0] * N + (kb.lo[1] + iy)) * N + (kb.lo[2] + iz);
        for (int ix = 0; ix < nx; ix++) {
            const T dx = cx - (T)ix;
            const T d2 = dx * dx + dyz2;
            if (d2 >= rho2) continue;
            const T v = lens_volume_dev<T>(r, s, sqrt(d2));
            const long long idx = row + (long long)ix * N * N;
            atomicAdd(acc + idx, (unsigned long long)to_fixed(wr * v));
            if (CPLX) atomicAdd(acc + N3 + idx, (unsigned long long)to_fixed(wi * v));
        }
    }
}

// Thread per obstacle knot (for small footprints, where a warp per knot idles most lanes):
// the thread walks the grid points INSIDE the obstacle ball (per (x, y) row its z range from
// the chord), B's balls taken in order of radius (a.permB) so a warp's 32 knots have similar
// footprints; the same fixed-point integer reductions as above.
template <typename T, bool CPLX>
__global__ void __launch_bounds__(256) exact_knot_kernel(ExactArgs a)
{
    const int b = blockIdx.z;
    const int i = a.i0 + blockIdx.y, jj = blockIdx.x * 256 + threadIdx.x;
    if (jj >= a.nB) return;
    const int j = a.permB[jj];
    const KnotBox kb = knot_box(a, b, i, j);
    const int nx = kb.hi[0] - kb.lo[0] + 1, ny = kb.hi[1] - kb.lo[1] + 1, nz = kb.hi[2] - kb.lo[2] + 1;
    if (nx <= 0 || ny <= 0 || nz <= 0) return;
    const double ih = a.inv_h;
    const T cx = (T)((kb.cx - a.t0x) * ih - kb.lo[0]), cy = (T)((kb.cy - a.t0y) * ih - kb.lo[1]),
            cz = (T)((kb.cz - a.t0z) * ih - kb.lo[2]);
    const double rr = a.A[i].w * ih, ss = a.B[j].w * ih;
    const T r = (T)rr, s = (T)ss, rho2 = (T)((rr + ss) * (rr + ss));
    const double2 wa = a.wA[i], wb = a.wB[j];
    const double h3q = a.h * a.h * a.h * a.qscale;
    const T wr = (T)((wa.x * wb.x - wa.y * wb.y) * h3q), wi = (T)((wa.x * wb.y + wa.y * wb.x) * h3q);
    const long long N = a.N, N3 = N * N * N;
    unsigned long long *acc = (unsigned long long *)a.iacc + (long long)b * a.acc_bstride;
    for (int ix = 0; ix < nx; ix++) {
        const T dx = cx - (T)ix;
        for (int iy = 0; iy < ny; iy++) {
            const T dy = cy - (T)iy;
            const T dxy2 = dx * dx + dy * dy;
            if (dxy2 >= rho2) continue;
            const T hz = sqrt(rho2 - dxy2);
            const int z0 = max(0, (int)ceil(cz - hz)), z1 = min(nz - 1, (int)floor(cz + hz));
            const long long row = ((long long)(kb.lo[0] + ix) * N + (kb.lo[1] + iy)) * N + kb.lo[2];
            for (int iz = z0; iz <= z1; iz++) {
                const T dz = cz - (T)iz;
                const T d2 = dxy2 + dz * dz;
                if (d2 >= rho2) continue;
                const T v = lens_volume_dev<T>(r, s, sqrt(d2));
                atomicAdd(acc + row + iz, (unsigned long long)to_fixed(wr * v));
                if (CPLX) atomicAdd(acc + N3 + row + iz, (unsigned long long)to_fixed(wi * v));
            }
        }
    }
}

// ---------------------------------------------------------------- fp32 lens, branch-free
// The fp32 exact mode (tolerance 1e-4 of max|f|; the fp64 mode keeps lens_volume_dev<double>)
// evaluates the lens volume division-free:
//   V = pi/12 e^2 (d^2 + 2 d S - 3 D^2) / d = pi/12 e^2 (d + 2 S - 3 D^2 / d),  e = S - d,
//   S = r + s, D = r - s;  V = 4/3 pi min(r, s)^3 when d <= |D|;  0 when d >= S (the chord test).
// 1/d from one MUFU.RSQ (d = d^2 rsqrt(d^2), d^2 floored at 1e-30 so d = 0 gives 0, not NaN:
// it is then inside the containment branch, or D = 0 and the 3 D^2 / d term is 0 x finite).
// The weight w_i v_j (x h^3 x the fixed-point scale) is folded into two per-knot constants.
struct LensF32 {
    float cx, cy, cz;   // knot centre relative to its box's first point (grid units)
    float rho2, S, aD, c1, c2;
    float kr, ki;       // pi/12 x weight (re, im) x scale
    float fr, fi;       // 4/3 pi min(r, s)^3 x weight x scale
};

__device__ __forceinline__ LensF32 lens_f32_setup(const ExactArgs &a, const KnotBox &kb, int i, int j, double scale)
{
    LensF32 L;
    const double ih = a.inv_h;
    L.cx = (float)((kb.cx - a.t0x) * ih - kb.lo[0]);
    L.cy = (float)((kb.cy - a.t0y) * ih - kb.lo[1]);
    L.cz = (float)((kb.cz - a.t0z) * ih - kb.lo[2]);
    const double rr = a.A[i].w * ih, ss = a.B[j].w * ih;
    L.rho2 = (float)((rr + ss) * (rr + ss));
    L.S = (float)(rr + ss);
    L.aD = (float)fabs(rr - ss);
    L.c1 = 2.f * L.S;
    L.c2 = (float)(3.0 * (rr - ss) * (rr - ss));
    const double2 wa = a.wA[i], wb = a.wB[j];
    const double h3q = a.h * a.h * a.h * scale;
    const double wr = (wa.x * wb.x - wa.y * wb.y) * h3q, wi = (wa.x * wb.y + wa.y * wb.x) * h3q;
    const double pi = 3.14159265358979323846, m = rr < ss ? rr : ss, vf = 4.0 / 3.0 * pi * m * m * m;
    L.kr = (float)(pi / 12.0 * wr);
    L.ki = (float)(pi / 12.0 * wi);
    L.fr = (float)(vf * wr);
    L.fi = (float)(vf * wi);
    return L;
}

// visit the grid points inside the knot's ball (per (x, y) row its z range from the chord):
// f(x, y, z, term_re, term_im) with box-relative indices
template <bool CPLX, typename F>
__device__ __forceinline__ void lens_f32_walk(const LensF32 &L, int nx, int ny, int nz, F &&f)
{
    for (int ix = 0; ix < nx; ix++) {
        const float dx = L.cx - (float)ix;
        for (int iy = 0; iy < ny; iy++) {
            const float dy = L.cy - (float)iy;
            const float dxy2 = fmaf(dx, dx, dy * dy);
            if (dxy2 >= L.rho2) continue;
            const float hz = sqrtf(L.rho2 - dxy2);
            const int z0 = max(0, (int)ceilf(L.cz - hz)), z1 = min(nz - 1, (int)floorf(L.cz + hz));
            for (int iz = z0; iz <= z1; iz++) {
                const float dz = L.cz - (float)iz;
                const float d2 = fmaf(dz, dz, dxy2);
                if (d2 >= L.rho2) continue;
                const float rd = rsqrtf(fmaxf(d2, 1e-30f));
                const float d = d2 * rd;
                const float e = L.S - d;
                const float t = e * e * fmaf(-L.c2, rd, d + L.c1);
                const bool inside = d <= L.aD;
                f(ix, iy, iz, inside ? L.fr : L.kr * t, CPLX ? (inside ? L.fi : L.ki * t) : 0.f);
            }
        }
    }
}

// fp32 thread-per-knot kernel (B by radius, as exact_knot_kernel; the same 64-bit integer
// reductions)
template <bool CPLX>
__global__ void __launch_bounds__(256) exact_knot_f32_kernel(ExactArgs a)
{
    const int b = blockIdx.z;
    const int i = a.i0 + blockIdx.y, jj = blockIdx.x * 256 + threadIdx.x;
    if (jj >= a.nB) return;
    const int j = a.permB[jj];
    const KnotBox kb = knot_box(a, b, i, j);
    const int nx = kb.hi[0] - kb.lo[0] + 1, ny = kb.hi[1] - kb.lo[1] + 1, nz = kb.hi[2] - kb.lo[2] + 1;
    if (nx <= 0 || ny <= 0 || nz <= 0) return;
    const LensF32 L = lens_f32_setup(a, kb, i, j, a.qscale);
    const long long N = a.N, N3 = N * N * N;
    unsigned long long *acc = (unsigned long long *)a.iacc + (long long)b * a.acc_bstride;
    lens_f32_walk<CPLX>(L, nx, ny, nz, [&](int ix, int iy, int iz, float tr, float ti) {
        const long long idx = ((long long)(kb.lo[0] + ix) * N + (kb.lo[1] + iy)) * N + kb.lo[2] + iz;
        atomicAdd(acc + idx, (unsigned long long)__float2ll_rn(tr));
        if (CPLX) atomicAdd(acc + N3 + idx, (unsigned long long)__float2ll_rn(ti));
    });
}

// Packed pairs (fp32 mode, even N): the kernel above is bound by its global 64-bit reductions
// (4.9e7 for Single; without the lens arithmetic it takes 90 % of the time).  Here each 64-bit
// word holds the 32-bit fixed-point sums of two neighbouring grid points (flat index 2m in the
// low half, 2m + 1 in the high half), so a chord adds two points with one reduction: the word
// gets t0 + 2^32 t1 (signed 64-bit arithmetic), and as long as each point's sum fits int32 the
// word decodes exactly (low = int32(word), high = (word - low) / 2^32).  The host's scale
// (2^30 / a tight bound on sum |terms| at any point, exact_plan) guarantees the fit; integer
// sums stay order-independent (deterministic).
template <bool CPLX>
__global__ void __launch_bounds__(256) exact_knot_pack_kernel(ExactArgs a)
{
    const int b = blockIdx.z;
    const int i = a.i0 + blockIdx.y, jj = blockIdx.x * 256 + threadIdx.x;
    if (jj >= a.nB) return;
    const int j = a.permB[jj];
    const KnotBox kb = knot_box(a, b, i, j);
    const int nx = kb.hi[0] - kb.lo[0] + 1, ny = kb.hi[1] - kb.lo[1] + 1, nz = kb.hi[2] - kb.lo[2] + 1;
    if (nx <= 0 || ny <= 0 || nz <= 0) return;
    const LensF32 L = lens_f32_setup(a, kb, i, j, a.qscale);
    const long long N = a.N, N3 = N * N * N;
    unsigned long long *acc = (unsigned long long *)a.iacc + (long long)b * a.acc_bstride;
    auto term = [&](float dxy2, int iz, int z0, int z1, long long &tr, long long &ti) {
        tr = ti = 0;
        if (iz < z0 || iz > z1) return;
        const float dz = L.cz - (float)iz;
        const float d2 = fmaf(dz, dz, dxy2);
        if (d2 >= L.rho2) return;
        const float rd = rsqrtf(fmaxf(d2, 1e-30f));
        const float d = d2 * rd;
        const float e = L.S - d;
        const float t = e * e * fmaf(-L.c2, rd, d + L.c1);
        const bool inside = d <= L.aD;
        tr = __float2ll_rn(inside ? L.fr : L.kr * t);
        if (CPLX) ti = __float2ll_rn(inside ? L.fi : L.ki * t);
    };
    const int pz = kb.lo[2] & 1;  // parity of the box's first z (N even: the flat index's parity)
    for (int ix = 0; ix < nx; ix++) {
        const float dx = L.cx - (float)ix;
        for (int iy = 0; iy < ny; iy++) {
            const float dy = L.cy - (float)iy;
            const float dxy2 = fmaf(dx, dx, dy * dy);
            if (dxy2 >= L.rho2) continue;
            const float hz = sqrtf(L.rho2 - dxy2);
            const int z0 = max(0, (int)ceilf(L.cz - hz)), z1 = min(nz - 1, (int)floorf(L.cz + hz));
            if (z0 > z1) continue;
            // word of box-relative z: (lo_z + z) >> 1; pairs start at the even flat index
            const long long rowp = ((long long)(kb.lo[0] + ix) * N + (kb.lo[1] + iy)) * N + kb.lo[2] - pz;  // even
            unsigned long long *w = acc + (rowp >> 1);
            for (int q = (z0 + pz) & ~1; q <= z1 + pz; q += 2) {  // q = z + pz of the pair's even point
                long long r0, i0, r1, i1;
                term(dxy2, q - pz, z0, z1, r0, i0);
                term(dxy2, q - pz + 1, z0, z1, r1, i1);
                atomicAdd(w + (q >> 1), (unsigned long long)r0 + ((unsigned long long)r1 << 32));
                if (CPLX) atomicAdd(w + (N3 >> 1) + (q >> 1), (unsigned long long)i0 + ((unsigned long long)i1 << 32));
            }
        }
    }
}

void launch_exact_scatter(const ExactArgs &a_in, int batch, cudaStream_t s)
{
    ExactArgs a = a_in;
    for (int i0 = 0; i0 < a_in.nA; i0 += 65535) {  // grid.y limit: A in chunks
        a.i0 = i0;
        const unsigned ny = (unsigned)std::min(65535, a_in.nA - i0);
        if (a.thread_per_knot) {
            dim3 grid((unsigned)((a.nB + 255) / 256), ny, batch);
            if (a.fp64) {
                if (a.complex_w) exact_knot_kernel<double, true><<<grid, 256, 0, s>>>(a);
                else exact_knot_kernel<double, false><<<grid, 256, 0, s>>>(a);
            } else {
                if (a.packed) {
                    if (a.complex_w) exact_knot_pack_kernel<true><<<grid, 256, 0, s>>>(a);
                    else exact_knot_pack_kernel<false><<<grid, 256, 0, s>>>(a);
                } else if (a.complex_w) {
                    exact_knot_f32_kernel<true><<<grid, 256, 0, s>>>(a);
                } else {
                    exact_knot_f32_kernel<false><<<grid, 256, 0, s>>>(a);
                }
            }
        } else {
            dim3 grid((unsigned)((a.nB + 7) / 8), ny, batch);
            if (a.fp64) {
                if (a.complex_w) exact_scatter_kernel<double, true><<<grid, 256, 0, s>>>(a);
                else exact_scatter_kernel<double, false><<<grid, 256, 0, s>>>(a);
            } else {
                if (a.complex_w) exact_scatter_kernel<float, true><<<grid, 256, 0, s>>>(a);
                else exact_scatter_kernel<float, false><<<grid, 256, 0, s>>>(a);
            }
        }
    }
}

// ---------------------------------------------------------------- outputs of exact mode

// accumulator value of point i (part offset applied by the caller): 64-bit, or packed pairs
__device__ __forceinline__ long long acc_value(const long long *acc, long long i, int packed)
{
    if (!packed) return acc[i];
    const long long w = acc[i >> 1];
    const long long lo = (long long)(int)(unsigned)w;  // the even point's int32 sum
    return (i & 1) ? (w - lo) >> 32 : lo;
}

__global__ void exact_full_kernel(ExactOutArgs a)
{
    const int b = blockIdx.y;
    const long long N3 = (long long)a.N * a.N * a.N;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N3) return;
    const long long *acc = a.iacc + (long long)b * a.acc_bstride;
    const long long *acci = acc + (a.packed ? N3 / 2 : N3);
    const double re = (double)acc_value(acc, i, a.packed) * a.inv_qscale,
                 im = a.complex_w ? (double)acc_value(acci, i, a.packed) * a.inv_qscale : 0.0;
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
    const long long *acc = a.iacc + (long long)b * a.acc_bstride;
    ValIdx mn = {1e300, 0x7fffffffffffffffll}, mx = {-1e300, 0x7fffffffffffffffll};
    for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < N3; i += (long long)nblk * 256) {
        const ValIdx c = {(double)acc_value(acc, i, a.packed) * a.inv_qscale + 0.0, i};
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
