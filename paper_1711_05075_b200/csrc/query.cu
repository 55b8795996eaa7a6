// query.cu -- the time-critical single-configuration query.
//
// PAPER.md L432-L439 / L539-L546: when only a few configurations (R, t) are asked for, the
// full translation grid is wasted work; the paper evaluates g(R, t) directly, at a cost that
// grows only with the retained terms.  Here the directly evaluated sum is the exact one of
// the combinatorial route (eq_ORP / eq_convgP):
//     f_R(t) = sum_ij w_i v_j V(r_i, s_j, |a_i - (R b_j + t)|),
// restricted to the pairs that overlap, found through a uniform grid of A's centres with
// cell size >= max r + max s (an overlapping pair's A ball lies in one of the 27 cells
// around R b_j + t).  fp64 throughout; deterministic (fixed per-thread order, fixed-shape
// block reduction, partials summed in order).
#include "kernels.cuh"

#include "ballcorr.h"

__device__ __forceinline__ double lens_volume_q(double r, double s, double d)
{
    const double pi = 3.14159265358979323846;
    if (d >= r + s) return 0.0;
    const double m = r < s ? r : s;
    const double rs = r - s;
    if (d <= fabs(rs)) return 4.0 / 3.0 * pi * m * m * m;
    const double e = r + s - d;
    return pi * e * e * (d * d + 2.0 * d * (r + s) - 3.0 * rs * rs) / (12.0 * d);
}

// grid: (ceil(nB / 256), n_queries); thread = one ball j of B for query q
__global__ void __launch_bounds__(256) query_pairs_kernel(QueryArgs a)
{
    const int q = blockIdx.y;
    const int j = blockIdx.x * 256 + threadIdx.x;
    double sr = 0.0, si = 0.0;
    if (j < a.nB) {
        const double *R = a.R + 9 * q;
        const double *t = a.t + 3 * q;
        const double4 bj = a.B[j];
        // eq_Mink0 (L235): R B, then the translation t
        const double cx = R[0] * bj.x + R[1] * bj.y + R[2] * bj.z + t[0];
        const double cy = R[3] * bj.x + R[4] * bj.y + R[5] * bj.z + t[1];
        const double cz = R[6] * bj.x + R[7] * bj.y + R[8] * bj.z + t[2];
        const int gx = (int)floor((cx - a.gx0) * a.inv_cs), gy = (int)floor((cy - a.gy0) * a.inv_cs),
                  gz = (int)floor((cz - a.gz0) * a.inv_cs);
        const double2 wb = a.wB[j];
        for (int ix = max(gx - 1, 0); ix <= min(gx + 1, a.nx - 1); ix++)
            for (int iy = max(gy - 1, 0); iy <= min(gy + 1, a.ny - 1); iy++)
                for (int iz = max(gz - 1, 0); iz <= min(gz + 1, a.nz - 1); iz++) {
                    const int cell = (ix * a.ny + iy) * a.nz + iz;
                    for (int e = a.start[cell]; e < a.start[cell + 1]; e++) {
                        const int i = a.idx[e];
                        const double4 ai = a.A[i];
                        const double dx = ai.x - cx, dy = ai.y - cy, dz = ai.z - cz;
                        const double v = lens_volume_q(ai.w, bj.w, sqrt(dx * dx + dy * dy + dz * dz));
                        if (v == 0.0) continue;
                        const double2 wa = a.wA[i];
                        sr += (wa.x * wb.x - wa.y * wb.y) * v;
                        si += (wa.x * wb.y + wa.y * wb.x) * v;
                    }
                }
    }
    __shared__ double red[2][256];
    red[0][threadIdx.x] = sr;
    red[1][threadIdx.x] = si;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            red[0][threadIdx.x] += red[0][threadIdx.x + o];
            red[1][threadIdx.x] += red[1][threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.partial[2 * ((long long)q * gridDim.x + blockIdx.x)] = red[0][0];
        a.partial[2 * ((long long)q * gridDim.x + blockIdx.x) + 1] = red[1][0];
    }
}

__global__ void query_sum_kernel(QueryArgs a, int nblk)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.nq) return;
    double sr = 0.0, si = 0.0;
    for (int k = 0; k < nblk; k++) {
        sr += a.partial[2 * ((long long)q * nblk + k)];
        si += a.partial[2 * ((long long)q * nblk + k) + 1];
    }
    if (a.complex_w) {
        a.out[2 * q] = sr;
        a.out[2 * q + 1] = si;
    } else {
        a.out[q] = sr;
    }
}

int query_blocks(int nB) { return (nB + 255) / 256; }

void launch_query(const QueryArgs &a, cudaStream_t s)
{
    const int nblk = query_blocks(a.nB);
    query_pairs_kernel<<<dim3(nblk, a.nq), 256, 0, s>>>(a);
    query_sum_kernel<<<(a.nq + 127) / 128, 128, 0, s>>>(a, nblk);
}
