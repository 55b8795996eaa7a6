// collectives.cu -- compute fused with the two exchanges of the rotation-sharded path over
// peer memory (north_star (e)).
//
// 1. A's band spectrum, sharded by BALLS: rho_hat_A is linear in the knots (PAPER.md L280-L283
//    eq_rhoPhat), so rank g computes the partial spectrum of its slice of A's balls, and the
//    all-reduce of the partials is fused into the kernel that consumes the sum -- the build
//    of A'' (origin phase, B's x multipliers, B's radial deconvolution, coset-major order:
//    the permute step of permute_cm_kernel).  Every rank reads all G partial spectra straight
//    from its peers' memory (cudaIpc-mapped pointers over NVLink / NVSwitch), sums them in a
//    fixed rank order (bitwise identical on every rank) and writes its own reduced A_hat and
//    A'': no separate all-reduce launch, no staging copy.
// 2. The per-rotation results: the reduction epilogue (a7) of each rank stores its
//    {val, idx} records directly into every peer's result buffer at the rotations' global
//    indices, so no all-gather launch follows the step.
#include "kernels.cuh"

#include "ballcorr.h"

__global__ void reduce_permute_kernel(ReducePermuteArgs a)
{
    const int M = 2 * a.K + 1;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.rows * M) return;
    float2 v = make_float2(0.f, 0.f);
#pragma unroll 1
    for (int r = 0; r < a.n_parts; r++) v = cadd(v, a.parts[r][e]);  // fixed rank order
    a.Ahat[e] = v;                                                     // the reduced A_hat (queries, re-permutes)
    const long long row = e / M;
    const int k = (int)(e % M) - a.K;
    float2 u = a.neg ? cmul(v, a.mult[-k + a.K]) : cmulc(v, a.mult[k + a.K]);
    const long long ky = row / a.Kz - a.K, kz = (row % a.Kz) - (a.Kz == M ? a.K : 0);
    const long long k2 = k * (long long)k + ky * ky + kz * kz;
    if (a.dec) u = cscale(u, a.dec[k2]);
    if (a.mult_y)  // as permute_cm_kernel
        u = a.neg ? cmul(cmul(u, a.mult_y[-ky + a.K]), a.mult_z[-kz + a.K])
                  : cmulc(cmulc(u, a.mult_y[ky + a.K]), a.mult_z[kz]);
    if (a.R2 > 0 && (double)k2 > a.R2) u = make_float2(0.f, 0.f);
    a.out[row * a.MS + cm_of_k(a.neg ? -k : k, a.L, a.c, a.G, a.K)] = u;
}

void launch_reduce_permute(const ReducePermuteArgs &a, cudaStream_t s)
{
    const long long n = a.rows * (2LL * a.K + 1);
    cudaMemsetAsync(a.out, 0, sizeof(float2) * a.rows * a.MS, s);
    reduce_permute_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a);
}
