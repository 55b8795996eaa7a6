// spectral64.cu -- the spectral route in fp64 (BC_MODE_SPECTRAL + BC_FP64): a parity mode.
//
// SURVEY §8(c) reading C-1 (iii): the spectral implementation pinned at 1e-9 against the
// band-limited reference.  The same method and the same host plan as the fp32 pipeline --
// each ball's indicator smoothed by the plan's Gaussian window (eps 1e-15 here) on the plan's
// box of the fine lattice (spacing h_f = P / G, origin o), one axis DFT at a time onto the band
// |k_i| <= K with the plan's per-axis multipliers (h_f, the box shift e^{-2 pi i k o / G}, the
// Gaussian deconvolution e^{2 pi^2 tau^2 k^2 / P^2}, A's origin phase e^{2 pi i k t0 / P}),
// the spectral product A_hat'(k) B_hat_R(-k) (PAPER.md L398-L419 eq_ccghat, reading C-3),
// and the inverse transform onto the grid t_m = t0 + m h (1/P^3) -- written as direct fp64
// sums (thread per output, exact integer phase reduction into an e^{-2 pi i r / G} table)
// instead of FFTs: slow, small problems only (box L <= 160, band M <= 129), no fp32 anywhere.
#include "kernels.cuh"

__device__ double smoothed_ball64(double s, double d, double tau)
{
    // (1_{B(0,s)} * G_tau)(d), the closed form of api.cu's smoothed_ball_host (fp64)
    const double pi = 3.14159265358979323846;
    const double a = (s - d) / (1.4142135623730950488 * tau), b = (s + d) / (1.4142135623730950488 * tau);
    const double t1 = a >= 0 ? 0.5 * (erf(a) + erf(b)) : 0.5 * (erfc(-a) - erfc(b));
    const double x = s * d / (tau * tau);
    double t2;
    if (x < 1e-2) {
        const double x2 = x * x;
        t2 = 2 * s / (tau * sqrt(2 * pi)) * exp(-(s * s + d * d) / (2 * tau * tau)) * (1 + x2 / 6 + x2 * x2 / 120);
    } else {
        t2 = tau / (d * sqrt(2 * pi)) * (exp(-(s - d) * (s - d) / (2 * tau * tau)) - exp(-(s + d) * (s + d) / (2 * tau * tau)));
    }
    return t1 - t2;
}

// box[ix][iy][iz] = sum_j w_j g(s_j, |x_n - R c_j|),  x_n = (o + n) h_f
__global__ void sp64_spread_kernel(Sp64SpreadArgs a)
{
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long L = a.L, n3 = L * L * L;
    if (e >= n3) return;
    const int ix = (int)(e / (L * L)), iy = (int)((e / L) % L), iz = (int)(e % L);
    const double x = (a.o[0] + ix) * a.hf, y = (a.o[1] + iy) * a.hf, z = (a.o[2] + iz) * a.hf;
    const double *R = a.rot;
    double sr = 0.0, si = 0.0;
    for (int j = 0; j < a.n; j++) {
        const double4 bl = a.balls[j];
        double cx = bl.x, cy = bl.y, cz = bl.z;
        if (R) {  // eq_Mink0 (L235): the rotation relocates the centre only
            cx = R[0] * bl.x + R[1] * bl.y + R[2] * bl.z;
            cy = R[3] * bl.x + R[4] * bl.y + R[5] * bl.z;
            cz = R[6] * bl.x + R[7] * bl.y + R[8] * bl.z;
        }
        const double dx = x - cx, dy = y - cy, dz = z - cz;
        const double d = sqrt(dx * dx + dy * dy + dz * dz);
        if (d >= bl.w + a.cut) continue;
        const double g = smoothed_ball64(bl.w, d, a.tau);
        const double2 w = a.w[j];
        sr += w.x * g;
        si += w.y * g;
    }
    a.out[e] = make_double2(sr, si);
}

// out[o][q][i] = mult(k) sum_{n < Lin} in[o][n][i] e^{sign 2 pi i (qlo + q)(nlo + n) / G}
__global__ void sp64_dft_kernel(Sp64DftArgs a)
{
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = (long long)a.O * a.nq * a.I;
    if (e >= total) return;
    const long long i = e % a.I, q = (e / a.I) % a.nq, o = e / ((long long)a.I * a.nq);
    const long long kq = a.qlo + q;
    const double2 *in = a.in + o * (long long)a.Lin * a.I + i;
    double sr = 0.0, si = 0.0;
    for (int n = 0; n < a.Lin; n++) {
        long long r = (kq * (a.nlo + n)) % a.G;
        if (r < 0) r += a.G;
        const double2 w = a.tw[r];  // e^{-2 pi i r / G}
        const double wy = a.sign < 0 ? w.y : -w.y;
        const double2 x = in[(long long)n * a.I];
        sr += x.x * w.x - x.y * wy;
        si += x.x * wy + x.y * w.x;
    }
    double mr = 1.0, mi = 0.0;
    if (a.mult) {
        // h_f e^{-2 pi i k o / G} e^{2 pi^2 tau^2 k^2 / P^2} (x e^{2 pi i k t0 / P} for A)
        const double pi = 3.14159265358979323846;
        long long r = (kq * a.off) % a.G;
        if (r < 0) r += a.G;
        double ang = -2 * pi * (double)r / a.G;
        if (a.origin) {
            const double f = (double)kq * a.t0 / a.P;
            ang += 2 * pi * (f - floor(f));
        }
        const double amp = a.hf * exp(2 * pi * pi * a.tau * a.tau * (double)(kq * kq) / (a.P * a.P));
        double s, c;
        sincos(ang, &s, &c);
        mr = amp * c;
        mi = amp * s;
    }
    a.out[o * (long long)a.nq * a.I + q * a.I + i] = make_double2(sr * mr - si * mi, sr * mi + si * mr);
}

// G(k) = A'(k) B_hat_R(-k) on the full band [kx][ky][kz], each axis k in [-K, K]
__global__ void sp64_product_kernel(const double2 *A, const double2 *B, double2 *Gk, int M)
{
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long M3 = (long long)M * M * M;
    if (e >= M3) return;
    const long long ix = e / ((long long)M * M), iy = (e / M) % M, iz = e % M;
    const double2 a = A[e], b = B[((M - 1 - ix) * M + (M - 1 - iy)) * M + (M - 1 - iz)];
    Gk[e] = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__global__ void sp64_output_kernel(const double2 *f, long long n, double scale, int complex_w, double *out)
{
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    if (complex_w) {
        out[2 * e] = f[e].x * scale;
        out[2 * e + 1] = f[e].y * scale;
    } else {
        out[e] = f[e].x * scale;  // real weights: the result is real (imaginary part ~1e-17)
    }
}

static unsigned blocks_for(long long n) { return (unsigned)((n + 255) / 256); }

void launch_sp64_spread(const Sp64SpreadArgs &a, cudaStream_t s)
{
    sp64_spread_kernel<<<blocks_for((long long)a.L * a.L * a.L), 256, 0, s>>>(a);
}
void launch_sp64_dft(const Sp64DftArgs &a, cudaStream_t s)
{
    sp64_dft_kernel<<<blocks_for((long long)a.O * a.nq * a.I), 256, 0, s>>>(a);
}
void launch_sp64_product(const double2 *A, const double2 *B, double2 *Gk, int M, cudaStream_t s)
{
    sp64_product_kernel<<<blocks_for((long long)M * M * M), 256, 0, s>>>(A, B, Gk, M);
}
void launch_sp64_output(const double2 *f, long long n, double scale, int complex_w, double *out, cudaStream_t s)
{
    sp64_output_kernel<<<blocks_for(n), 256, 0, s>>>(f, n, scale, complex_w, out);
}
