// query_spectral.cu -- the paper's time-critical single-configuration query.
//
// PAPER.md L432-L439 (eq_single): by Parseval, g(R, t) = < f_A, f_{RB} o T^{-1} > =
// < f_A_hat, sigma_t_hat f_RB_hat >, evaluated over a truncated set of m' frequency modes
// "by a spiral traversal of the frequency grid starting from the dominant modes until the
// available time is over" -- accuracy traded for time, cost linear in m' (L539-L546, Fig. 9).
// On the P-periodic lattice of the spectral path (modes k / P, DFT as a Riemann sum of the
// CFT, L829-L833) the truncated sum is
//
//     f_m'(t) = (1/P^3) sum_{k in S_m'} A_hat(k) B_hat_R(-k) e^{2 pi i k . t / P},
//     B_hat_R(-k) = sum_j v_j beta_hat(s_j, |k| / P) e^{+2 pi i k . R b_j / P}       (eq_rhoPhat)
//
// with S_m' the first m' modes in radial-shell order (|k|^2, then lexicographic; a mode and
// its mirror -k kept together for real weights, where the pair contributes 2 Re).  A_hat(k)
// is the band spectrum bc_spectrum_A keeps (A' = A_hat e^{2 pi i k . t0 / P}); B_hat_R is the
// direct NDFT of the rotated knots (eq_rhoPhat, one-sided) times the ball transform, from a
// per-shell table beta_hat(s_j, |k| / P) v_j.  The phase of (mode, ball) is reduced in fp64
// (k . q_j, q_j = (R b_j + t - t0) / P) before an fp32 sincospi; per-mode sums in fp32, the
// reduction over modes in fp64 (fixed-shape trees, ordered partial sums: deterministic).
#include "kernels.cuh"

namespace {
constexpr int QS_MT = 128;  // modes per block
constexpr int QS_BT = 256;  // balls per block (chunk of B)
}  // namespace

// shell table: bv[j][s] = v_j beta_hat(s_j, sqrt(k2_s) / P), beta_hat(r, rho) = 4 pi (sin x - x cos x) / k^3,
// k = 2 pi rho, x = k r (series below x = 0.05)
__global__ void qs_shell_table_kernel(const double4 *B, const double2 *wB, int nB, const int *k2, int nsh, double P,
                                      int complex_w, float2 *bv)
{
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)nB * nsh) return;
    const int j = (int)(e / nsh), sidx = (int)(e % nsh);
    const double pi = 3.14159265358979323846;
    const double r = B[j].w;
    const double kk = 2 * pi * sqrt((double)k2[sidx]) / P, x = kk * r;
    double beta;
    if (x < 0.05) {
        const double x2 = x * x;
        beta = 4 * pi * r * r * r * (1.0 / 3 - x2 / 30 + x2 * x2 / 840 - x2 * x2 * x2 / 45360);
    } else {
        double sx, cx;
        sincos(x, &sx, &cx);
        beta = 4 * pi * (sx - x * cx) / (kk * kk * kk);
    }
    const double2 w = wB[j];
    bv[e] = make_float2((float)(w.x * beta), complex_w ? (float)(w.y * beta) : 0.f);
}

// partial B sums: part[q][ball chunk][mode] = sum_{j in chunk} bv[j][shell(m)] e^{2 pi i k_m . q_j}
__global__ void __launch_bounds__(QS_MT) qs_partial_kernel(QsArgs a)
{
    __shared__ double3 qj[QS_BT];
    const int q = blockIdx.z, jc = blockIdx.y;
    const int m = blockIdx.x * QS_MT + threadIdx.x;
    const double *R = a.R + 9 * q, *t = a.t + 3 * q;
    const int j0 = jc * QS_BT, nj = min(QS_BT, a.nB - j0);
    for (int u = threadIdx.x; u < nj; u += QS_MT) {
        const double4 b = a.B[j0 + u];
        // knot of R B translated by t, relative to the grid origin (the A' phase), in periods
        qj[u] = make_double3((R[0] * b.x + R[1] * b.y + R[2] * b.z + t[0] - a.t0x) * a.invP,
                             (R[3] * b.x + R[4] * b.y + R[5] * b.z + t[1] - a.t0y) * a.invP,
                             (R[6] * b.x + R[7] * b.y + R[8] * b.z + t[2] - a.t0z) * a.invP);
    }
    __syncthreads();
    if (m >= a.nm) return;
    const int4 km = a.modes[m];
    const double kx = km.x, ky = km.y, kz = km.z;
    const float2 *bv = a.bv + (long long)j0 * a.nsh + km.w;
    float sr = 0.f, si = 0.f;
    for (int u = 0; u < nj; u++) {
        const double3 p = qj[u];
        double ph = kx * p.x + ky * p.y + kz * p.z;
        ph -= rint(ph);                          // e^{2 pi i ph} is 1-periodic: reduce in fp64
        float s, c;
        sincospif(2.f * (float)ph, &s, &c);
        const float2 w = bv[(long long)u * a.nsh];
        sr += w.x * c - w.y * s;
        si += w.x * s + w.y * c;
    }
    a.part[((long long)q * gridDim.y + jc) * a.nm + m] = make_float2(sr, si);
}

// per mode: B_hat sum over the ball chunks (ordered), times A'(k) and the pair multiplicity;
// block reduction over the block's modes -> mpart[q][mode block]
__global__ void __launch_bounds__(QS_MT) qs_mode_kernel(QsArgs a, int nbc)
{
    __shared__ double red[2][QS_MT];
    const int q = blockIdx.y;
    const int m = blockIdx.x * QS_MT + threadIdx.x;
    double vr = 0.0, vi = 0.0;
    if (m < a.nm) {
        double br = 0.0, bi = 0.0;
        for (int jc = 0; jc < nbc; jc++) {
            const float2 p = a.part[((long long)q * nbc + jc) * a.nm + m];
            br += p.x;
            bi += p.y;
        }
        const float2 A = a.Aq[m];
        const double mult = a.mult[m];
        vr = mult * ((double)A.x * br - (double)A.y * bi);
        vi = mult * ((double)A.x * bi + (double)A.y * br);
    }
    red[0][threadIdx.x] = vr;
    red[1][threadIdx.x] = vi;
    __syncthreads();
    for (int o = QS_MT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            red[0][threadIdx.x] += red[0][threadIdx.x + o];
            red[1][threadIdx.x] += red[1][threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.mpart[2 * ((long long)q * gridDim.x + blockIdx.x)] = red[0][0];
        a.mpart[2 * ((long long)q * gridDim.x + blockIdx.x) + 1] = red[1][0];
    }
}

__global__ void qs_sum_kernel(QsArgs a, int nmb)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.nq) return;
    double sr = 0.0, si = 0.0;
    for (int b = 0; b < nmb; b++) {
        sr += a.mpart[2 * ((long long)q * nmb + b)];
        si += a.mpart[2 * ((long long)q * nmb + b) + 1];
    }
    if (a.complex_w) {
        a.out[2 * q] = sr * a.scale;
        a.out[2 * q + 1] = si * a.scale;
    } else {
        a.out[q] = sr * a.scale;  // real weights: the imaginary parts of the pairs cancel
    }
}

// A'(k) of the retained modes, gathered from the band spectrum ([ky][kz][kx], kz >= 0 for real)
__global__ void qs_gather_kernel(const float2 *Ahat, const int4 *modes, int nm, int K, int Kz, int complex_w, float2 *Aq)
{
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= nm) return;
    const int4 k = modes[m];
    const int M = 2 * K + 1;
    const int kzi = complex_w ? k.z + K : k.z;
    Aq[m] = Ahat[((long long)(k.y + K) * Kz + kzi) * M + (k.x + K)];
}

int qs_ball_chunks(int nB) { return (nB + QS_BT - 1) / QS_BT; }
int qs_mode_blocks(int nm) { return (nm + QS_MT - 1) / QS_MT; }

void launch_qs_tables(const QsTableArgs &t, cudaStream_t s)
{
    const long long n = (long long)t.nB * t.nsh;
    if (n > 0)
        qs_shell_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(t.B, t.wB, t.nB, t.k2, t.nsh, t.P, t.complex_w,
                                                                          t.bv);
    if (t.nm > 0)
        qs_gather_kernel<<<(t.nm + 255) / 256, 256, 0, s>>>(t.Ahat, t.modes, t.nm, t.K, t.Kz, t.complex_w, t.Aq);
}

void launch_qs(const QsArgs &a, cudaStream_t s)
{
    const int nbc = qs_ball_chunks(a.nB), nmb = qs_mode_blocks(a.nm);
    qs_partial_kernel<<<dim3(nmb, nbc, a.nq), QS_MT, 0, s>>>(a);
    qs_mode_kernel<<<dim3(nmb, a.nq), QS_MT, 0, s>>>(a, nbc);
    qs_sum_kernel<<<(a.nq + 127) / 128, 128, 0, s>>>(a, nmb);
}
