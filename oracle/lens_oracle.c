/*
 * oracle/lens_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU definition of the correlation the CUDA path
 * approximates.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or helper with paper_1711_05075_b200/.
 *
 * What it computes (eq_relg_0 / eq_relg, with the
 * equiradius obstacle algebra of L343-L360, eq_ORP / eq_convgP, specialised
 * per pair to indicator primitives):
 *
 *   g(R, t) = < f_A , f_{RB} o T^{-1} > = integral rho_A(x) rho_{RB}(x - t) dx
 *
 *   rho_A(x)  = sum_i w_i 1{ |x - a_i| <= r_i }          (eq_un: union -> sum)
 *   rho_RB(x) = sum_j v_j 1{ |x - R b_j| <= s_j }         (eq_Mink0: balls move
 *                                                          by relocating centres)
 *   =>  f_R(t) = sum_{i,j} w_i v_j V(r_i, s_j, |a_i - R b_j - t|)
 *
 * The obstacle knot of pair (i,j) sits at a_i - R b_j (P_O|_R = P_1 (+) (-R P_2),
 * L347-L352) and the primitive obstacle kernel f_{B_O} = f_{B_1} * f_{B_2}
 * (L355-L360) is, for indicator primitives (the alpha -> infinity limit of
 * eq_psi), the two-ball intersection ("lens") volume V(r, s, d):
 *
 *   V = (4/3) pi min(r,s)^3                                 d <= |r - s|
 *     = pi (r+s-d)^2 (d^2 + 2 d (r+s) - 3 (r-s)^2) / (12 d)  |r-s| < d < r+s
 *     = 0                                                   d >= r + s
 *
 * Complex weights (docking) follow reading C-3: f is defined
 * without conjugation, so pair weight = w_i * v_j.
 *
 * Grid: t_m = t0 + m h, m in [0, N)^3, output index (mx*N + my)*N + mz
 * (C order, z fastest).
 *
 * Parity status: V pinned by closed-form integrals, Monte Carlo and limits;
 * the pair sum pinned by brute force, swap symmetry, rotation covariance and
 * the total-mass identity (tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_PI 3.14159265358979323846

/* Two-ball intersection volume; d is the centre distance. */
double oracle_lens_volume(double r, double s, double d)
{
    if (d < 0) d = -d;
    if (d >= r + s) return 0.0;
    double m = r < s ? r : s;
    if (d <= fabs(r - s)) return 4.0 / 3.0 * ORACLE_PI * m * m * m;
    double a = r + s - d;
    return ORACLE_PI * a * a * (d * d + 2.0 * d * (r + s) - 3.0 * (r - s) * (r - s)) / (12.0 * d);
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Rotated B centres c_j = R b_j (action x -> R x). */
static void rotate_centres(const double *B, int64_t nB, const double *R, double *out)
{
    for (int64_t j = 0; j < nB; j++) {
        const double *b = B + 4 * j;
        for (int k = 0; k < 3; k++)
            out[3 * j + k] = R[3 * k + 0] * b[0] + R[3 * k + 1] * b[1] + R[3 * k + 2] * b[2];
    }
}

/*
 * f_R on the sub-box m in [lo, hi) (per axis) of the N^3 grid.
 * A, B: n x 4 rows (x, y, z, r).  wA_re/wB_re: real parts (NULL => 1);
 * wA_im/wB_im: imaginary parts (NULL => 0).  R: 9 doubles row-major.
 * out_re (and out_im if non-NULL) are full N^3 arrays; only the sub-box is
 * written (overwritten, not accumulated).
 * Threads own x-slabs: no atomics, a fixed summation order (pairs i-major).
 */
void oracle_correlate_grid(const double *A, const double *wA_re, const double *wA_im, int64_t nA,
                           const double *B, const double *wB_re, const double *wB_im, int64_t nB,
                           const double *R, int64_t N, double h, const double *t0,
                           const int64_t *lo, const int64_t *hi,
                           double *out_re, double *out_im)
{
    double *c = (double *)malloc(sizeof(double) * 3 * (size_t)(nB > 0 ? nB : 1));
    rotate_centres(B, nB, R, c);
    double smax = 0.0;
    for (int64_t j = 0; j < nB; j++) smax = B[4 * j + 3] > smax ? B[4 * j + 3] : smax;
    double cxmin = 1e300, cxmax = -1e300;
    for (int64_t j = 0; j < nB; j++) {
        cxmin = c[3 * j] < cxmin ? c[3 * j] : cxmin;
        cxmax = c[3 * j] > cxmax ? c[3 * j] : cxmax;
    }

#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t mx = lo[0]; mx < hi[0]; mx++) {
        const double tx = t0[0] + (double)mx * h;
        for (int64_t my = lo[1]; my < hi[1]; my++)
            for (int64_t mz = lo[2]; mz < hi[2]; mz++) {
                int64_t idx = (mx * N + my) * N + mz;
                out_re[idx] = 0.0;
                if (out_im) out_im[idx] = 0.0;
            }
        for (int64_t i = 0; i < nA; i++) {
            const double *a = A + 4 * i;
            /* x-extent prefilter: every pair centre has x in a_x - [cxmin, cxmax] */
            if (a[0] - cxmax - tx >= a[3] + smax) continue;
            if (tx - (a[0] - cxmin) >= a[3] + smax) continue;
            double wr = wA_re ? wA_re[i] : 1.0, wi = wA_im ? wA_im[i] : 0.0;
            for (int64_t j = 0; j < nB; j++) {
                double px = a[0] - c[3 * j + 0];
                double rs = a[3] + B[4 * j + 3];
                double dx = px - tx;
                if (fabs(dx) >= rs) continue;
                double py = a[1] - c[3 * j + 1];
                double pz = a[2] - c[3 * j + 2];
                double vr = wB_re ? wB_re[j] : 1.0, vi = wB_im ? wB_im[j] : 0.0;
                double pr = wr * vr - wi * vi, pi_ = wr * vi + wi * vr;
                /* grid index range of the pair's support along y, z */
                int64_t y0 = (int64_t)ceil((py - rs - t0[1]) / h), y1 = (int64_t)floor((py + rs - t0[1]) / h);
                int64_t z0 = (int64_t)ceil((pz - rs - t0[2]) / h), z1 = (int64_t)floor((pz + rs - t0[2]) / h);
                if (y0 < lo[1]) y0 = lo[1];
                if (y1 > hi[1] - 1) y1 = hi[1] - 1;
                if (z0 < lo[2]) z0 = lo[2];
                if (z1 > hi[2] - 1) z1 = hi[2] - 1;
                for (int64_t my = y0; my <= y1; my++) {
                    double dy = py - (t0[1] + (double)my * h);
                    for (int64_t mz = z0; mz <= z1; mz++) {
                        double dz = pz - (t0[2] + (double)mz * h);
                        double d = sqrt(dx * dx + dy * dy + dz * dz);
                        double v = oracle_lens_volume(a[3], B[4 * j + 3], d);
                        if (v == 0.0) continue;
                        int64_t idx = (mx * N + my) * N + mz;
                        out_re[idx] += pr * v;
                        if (out_im) out_im[idx] += pi_ * v;
                    }
                }
            }
        }
    }
    free(c);
}

/*
 * f_R at an explicit list of grid indices (flat C-order index into N^3),
 * brute force over ALL pairs with no pruning at all (the definition as
 * written).  Parallel over points.
 */
void oracle_correlate_points(const double *A, const double *wA_re, const double *wA_im, int64_t nA,
                             const double *B, const double *wB_re, const double *wB_im, int64_t nB,
                             const double *R, int64_t N, double h, const double *t0,
                             const int64_t *flat_idx, int64_t n_pts,
                             double *out_re, double *out_im)
{
    double *c = (double *)malloc(sizeof(double) * 3 * (size_t)(nB > 0 ? nB : 1));
    rotate_centres(B, nB, R, c);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < n_pts; p++) {
        int64_t f = flat_idx[p];
        int64_t mz = f % N, my = (f / N) % N, mx = f / (N * N);
        double t[3] = {t0[0] + (double)mx * h, t0[1] + (double)my * h, t0[2] + (double)mz * h};
        double acc_r = 0.0, acc_i = 0.0;
        for (int64_t i = 0; i < nA; i++) {
            const double *a = A + 4 * i;
            double wr = wA_re ? wA_re[i] : 1.0, wi = wA_im ? wA_im[i] : 0.0;
            for (int64_t j = 0; j < nB; j++) {
                double dx = a[0] - c[3 * j + 0] - t[0];
                double dy = a[1] - c[3 * j + 1] - t[1];
                double dz = a[2] - c[3 * j + 2] - t[2];
                double v = oracle_lens_volume(a[3], B[4 * j + 3], sqrt(dx * dx + dy * dy + dz * dz));
                if (v == 0.0) continue;
                double vr = wB_re ? wB_re[j] : 1.0, vi = wB_im ? wB_im[j] : 0.0;
                acc_r += (wr * vr - wi * vi) * v;
                acc_i += (wr * vi + wi * vr) * v;
            }
        }
        out_re[p] = acc_r;
        if (out_im) out_im[p] = acc_i;
    }
    free(c);
}
