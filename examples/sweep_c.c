/*
 * A plain-C consumer of libballcorr (include/ballcorr.h): no Python, no torch.
 *
 * Builds a sweep-shaped workload (the BASELINE.json "sweep" recipe: A = 50,000 balls in the
 * cube shell [-0.4,0.4]^3 \ (-0.3,0.3)^3 with r ~ U[0.005,0.03]; B = 5,000 balls in the ball
 * of radius 0.2 with r ~ U[0.005,0.02]; N = 256 over [-1,1)^3) from its own xorshift
 * generator, runs the spectral sweep plan (Np = 256, K = 255) over a batch of rotations with
 * host buffers, and checks every rotation's grid extrema against the exact single-
 * configuration query at the same translations (bc_evaluate_points, fp64 pair-lens sum):
 * |f_grid - f_exact| <= 1e-4 max|f_exact| (the north_star tolerance).
 *
 *     make examples && ./examples/sweep_c [n_rot]
 *
 * Prints one line per rotation, the throughput of the host-buffer call, and "OK" (exit 0)
 * or the failure (exit 1).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include "ballcorr.h"

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static double urand(void) /* xorshift64*, uniform in [0, 1) */
{
    rng_state ^= rng_state >> 12;
    rng_state ^= rng_state << 25;
    rng_state ^= rng_state >> 27;
    return (double)((rng_state * 0x2545F4914F6CDD1Dull) >> 11) * 0x1.0p-53;
}
static double uni(double lo, double hi) { return lo + (hi - lo) * urand(); }

static void random_rotation(double *R) /* Shoemake: uniform unit quaternion -> matrix */
{
    const double u1 = urand(), u2 = 2 * M_PI * urand(), u3 = 2 * M_PI * urand();
    const double a = sqrt(1 - u1), b = sqrt(u1);
    const double w = a * sin(u2), x = a * cos(u2), y = b * sin(u3), z = b * cos(u3);
    const double m[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - z * w),     2 * (x * z + y * w),
                         2 * (x * y + z * w),     1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
                         2 * (x * z - y * w),     2 * (y * z + x * w),     1 - 2 * (x * x + y * y)};
    for (int i = 0; i < 9; i++) R[i] = m[i];
}

#define CHECK(call)                                                                            \
    do {                                                                                       \
        bc_status st_ = (call);                                                                \
        if (st_ != BC_OK) {                                                                    \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, bc_status_string(st_), bc_last_error(ctx)); \
            return 1;                                                                          \
        }                                                                                      \
    } while (0)

int main(int argc, char **argv)
{
    const int n_rot = argc > 1 ? atoi(argv[1]) : 16;
    const int nA = 50000, nB = 5000, N = 256;
    double *A = malloc(sizeof(double) * 4 * nA), *B = malloc(sizeof(double) * 4 * nB);
    double *R = malloc(sizeof(double) * 9 * n_rot);
    bc_extremum *mm = malloc(sizeof(bc_extremum) * 2 * n_rot);
    if (n_rot < 1 || !A || !B || !R || !mm) return 1;
    for (int i = 0; i < nA;) { /* cube shell by rejection */
        const double x = uni(-0.4, 0.4), y = uni(-0.4, 0.4), z = uni(-0.4, 0.4);
        if (fabs(x) < 0.3 && fabs(y) < 0.3 && fabs(z) < 0.3) continue;
        A[4 * i] = x, A[4 * i + 1] = y, A[4 * i + 2] = z, A[4 * i + 3] = uni(0.005, 0.03);
        i++;
    }
    for (int j = 0; j < nB;) { /* solid ball of radius 0.2 by rejection */
        const double x = uni(-0.2, 0.2), y = uni(-0.2, 0.2), z = uni(-0.2, 0.2);
        if (x * x + y * y + z * z >= 0.04) continue;
        B[4 * j] = x, B[4 * j + 1] = y, B[4 * j + 2] = z, B[4 * j + 3] = uni(0.005, 0.02);
        j++;
    }
    for (int r = 0; r < n_rot; r++) random_rotation(R + 9 * r);

    bc_ctx *ctx = NULL;
    bc_params p = {0};
    p.N = N, p.h = 2.0 / N, p.t0[0] = p.t0[1] = p.t0[2] = -1.0;
    p.Np = 256, p.K = 255, p.precision = BC_FP32, p.mode = BC_MODE_SPECTRAL, p.weights = BC_WEIGHTS_REAL;
    CHECK(bc_create(0, &p, &ctx));
    CHECK(bc_shape_upload(ctx, 0, A, NULL, nA));
    CHECK(bc_shape_upload(ctx, 1, B, NULL, nB));
    CHECK(bc_spectrum_A(ctx, NULL));
    CHECK(bc_correlate_rotations(ctx, R, n_rot, BC_OUT_MINMAX, mm, NULL)); /* warm-up */

    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    CHECK(bc_correlate_rotations(ctx, R, n_rot, BC_OUT_MINMAX, mm, NULL));
    clock_gettime(CLOCK_MONOTONIC, &t1);
    const double sec = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);

    /* exact f at each rotation's grid argmin and argmax */
    double *Rq = malloc(sizeof(double) * 9 * 2 * n_rot), *tq = malloc(sizeof(double) * 3 * 2 * n_rot);
    double *fq = malloc(sizeof(double) * 2 * n_rot);
    for (int r = 0; r < n_rot; r++)
        for (int e = 0; e < 2; e++) {
            const int64_t idx = mm[2 * r + e].idx;
            const int64_t m[3] = {idx / ((int64_t)N * N), (idx / N) % N, idx % N};
            for (int i = 0; i < 9; i++) Rq[9 * (2 * r + e) + i] = R[9 * r + i];
            for (int i = 0; i < 3; i++) tq[3 * (2 * r + e) + i] = p.t0[i] + p.h * (double)m[i];
        }
    CHECK(bc_evaluate_points(ctx, Rq, tq, 2 * n_rot, fq, NULL));
    double scale = 0;
    for (int q = 0; q < 2 * n_rot; q++) scale = fmax(scale, fabs(fq[q]));
    int bad = 0;
    for (int r = 0; r < n_rot; r++) {
        const double emin = fabs(mm[2 * r].val - fq[2 * r]), emax = fabs(mm[2 * r + 1].val - fq[2 * r + 1]);
        printf("rot %d  min %.6e @ %lld (exact %.6e)  max %.6e @ %lld (exact %.6e)\n", r, mm[2 * r].val,
               (long long)mm[2 * r].idx, fq[2 * r], mm[2 * r + 1].val, (long long)mm[2 * r + 1].idx, fq[2 * r + 1]);
        if (emin > 1e-4 * scale || emax > 1e-4 * scale) bad++;
    }
    printf("host-buffer call: %d rotations in %.3f ms = %.3e translations*rotations/s\n", n_rot, sec * 1e3,
           (double)n_rot * N * N * N / sec);
    bc_destroy(ctx);
    printf(bad ? "FAIL: %d rotations outside 1e-4 max|f|\n" : "OK\n", bad);
    free(A), free(B), free(R), free(mm), free(Rq), free(tq), free(fq);
    return bad ? 1 : 0;
}
