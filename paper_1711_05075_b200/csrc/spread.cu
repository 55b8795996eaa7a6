// spread.cu -- Gaussian-smoothed ball spreading onto the fine box (sm_100a).
//
// rho_s(x_n) = sum_j v_j (1_{B(R b_j, s_j)} * G_tau)(x_n): the knot density of
// PAPER.md L150 (eq_rhoP) relocated by the rotation (eq_rhoAtrans) and
// convolved with each ball primitive (eq_ballconv) and with an isotropic
// Gaussian G_tau.  Its box DFT divided by the Gaussian's transform
// exp(-2 pi^2 tau^2 |k/P|^2) is exactly sum_j v_j beta_hat(s_j, |k|/P) exp(-2 pi i k.R b_j/P)
// (eq_fballhat) up to the aliasing level eps the plan chooses tau for.
#include "kernels.cuh"

#include "ballcorr.h"

#define SP_T 16

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

// Block = 16^3-cell tile, 256 threads; thread t owns the z-column (x, y) of the tile
// and accumulates into its own shared-memory column (no atomics; balls are added in
// ball-index order, so the result is bitwise deterministic).  The block first
// compacts the candidate balls overlapping the tile (order-preserving) into a
// shared list, then every thread walks the list for its column.
// TABLE: the radial profile comes from the per-ball cubic-Hermite table
// (SpreadArgs::prof, built once per shape on the host from the same closed form);
// otherwise it is evaluated directly (smoothed_ball).
template <bool CPLX, bool TABLE>
__global__ void __launch_bounds__(256) spread_kernel(SpreadArgs a)
{
    constexpr int SP_LCAP = CPLX ? 448 : 768;  // static shared memory stays below 48 KB
    __shared__ float4 sb[SP_LCAP];
    __shared__ float4 sw[SP_LCAP];
    __shared__ int wcount[8];
    __shared__ int list_n;
    __shared__ float accr[SP_T * SP_T * SP_T];
    __shared__ float acci[CPLX ? SP_T * SP_T * SP_T : 1];

    const int b = blockIdx.y;
    const int tile = blockIdx.x;
    const int tpa = a.tiles_per_axis;
    const int tz = tile % tpa, ty = (tile / tpa) % tpa, tx = tile / (tpa * tpa);
    const int X0 = tx * SP_T, Y0 = ty * SP_T, Z0 = tz * SP_T;
    const int cx_ = threadIdx.x >> 4, cy_ = threadIdx.x & 15;
    const int x = X0 + cx_, y = Y0 + cy_;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // z-major: cell (column t, z) at [z * 256 + t] -> a warp touches 32 consecutive words
    float *col_r = accr + threadIdx.x;
    float *col_i = acci + (CPLX ? threadIdx.x : 0);
#pragma unroll
    for (int z = 0; z < SP_T; z++) {
        col_r[z * 256] = 0.f;
        if (CPLX) col_i[z * 256] = 0.f;
    }

    float R[9];
    if (a.rot) {
#pragma unroll
        for (int q = 0; q < 9; q++) R[q] = a.rot[9 * b + q];
    }

    int c0 = 0, ncand = a.n_balls;
    const int *cidx = a.csr_idx;
    if (a.csr_off) {
        c0 = a.csr_off[tile];
        ncand = a.csr_off[tile + 1] - c0;
    } else if (a.bin_counts) {  // B: this rotation's column bin (ball order)
        const int bin = tx * a.bpa + ty;
        ncand = a.bin_counts[b * a.nbins + bin];
        cidx = a.bin_lists + (long long)b * a.bin_stride + a.bin_offs[b * a.nbins + bin];
    }
    const float fx0 = (float)X0, fy0 = (float)Y0, fz0 = (float)Z0, fe = (float)(SP_T - 1);
    const float tau = a.tau;
    if (threadIdx.x == 0) list_n = 0;
    __syncthreads();

    int base = 0;
    while (base < ncand) {
        // ---- build the list (order-preserving compaction) until full or exhausted
        while (base < ncand) {
            const int cnt0 = list_n;
            if (cnt0 + 256 > SP_LCAP) break;
            const int q = base + threadIdx.x;
            bool ok = false;
            float4 u = make_float4(0, 0, 0, 0), wv = make_float4(0, 0, 0, 0);
            if (q < ncand) {
                const int j = cidx ? cidx[c0 + q] : q;
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
                    wv.x = TABLE ? __int_as_float(a.prof_off[j]) : bl.w;
                    wv.y = a.w_re ? a.w_re[j] : 1.f;
                    wv.z = (CPLX && a.w_im) ? a.w_im[j] : 0.f;
                }
            }
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
                const int pos = cnt0 + off + __popc(m & ((1u << lane) - 1u));
                sb[pos] = u;
                sw[pos] = wv;
            }
            base += 256;
            __syncthreads();
            if (threadIdx.x == 0) list_n = cnt0 + total;
            __syncthreads();
        }
        // ---- accumulate the list into this thread's column
        const int total = list_n;
        for (int e = 0; e < total; e++) {
            const float4 ue = sb[e];
            const float dx = (float)x - ue.x, dy = (float)y - ue.y;
            const float dxy2 = dx * dx + dy * dy;
            const float rc2 = ue.w * ue.w;
            if (dxy2 >= rc2) continue;
            const float hz = sqrtf(rc2 - dxy2);
            const int zlo = max(0, (int)ceilf(ue.z - hz - fz0));
            const int zhi = min(SP_T - 1, (int)floorf(ue.z + hz - fz0));
            if (zlo > zhi) continue;
            const float4 we = sw[e];
            for (int z = zlo; z <= zhi; z++) {
                const float dz = (fz0 + (float)z) - ue.z;
                const float d = sqrtf(dxy2 + dz * dz) * a.hf;
                float g;
                if (TABLE) {
                    const float uu = d * a.inv_dprof;
                    const int k = (int)uu;
                    const float t = uu - (float)k;
                    const float4 c = a.prof[__float_as_int(we.x) + k];
                    g = c.x + t * (c.y + t * (c.z + t * c.w));
                } else {
                    g = smoothed_ball(we.x, d, tau);
                }
                col_r[z * 256] += we.y * g;
                if (CPLX) col_i[z * 256] += we.z * g;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) list_n = 0;
        __syncthreads();
    }

    // write the tile: the 16 z-values of column (x, y) are contiguous in the box
    const int L = a.L;
    if (x < L && y < L) {
        const long long rowoff = (long long)b * a.out_batch_stride + ((long long)x * L + y) * L;
        if (CPLX) {
            float2 *o = (float2 *)a.out + rowoff;
#pragma unroll
            for (int z = 0; z < SP_T; z++)
                if (Z0 + z < L) o[Z0 + z] = make_float2(col_r[z * 256], col_i[z * 256]);
        } else {
            float *o = (float *)a.out + rowoff;
#pragma unroll
            for (int z = 0; z < SP_T; z++)
                if (Z0 + z < L) o[Z0 + z] = col_r[z * 256];
        }
    }
}

void launch_spread(const SpreadArgs &a, int batch, cudaStream_t s)
{
    const int tpa = a.tiles_per_axis;
    dim3 grid(tpa * tpa * tpa, batch);
    if (a.prof) {
        if (a.complex_w) spread_kernel<true, true><<<grid, 256, 0, s>>>(a);
        else spread_kernel<false, true><<<grid, 256, 0, s>>>(a);
    } else {
        if (a.complex_w) spread_kernel<true, false><<<grid, 256, 0, s>>>(a);
        else spread_kernel<false, false><<<grid, 256, 0, s>>>(a);
    }
}

