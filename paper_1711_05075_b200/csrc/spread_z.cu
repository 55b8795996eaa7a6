// spread_z.cu -- fused spreading of R B + z axis of its box DFT (real weights, sm_100a).
//
// Same quantity as spread.cu followed by the z pass of passes.cu, with a compact window phi
// in place of the Gaussian: the smoothed knot density rho_s(x_n) = sum_j v_j (1_{B(R b_j, s_j)}
// * phi)(x_n) on the fine box
// (PAPER.md L150 eq_rhoP relocated by the rotation, eq_rhoAtrans; ball primitive
// eq_ballconv), immediately transformed along z:
//     T1[ix][iy][kz] = mult_z(kz) sum_{n<L} rho_s(ix, iy, n) exp(-2 pi i kz n / G),  kz in [0, K].
// The box never reaches HBM.
//
// Block = 4 x 4 columns (full z).  Spreading: warp w owns columns 2w, 2w+1 (one per
// half-warp); lane hl of a half owns the cells z = hl (mod 16) of its column and adds the
// candidate balls in list order (deterministic, no atomics).  The radial profile of a ball
// smoothed by a radial window of support U (the KB blob, api.cu), in cell units,
//     g(s, d) = Phi1(s - d) + Phi1(s + d) - (Phi2(s - d) - Phi2(s + d)) / d,
// is read from one universal cubic table of (Phi1, Phi2) over u in [-U, U] (beyond it
// Phi1 = +-1/2, Phi2 = 0) held in shared memory; near the centre (d < 0.1 cells) the series
// g(s, d) = g0(s) + g2(s) d^2 (per-ball constants) avoids the 1/d cancellation.
// Transform: columns (2l, 2l+1) form one complex line z = a + i b; its c coset FFTs give
// Z(k) on the band |k| <= K, and A(k) = (Z(k) + conj Z(-k)) / 2, B(k) = (Z(k) - conj Z(-k)) / 2i.
#include <algorithm>

#include "kernels.cuh"
#include "fft_ct.cuh"

using namespace fct;

namespace {

constexpr int SZ_COLS = 16;    // columns per block (4 x 4)
constexpr int SZ_LINES = 8;    // complex lines (column pairs)
constexpr int SZ_LCAP = 256;   // candidate list chunk

struct PhiVal {
    float p1, p2;
};

// (Phi1, Phi2)(u) from the cubic pieces; u is clamped to the table, whose end knots carry the
// exact limits (Phi1(+-U) = +-1/2, Phi2(+-U) = 0, zero slopes), so no range branch is needed.
__device__ __forceinline__ PhiVal phi_lookup(const float4 *__restrict__ tab, float tmax, float U, float invD, float u)
{
    const float t = fminf(fmaxf((u + U) * invD, 0.f), tmax);
    const int i = (int)t;
    const float f = t - (float)i;
    const float4 a = tab[2 * i], b = tab[2 * i + 1];
    return PhiVal{fmaf(f, fmaf(f, fmaf(f, a.w, a.z), a.y), a.x), fmaf(f, fmaf(f, fmaf(f, b.w, b.z), b.y), b.x)};
}

}  // namespace

// FFT phase: NG = 128 / TPL thread groups (the other half of the block idles) keep the
// exchange buffer small enough for 3 blocks / SM.
template <int L>
__global__ void __launch_bounds__(256, 3) spread_z_kernel(SpreadZArgs a)
{
    constexpr int TPL = Plan<L>::TPL, E = L / TPL, NG = 128 / TPL;
    constexpr int LS = line_stride(L);
    static_assert(256 % TPL == 0 && Plan<L>::n == 2, "spread_z plan");
    extern __shared__ float4 smz[];
    const int K = a.K, M = 2 * a.K + 1, Kz = a.K + 1;
    // layout: phi table | tw | Abuf (NG lines) | region {acc + lists  /  zb}
    float4 *phi = smz;
    float2 *tw = (float2 *)(phi + 2 * a.phi_n);
    float2 *Abuf = tw + L;
    constexpr int CS = L + 16;                        // column stride: the two half-warps of a warp
                                                      // (adjacent columns) sit 16 banks apart
    float *acc = (float *)(Abuf + NG * LS);           // [16][CS]
    float4 *sb = (float4 *)(acc + SZ_COLS * CS);      // [LCAP] (ux, uy, uz, rc^2)
    float4 *sw = sb + SZ_LCAP;                        // [LCAP] (s, w, g0, g2)
    float2 *zb = (float2 *)acc;                       // [8][M] (after the spread)
    __shared__ int wcount[8];
    __shared__ int list_n;

    const int b = blockIdx.y;
    const int tpa = L / 4;
    const int X0 = (blockIdx.x / tpa) * 4, Y0 = (blockIdx.x % tpa) * 4;
    float2 *T1 = a.out + (long long)b * a.out_bstride;

    // tiles outside B's (rotation-invariant) support cylinder: T1 rows are zero
    {
        const float dx = fmaxf(fmaxf((float)X0 - a.cx, a.cx - (float)(X0 + 3)), 0.f);
        const float dy = fmaxf(fmaxf((float)Y0 - a.cy, a.cy - (float)(Y0 + 3)), 0.f);
        if (dx * dx + dy * dy > a.live_r2) {
            for (int e = threadIdx.x; e < SZ_COLS * Kz; e += 256) {
                const int col = e / Kz, k = e % Kz;
                T1[((long long)(X0 + (col >> 2)) * L + Y0 + (col & 3)) * Kz + k] = make_float2(0.f, 0.f);
            }
            return;
        }
    }

    for (int e = threadIdx.x; e < 2 * a.phi_n; e += 256) phi[e] = a.phi[e];
    for (int e = threadIdx.x; e < L; e += 256) tw[e] = a.tw[e];
    for (int e = threadIdx.x; e < SZ_COLS * CS; e += 256) acc[e] = 0.f;

    float R[9];
#pragma unroll
    for (int q = 0; q < 9; q++) R[q] = a.rot[9 * b + q];

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int h = lane >> 4, hl = lane & 15;
    const int col = 2 * wid + h;
    const float fx = (float)(X0 + (col >> 2)), fy = (float)(Y0 + (col & 3));
    float *accc = acc + col * CS;
    const float fyw = (float)(Y0 + ((2 * wid) & 3));  // the warp's columns: (fx, fyw) and (fx, fyw + 1)
    const float fX0 = (float)X0, fY0 = (float)Y0;
    const float U = a.phi_U, invD = a.phi_invD;
    const float tmax = (float)a.phi_n - 1e-3f;
    if (threadIdx.x == 0) list_n = 0;
    __syncthreads();

    const int nb_ = a.n_balls;
    int base = 0;
    while (base < nb_) {
        // ---- candidate list (order-preserving compaction) until full or exhausted
        while (base < nb_) {
            const int cnt0 = list_n;
            if (cnt0 + 256 > SZ_LCAP) break;
            const int j = base + threadIdx.x;
            bool ok = false;
            float4 u = make_float4(0, 0, 0, 0);
            if (j < nb_) {
                const float4 bl = a.balls[j];  // (x, y, z, s) in cells, B frame
                // eq_Mink0 (L235): the rigid motion relocates the centre only
                u.x = R[0] * bl.x + R[1] * bl.y + R[2] * bl.z - a.ox;
                u.y = R[3] * bl.x + R[4] * bl.y + R[5] * bl.z - a.oy;
                u.z = R[6] * bl.x + R[7] * bl.y + R[8] * bl.z - a.oz;
                const float rc = bl.w + a.cut;
                u.w = rc * rc;
                const float dx = fmaxf(fmaxf(fX0 - u.x, u.x - (fX0 + 3.f)), 0.f);
                const float dy = fmaxf(fmaxf(fY0 - u.y, u.y - (fY0 + 3.f)), 0.f);
                ok = dx * dx + dy * dy < u.w;
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
                const float2 g = a.g02[j];
                sw[pos] = make_float4(a.balls[j].w, a.w[j], g.x, g.y);
            }
            base += 256;
            __syncthreads();
            if (threadIdx.x == 0) list_n = cnt0 + total;
            __syncthreads();
        }
        // ---- accumulate the list into this lane's cells.  A half-warp covers the ball's chord
        // of its column in 16-cell steps from the chord start: within a step the lanes touch
        // distinct cells, steps and balls are sequential, so the sums are race-free and in
        // list order (deterministic).
        const int total = list_n;
        for (int base0 = 0; base0 < total; base0 += 32) {
            // the candidates that reach one of this warp's two columns (ballot, list order kept)
            bool rel = false;
            if (base0 + lane < total) {
                const float4 uc = sb[base0 + lane];
                const float ddx = fx - uc.x;
                const float ddy = fmaxf(fmaxf(fyw - uc.y, uc.y - (fyw + 1.f)), 0.f);
                rel = fmaf(ddx, ddx, ddy * ddy) < uc.w;
            }
            unsigned msk = __ballot_sync(0xffffffffu, rel);
        while (msk) {
            const int e = base0 + __ffs(msk) - 1;
            msk &= msk - 1;
            const float4 ue = sb[e];
            const float dx = fx - ue.x, dy = fy - ue.y;
            const float dxy2 = fmaf(dx, dx, dy * dy);
            const float hz2 = ue.w - dxy2;
            int zlo = 0, zhi = -1, nit = 0;
            if (hz2 > 0.f) {
                const float hz = hz2 * rsqrtf(hz2);
                zlo = max(0, (int)ceilf(ue.z - hz));
                zhi = min(L - 1, (int)floorf(ue.z + hz));
                nit = (zhi - zlo + 16) >> 4;
            }
            const int nmax = max(nit, __shfl_xor_sync(0xffffffffu, nit, 16));
            if (nmax <= 0) continue;
            const float4 we = sw[e];  // (s, w, g0, g2)
            for (int it = 0; it < nmax; it++) {
                const int z = zlo + (it << 4) + hl;
                if (z <= zhi) {
                    const float dz = (float)z - ue.z;
                    const float d2 = fmaf(dz, dz, dxy2);
                    float g;
                    if (d2 < 0.01f) {
                        g = fmaf(we.w, d2, we.z);
                    } else {
                        const float rd = rsqrtf(d2);
                        const float d = d2 * rd;
                        const PhiVal p = phi_lookup(phi, tmax, U, invD, we.x - d);
                        PhiVal q = PhiVal{0.5f, 0.f};
                        if (we.x + d < U) q = phi_lookup(phi, tmax, U, invD, we.x + d);
                        g = p.p1 + q.p1 - (p.p2 - q.p2) * rd;
                    }
                    accc[z] = fmaf(we.y, g, accc[z]);
                }
            }
        }
        }
        __syncthreads();
        if (threadIdx.x == 0) list_n = 0;
        __syncthreads();
    }

    // ---- z transform: line l = columns (2l, 2l+1); group g handles line g % 8, cosets g/8 + (NG/8) r
    const int g = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const bool fft_thread = g < NG;
    const int line = g % SZ_LINES;
    float2 x[E];
#pragma unroll
    for (int m = 0; m < E; m++) {
        const int n = tl + TPL * m;
        x[m] = fft_thread ? make_float2(acc[(2 * line) * CS + n], acc[(2 * line + 1) * CS + n]) : make_float2(0.f, 0.f);
    }
    __syncthreads();  // acc / lists dead: zb may overwrite them
    const int c = a.c, G = a.G;
    const int rounds = (SZ_LINES * c + NG - 1) / NG;
    for (int r = 0; r < rounds; r++) {
        const int p = g / SZ_LINES + (NG / SZ_LINES) * r;
        const bool active = fft_thread && p < c;
        float2 y[E];
#pragma unroll
        for (int m = 0; m < E; m++) y[m] = (active && p) ? cmul(x[m], a.ctw[p * L + tl + TPL * m]) : x[m];
        float2 *ab = Abuf + (fft_thread ? g : g - NG) * LS;  // idle groups shadow the active ones' buffers
        if (fft_thread) {
            fft_regs<L, -1>(y, ab, ab, tw, tl);
        } else {
            // keep the block-wide barriers of fft_regs (stage 0 -> last stage) in step
            __syncthreads();
        }
        if (active) {
#pragma unroll
            for (int m = 0; m < E; m++) {
                int k = c * (tl + TPL * m) + p;
                if (2 * k > G) k -= G;
                if (k >= -K && k <= K) zb[line * M + k + K] = y[m];
            }
        }
        __syncthreads();
    }
    // ---- unpack the column pairs, multiply by mult_z, store T1 rows (contiguous in kz)
    for (int e = threadIdx.x; e < SZ_LINES * Kz; e += 256) {
        const int l = e / Kz, k = e % Kz;
        const float2 Z = zb[l * M + K + k], Zm = zb[l * M + K - k];
        const float2 mu = a.mult_z[k];
        const float2 Xa = cmul(make_float2(0.5f * (Z.x + Zm.x), 0.5f * (Z.y - Zm.y)), mu);
        const float2 Xb = cmul(make_float2(0.5f * (Z.y + Zm.y), -0.5f * (Z.x - Zm.x)), mu);
        const int ca = 2 * l, cb = 2 * l + 1;
        T1[((long long)(X0 + (ca >> 2)) * L + Y0 + (ca & 3)) * Kz + k] = Xa;
        T1[((long long)(X0 + (cb >> 2)) * L + Y0 + (cb & 3)) * Kz + k] = Xb;
    }
}

bool spread_z_supported(int L) { return L == 128 || L == 256; }

template <int L>
static void spread_z_launch(const SpreadZArgs &a, int batch, cudaStream_t s)
{
    constexpr int NG = 128 / Plan<L>::TPL;
    const int tpa = L / 4;
    const size_t region = std::max((size_t)SZ_COLS * (L + 16) * 4 + (size_t)SZ_LCAP * 32, (size_t)SZ_LINES * (2 * a.K + 1) * 8);
    const size_t sm = (size_t)a.phi_n * 32 + (size_t)L * 8 + (size_t)NG * line_stride(L) * 8 + region;
    static_assert(NG == 128 / Plan<L>::TPL, "spread_z FFT groups");
    cudaFuncSetAttribute(spread_z_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    spread_z_kernel<L><<<dim3(tpa * tpa, batch), 256, sm, s>>>(a);
}

void launch_spread_z(const SpreadZArgs &a, int batch, cudaStream_t s)
{
    switch (a.L) {
    case 128: spread_z_launch<128>(a, batch, s); break;
    case 256: spread_z_launch<256>(a, batch, s); break;
    default: break;
    }
}
