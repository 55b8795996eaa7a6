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
#include <type_traits>

#include "kernels.cuh"
#include "fft_ct.cuh"

using namespace fct;

namespace {

constexpr int SZ_COLS = 16;    // columns per block (4 x 4)
constexpr int SZ_LINES = 8;    // complex lines (column pairs)
constexpr int SZ_BIN = 16;     // binning: 16 x 16 columns
constexpr int SZ_PHI_N = 96;   // profile table pieces over [-W, W], W = 4 cells
constexpr int ZB_RP = 132;     // coset row pitch of the band-4 z staging (= 4 mod 16 8-byte slots: the
                               // unpack reads of 4 cosets x 4 slots per half-warp are distinct)
constexpr float SZ_PHI_U = 4.f;

struct PhiVal {
    float p1, p2;
};

// (Phi1, Phi2)(u) from the cubic pieces; u is clamped to the table, whose end knots carry the
// exact limits (Phi1(+-U) = +-1/2, Phi2(+-U) = 0, zero slopes), so no range branch is needed.
// tab = [n] Phi1 pieces followed by [n] Phi2 pieces (split arrays: a 16-byte load at a random
// piece hits one of 8 bank groups, where interleaved 32-byte records would hit one of 4)
__device__ __forceinline__ PhiVal phi_lookup(const float4 *__restrict__ tab, int n, float tmax, float U, float invD, float u)
{
    const float t = fminf(fmaxf((u + U) * invD, 0.f), tmax);
    const int i = (int)t;
    const float f = t - (float)i;
    const float4 a = tab[i], b = tab[n + i];
    return PhiVal{fmaf(f, fmaf(f, fmaf(f, a.w, a.z), a.y), a.x), fmaf(f, fmaf(f, fmaf(f, b.w, b.z), b.y), b.x)};
}

// the same at the table coordinate t = (u + U) / D, unclamped (callers form it with one FFMA)
__device__ __forceinline__ PhiVal phi_lookup_t(const float4 *__restrict__ tab, int n, float tmax, float t)
{
    t = fminf(fmaxf(t, 0.f), tmax);
    const int i = (int)t;
    const float f = t - (float)i;
    const float4 a = tab[i], b = tab[n + i];
    return PhiVal{fmaf(f, fmaf(f, fmaf(f, a.w, a.z), a.y), a.x), fmaf(f, fmaf(f, fmaf(f, b.w, b.z), b.y), b.x)};
}

}  // namespace

// ============================================================================ per-rotation binning
// recA[b][j] = (R b_j / hf - o, (s_j + W)^2) in box cells; the moving ball's footprint disk
// (radius s_j + W around its centre) is listed, in ball order, in every 16 x 16-column bin
// of the box it reaches.  Counting pass, then a fill pass whose blocks find their own
// offsets by summing the counts of the bins before them (no separate scan, deterministic).
__global__ void szb_rotate_kernel(SzBinArgs a)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x, b = blockIdx.y;
    if (j >= a.n) return;
    const float *R = a.rot + 9 * b;
    const float4 bl = a.balls[j];  // (x, y, z, s) in cells, B frame
    // eq_Mink0 (L235): the rigid motion relocates the centre only
    const float rc = bl.w + a.cut;
    a.recA[(long long)b * a.n + j] = make_float4(R[0] * bl.x + R[1] * bl.y + R[2] * bl.z - a.ox,
                                                 R[3] * bl.x + R[4] * bl.y + R[5] * bl.z - a.oy,
                                                 R[6] * bl.x + R[7] * bl.y + R[8] * bl.z - a.oz, rc * rc);
}

__device__ __forceinline__ bool szb_hits(float4 u, int bin, int bpa)
{
    const float x0 = (float)((bin / bpa) * SZ_BIN), y0 = (float)((bin % bpa) * SZ_BIN);
    const float dx = fmaxf(fmaxf(x0 - u.x, u.x - (x0 + (SZ_BIN - 1))), 0.f);
    const float dy = fmaxf(fmaxf(y0 - u.y, u.y - (y0 + (SZ_BIN - 1))), 0.f);
    return dx * dx + dy * dy < u.w;
}

__global__ void __launch_bounds__(256) szb_count_kernel(SzBinArgs a)
{
    const int bin = blockIdx.x, b = blockIdx.y;
    const float4 *rec = a.recA + (long long)b * a.n;
    int cnt = 0;
    for (int j = threadIdx.x; j < a.n; j += 256) cnt += szb_hits(rec[j], bin, a.bpa) ? 1 : 0;
    __shared__ int red[8];
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < 8; w++) t += red[w];
        a.counts[b * a.nbins + bin] = t;
    }
}

__global__ void __launch_bounds__(256) szb_fill_kernel(SzBinArgs a)
{
    const int bin = blockIdx.x, b = blockIdx.y;
    const float4 *rec = a.recA + (long long)b * a.n;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ int red[8];
    __shared__ int base_s;
    int s = 0;
    for (int k = threadIdx.x; k < bin; k += 256) s += a.counts[b * a.nbins + k];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[wid] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < 8; w++) t += red[w];
        a.offs[b * a.nbins + bin] = t;
        base_s = t;
    }
    __syncthreads();
    int pos0 = base_s;
    int *lst = a.lists + (long long)b * a.list_stride;
    for (int j0 = 0; j0 < a.n; j0 += 256) {
        const int j = j0 + threadIdx.x;
        const bool ok = j < a.n && szb_hits(rec[j], bin, a.bpa);
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        __syncthreads();
        if (lane == 0) red[wid] = __popc(m);
        __syncthreads();
        int off = 0, total = 0;
#pragma unroll
        for (int w = 0; w < 8; w++) {
            off += (w < wid) ? red[w] : 0;
            total += red[w];
        }
        if (ok) lst[pos0 + off + __popc(m & ((1u << lane) - 1u))] = j;
        pos0 += total;
    }
}

// ============================================================================ spread + z transform
// Block = 128 threads, 4 x 4 columns (full z).  Spreading: warp w owns the 4 columns
// (X0 + w, Y0 + g), g = lane / 8; the 8 lanes of a group step along the ball's chord of
// their column 8 cells at a time (a ~15-cell chord takes 2 steps at ~94% lane use), so one
// ball visit serves 4 columns.  FFT phase: 128 / TPL thread groups, one pair-line each.
// The z transform of one 4 x 4 column tile held in shared memory (acc[16][CS] fp32):
// columns (2l, 2l+1) form one complex line z = a + i b; group g (TPL threads) handles line
// g % 8 and cosets g / 8 + (NG / 8) r; the band of Z(k), |k| <= K, goes to zb[8][2K + 1]
// (aliasing acc once the lines are in registers); A(k) = (Z(k) + conj Z(-k)) / 2,
// B(k) = (Z(k) - conj Z(-k)) / 2i, times mult_z, are stored as T1 rows.
// B4: the sweep plan's band (c = 4, G = 1024, K = 255) as compile-time constants
template <int L, int NT, bool B4 = false>
__device__ __forceinline__ void tile_z_transform(const SpreadZArgs &a, float *acc, float2 *Abuf, const float2 *tw,
                                                 float2 *T1, int X0, int Y0)
{
    constexpr int TPL = Plan<L>::TPL, E = L / TPL, NG = NT / TPL;
    constexpr int LS = line_stride(L);
    constexpr int CS = L + 8;
    const int K = B4 ? 255 : a.K, M = 2 * K + 1, Kz = K + 1;
    float2 *zb = (float2 *)acc;
    const int g = threadIdx.x / TPL, tl = threadIdx.x % TPL;
    const int line = g % SZ_LINES;
    float2 x[E];
#pragma unroll
    for (int m = 0; m < E; m++) {
        const int n = tl + TPL * m;
        x[m] = make_float2(acc[(2 * line) * CS + n], acc[(2 * line + 1) * CS + n]);
    }
    __syncthreads();  // acc dead: zb may overwrite it
    const int c = B4 ? 4 : a.c, G = B4 ? 1024 : a.G;
    const bool band4 = B4 || (c == 4 && G == 1024 && K == 255);  // block-uniform
    const int rounds = (SZ_LINES * c + NG - 1) / NG;
    for (int r = 0; r < rounds; r++) {
        const int p = g / SZ_LINES + (NG / SZ_LINES) * r;
        const bool active = p < c;
        // coset twiddle e^{-2 pi i p n / G} at n = tl + TPL m: the lane's first value times the
        // step e^{-2 pi i p TPL / G}, by recurrence (E steps, ~E ulp)
        float2 y[E];
        if (active && p) {
            float2 t = a.ctw[p * L + tl];
            const float2 Wp = a.ctw[p * L + TPL];
#pragma unroll
            for (int m = 0; m < E; m++) {
                y[m] = cmul(x[m], t);
                t = cmul(t, Wp);
            }
        } else {
#pragma unroll
            for (int m = 0; m < E; m++) y[m] = x[m];
        }
        fft_regs<L, -1, true>(y, Abuf + g * LS, Abuf + g * LS, tw, tl);
        if (L == 256 && band4) {
            // plan L = 256, c = 4, K = 255: outputs m < 4 (k = 4q + p) and m >= 12
            // (k = 4q + p - 1024) are the band, minus (p, q) = (0, 192).  Stored coset-major,
            // zb[line][p][s] (s = q, or q - 128 for q >= 192; rows of ZB_RP): a half-warp's
            // consecutive q land in consecutive 8-byte slots (the k-ordered row put lanes 32
            // bytes apart: 4-way bank conflicts)
#pragma unroll
            for (int m = 0; m < E; m++) {
                if (m >= 4 && m < 12) continue;
                const int q = tl + TPL * m;
                zb[line * (4 * ZB_RP) + p * ZB_RP + (m < 4 ? q : q - 128)] = y[m];
            }
        } else if (active) {
#pragma unroll
            for (int m = 0; m < E; m++) {
                int k = c * (tl + TPL * m) + p;
                if (2 * k > G) k -= G;
                if (k >= -K && k <= K) zb[line * M + k + K] = y[m];
            }
        }
        __syncwarp();  // the next round's FFT rewrites this group's buffer
    }
    __syncthreads();  // zb complete
    if (L == 256 && band4) {  // the coset-major zb above: Z(k) at (k & 3, k >> 2), Z(-k) at
                              // ((-k) & 3, ((1024 - k) >> 2) - 128) for k >= 1
#pragma unroll 1
        for (int l = 0; l < SZ_LINES; l++) {
            const int ca = 2 * l, cb = 2 * l + 1;
            float2 *Ta = T1 + ((long long)(X0 + (ca >> 2)) * L + Y0 + (ca & 3)) * Kz;
            float2 *Tb = T1 + ((long long)(X0 + (cb >> 2)) * L + Y0 + (cb & 3)) * Kz;
            const float2 *zl = zb + l * (4 * ZB_RP);
            for (int k = threadIdx.x; k < Kz; k += NT) {
                const float2 Z = zl[(k & 3) * ZB_RP + (k >> 2)];
                const float2 Zm = k ? zl[((-k) & 3) * ZB_RP + ((1024 - k) >> 2) - 128] : Z;
                const float2 za = make_float2(0.5f * (Z.x + Zm.x), 0.5f * (Z.y - Zm.y));
                const float2 zb2 = make_float2(0.5f * (Z.y + Zm.y), -0.5f * (Z.x - Zm.x));
                if (a.mult_z) {  // (nullptr: mult_z folded into A'', permute_cm_kernel)
                    const float2 mu = a.mult_z[k];
                    Ta[k] = cmul(za, mu);
                    Tb[k] = cmul(zb2, mu);
                } else {
                    Ta[k] = za;
                    Tb[k] = zb2;
                }
            }
        }
        return;
    }
#pragma unroll 1
    for (int l = 0; l < SZ_LINES; l++) {  // line l = columns 2l (real part) and 2l + 1 (imaginary)
        const int ca = 2 * l, cb = 2 * l + 1;
        float2 *Ta = T1 + ((long long)(X0 + (ca >> 2)) * L + Y0 + (ca & 3)) * Kz;
        float2 *Tb = T1 + ((long long)(X0 + (cb >> 2)) * L + Y0 + (cb & 3)) * Kz;
        const float2 *zl = zb + l * M + K;
        for (int k = threadIdx.x; k < Kz; k += NT) {
            const float2 Z = zl[k], Zm = zl[-k];
            const float2 mu = a.mult_z ? a.mult_z[k] : make_float2(1.f, 0.f);  // (nullptr: folded into A'')
            Ta[k] = cmul(make_float2(0.5f * (Z.x + Zm.x), 0.5f * (Z.y - Zm.y)), mu);
            Tb[k] = cmul(make_float2(0.5f * (Z.y + Zm.y), -0.5f * (Z.x - Zm.x)), mu);
        }
    }
}

// BOX = false: spread + z transform of the tile (one kernel).  BOX = true: spread only, the
// tile's 16 fp32 columns are written to the box (a.box) for pass_z_fast; without the FFT's
// registers and buffers the spread runs at twice the occupancy.  CPLX (BOX only): complex
// weights w = (recB.y, recWi), two accumulators per cell, float2 box cells (the z transform
// is then the complex-row pass of passes.cu, which skips the tiles left unwritten here).
// Accumulator slot -> column of the 4 x 4 tile.  Slot 4 w + g belongs to warp w, lane group g.
// QUAD: warp w owns the 2 x 2 quadrant (2 (w >> 1), 2 (w & 1)); else the 1 x 4 strip x = w.
// The slots (not the columns) index acc, so the groups' rows stay 8 banks apart either way.
template <bool QUAD>
__device__ __forceinline__ int slot_x(int s) { return QUAD ? 2 * (s >> 3) + ((s >> 1) & 1) : s >> 2; }
template <bool QUAD>
__device__ __forceinline__ int slot_y(int s) { return QUAD ? 2 * ((s >> 2) & 1) + (s & 1) : s & 3; }

template <int L, bool BOX, bool CPLX = false>
__global__ void __launch_bounds__(128, CPLX ? 4 : (BOX ? 8 : 4)) spread_z_kernel(SpreadZArgs a)
{
    // 2 x 2 quadrants when spreading to the box (the fused z transform reads the slots as strip
    // columns): fewer ball visits per warp and more even chords (sweep spread 0.1511 -> 0.1484,
    // torus 0.0489 -> 0.0472 ms per rotation)
    constexpr bool QUAD = BOX;
    static_assert(!CPLX || BOX, "complex weights: spread to the box only");
    constexpr int NT = 128;
    constexpr int TPL = Plan<L>::TPL, NG = NT / TPL;
    constexpr int LS = line_stride(L);
    static_assert(BOX || (NT % TPL == 0 && NG >= SZ_LINES && Plan<L>::n == 2 && warp_local<L>()), "spread_z plan");
    extern __shared__ float4 smz[];
    const int Kz = a.K + 1;
    // layout: phi table | tw | Abuf (NG lines) | region {acc  /  zb}   (BOX: phi table | acc)
    float4 *phi = smz;
    float2 *tw = (float2 *)(phi + 2 * a.phi_n);
    float2 *Abuf = tw + L;
    constexpr int CS = L + 8;                         // column stride: the 4 lane groups of a warp
                                                      // (4 columns) sit 8 banks apart
    float *acc = BOX ? (float *)(phi + 2 * a.phi_n) : (float *)(Abuf + NG * LS);  // [16][CS]
    float *acci = acc + SZ_COLS * CS;                 // CPLX: imaginary parts [16][CS]

    const int b = blockIdx.y;
    const int tpa = L / 4;
    const int X0 = (blockIdx.x / tpa) * 4, Y0 = (blockIdx.x % tpa) * 4;
    float2 *T1 = a.out + (long long)b * a.out_bstride;

    // tiles outside B's (rotation-invariant) support cylinder: T1 rows are zero.  When the
    // consumer is pass_y_fast (skip_zero) they are never read (it loads only rows within
    // live_r, and zero tiles lie beyond live_r + 1), so nothing is written.
    {
        const float dx = fmaxf(fmaxf((float)X0 - a.cx, a.cx - (float)(X0 + 3)), 0.f);
        const float dy = fmaxf(fmaxf((float)Y0 - a.cy, a.cy - (float)(Y0 + 3)), 0.f);
        if (dx * dx + dy * dy > a.zero_r2) {
            if (a.skip_zero) return;
            for (int e = threadIdx.x; e < SZ_COLS * Kz; e += NT) {
                const int col = e / Kz, k = e % Kz;
                T1[((long long)(X0 + (col >> 2)) * L + Y0 + (col & 3)) * Kz + k] = make_float2(0.f, 0.f);
            }
            return;
        }
    }

    for (int e = threadIdx.x; e < 2 * a.phi_n; e += NT) phi[e] = a.phi[e];
    if (!BOX) load_twiddles<L>(tw, a.tw, threadIdx.x, NT);
    for (int e = threadIdx.x; e < (CPLX ? 2 : 1) * SZ_COLS * CS / 4; e += NT)
        reinterpret_cast<float4 *>(acc)[e] = make_float4(0.f, 0.f, 0.f, 0.f);

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gi = lane >> 3, hl = lane & 7;
    const int col = 4 * wid + gi;                     // accumulator slot (column slot_x(col), slot_y(col))
    const float fx = (float)(X0 + slot_x<QUAD>(col)), fy = (float)(Y0 + slot_y<QUAD>(col));
    // the warp's column footprint: [wx0, wx0 + wxn] x [wy0, wy0 + wyn]
    const float wx0 = (float)(X0 + slot_x<QUAD>(4 * wid)), wy0 = (float)(Y0 + slot_y<QUAD>(4 * wid));
    constexpr float wxn = QUAD ? 1.f : 0.f, wyn = QUAD ? 1.f : 3.f;
    float *accc = acc + col * CS;
    float *acci_c = acci + col * CS;
    // the blob's profile table (pieces of W/48 over [-W, W], W = 4 cells: n = 96) as constants;
    // launch_spread_z refuses a table of another shape
    constexpr int nphi = SZ_PHI_N;
    constexpr float U = SZ_PHI_U, invD = (float)SZ_PHI_N / (2.f * SZ_PHI_U);
    constexpr float tmax = (float)SZ_PHI_N - 1e-3f;
    const int bin = (X0 / SZ_BIN) * (L / SZ_BIN) + Y0 / SZ_BIN;
    const int cnt = a.counts[b * a.nbins + bin];
    const int *lst = a.lists + (long long)b * a.list_stride + a.offs[b * a.nbins + bin];
    const float4 *recA = a.recA + (long long)b * a.n_balls;
    __syncthreads();

    // ---- accumulate the bin's balls (ball order) into this lane's cells.  The warp keeps the
    // balls whose footprint reaches one of its four columns (ballot); within a step the lanes
    // touch distinct cells, steps and balls are sequential, so the sums are race-free and in
    // ball order (deterministic).
    for (int base0 = 0; base0 < cnt; base0 += 32) {
        // lane k tests candidate base0 + k and keeps its two records for the broadcast below
        bool rel = false;
        float4 uc = make_float4(0.f, 0.f, 0.f, 0.f), wc = uc;
        float wic = 0.f;
        if (base0 + lane < cnt) {
            const int jl = lst[base0 + lane];
            uc = recA[jl];
            wc = a.recB[jl];
            if (CPLX) wic = a.recWi[jl];
            const float ddx = fmaxf(fmaxf(wx0 - uc.x, uc.x - (wx0 + wxn)), 0.f);
            const float ddy = fmaxf(fmaxf(wy0 - uc.y, uc.y - (wy0 + wyn)), 0.f);
            // zero-weight balls add nothing (the planar complex spreads see each docking ball in
            // one of their two passes only)
            rel = fmaf(ddx, ddx, ddy * ddy) < uc.w && (wc.y != 0.f || (CPLX && wic != 0.f));
        }
        unsigned msk = __ballot_sync(0xffffffffu, rel);
        while (msk) {
            const int src = __ffs(msk) - 1;
            msk &= msk - 1;
            const float4 ue = make_float4(__shfl_sync(0xffffffffu, uc.x, src), __shfl_sync(0xffffffffu, uc.y, src),
                                          __shfl_sync(0xffffffffu, uc.z, src), __shfl_sync(0xffffffffu, uc.w, src));
            const float dx = fx - ue.x, dy = fy - ue.y;
            const float dxy2 = fmaf(dx, dx, dy * dy);
            const float hz2 = ue.w - dxy2;
            int zlo = 0, zhi = -1, nit = 0;
            if (hz2 > 0.f) {
                const float hz = hz2 * rsqrtf(hz2);
                zlo = max(0, (int)ceilf(ue.z - hz));
                zhi = min(L - 1, (int)floorf(ue.z + hz));
                nit = (zhi - zlo + 8) >> 3;
            }
            int nmax = max(nit, __shfl_xor_sync(0xffffffffu, nit, 8));
            nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, 16));
            if (nmax <= 0) continue;
            const float4 we = make_float4(__shfl_sync(0xffffffffu, wc.x, src), __shfl_sync(0xffffffffu, wc.y, src),
                                          __shfl_sync(0xffffffffu, wc.z, src),
                                          __shfl_sync(0xffffffffu, wc.w, src));  // (s, w, g0, g2)
            const float wie = CPLX ? __shfl_sync(0xffffffffu, wic, src) : 0.f;
            // two cells per lane per step (z and z + 8: independent evaluation chains).  Table
            // coordinates of s -+ d as one FFMA each from tS = (s + U) / D; rsqrt without the
            // denormal fix-up (d^2 >= 0.01 on that path); the s + d lookup only for balls with
            // s < U (warp-uniform: two copies of the loop), beyond it Phi1 = 1/2, Phi2 = 0.
            const float tS = (we.x + U) * invD, tQ = 2.f * U * invD;
            auto cells = [&](auto small_ball) {
                auto prof = [&](float d2) {
                    if (d2 < 0.01f) return fmaf(we.w, d2, we.z);
                    float rd;
                    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rd) : "f"(d2));
                    const float d = d2 * rd;
                    const PhiVal p = phi_lookup_t(phi, nphi, tmax, fmaf(-d, invD, tS));
                    PhiVal q = PhiVal{0.5f, 0.f};
                    if (decltype(small_ball)::value) {
                        const float t = fmaf(d, invD, tS);
                        if (t < tQ) q = phi_lookup_t(phi, nphi, tmax, t);
                    }
                    return p.p1 + q.p1 - (p.p2 - q.p2) * rd;
                };
                for (int it = 0; it < nmax; it += 2) {
                    const int z0 = zlo + (it << 3) + hl, z1 = z0 + 8;
                    const bool ok0 = z0 <= zhi, ok1 = z1 <= zhi;
                    const float dz0 = (float)z0 - ue.z, dz1 = (float)z1 - ue.z;
                    const float g0 = ok0 ? prof(fmaf(dz0, dz0, dxy2)) : 0.f;
                    const float g1 = ok1 ? prof(fmaf(dz1, dz1, dxy2)) : 0.f;
                    // complex weights: a ball whose weight is purely real or purely imaginary
                    // (the docking recipe's skin and core balls) updates one accumulator
                    if (!CPLX || we.y != 0.f) {
                        if (ok0) accc[z0] = fmaf(we.y, g0, accc[z0]);
                        if (ok1) accc[z1] = fmaf(we.y, g1, accc[z1]);
                    }
                    if (CPLX && wie != 0.f) {
                        if (ok0) acci_c[z0] = fmaf(wie, g0, acci_c[z0]);
                        if (ok1) acci_c[z1] = fmaf(wie, g1, acci_c[z1]);
                    }
                }
            };
            if (we.x < U) cells(std::true_type());
            else cells(std::false_type());
        }
    }
    __syncthreads();

    if (CPLX) {  // the tile's 16 complex columns to the box, two cells per 16-byte store
        float2 *box = reinterpret_cast<float2 *>(a.box + (long long)b * a.box_bstride);
        for (int e = threadIdx.x; e < SZ_COLS * L / 2; e += NT) {
            const int cc = e / (L / 2), z2 = 2 * (e % (L / 2));
            *reinterpret_cast<float4 *>(box + ((long long)(X0 + slot_x<QUAD>(cc)) * L + Y0 + slot_y<QUAD>(cc)) * L + z2) =
                make_float4(acc[cc * CS + z2], acci[cc * CS + z2], acc[cc * CS + z2 + 1], acci[cc * CS + z2 + 1]);
        }
    } else if (BOX) {  // the tile's 16 columns (1 KB each) to the box
        float *box = a.box + (long long)b * a.box_bstride;
        for (int e = threadIdx.x; e < SZ_COLS * L / 4; e += NT) {  // 16-byte rows (CS, L multiples of 4)
            const int cc = e / (L / 4), z4 = e % (L / 4);
            *reinterpret_cast<float4 *>(box + ((long long)(X0 + slot_x<QUAD>(cc)) * L + Y0 + slot_y<QUAD>(cc)) * L + 4 * z4) =
                *reinterpret_cast<const float4 *>(acc + cc * CS + 4 * z4);
        }
    } else {
        tile_z_transform<L, NT>(a, acc, Abuf, tw, T1, X0, Y0);
    }
}

// z transform of the box written by spread_z_kernel<L, true>, tile by tile (4 x 4 columns):
// the same FFT phase as the fused kernel, its input read from HBM (1 KB column rows).
template <int L, bool B4>
__global__ void __launch_bounds__(128, 4) pass_z_fast_kernel(SpreadZArgs a)
{
    constexpr int NT = 128;
    constexpr int TPL = Plan<L>::TPL, NG = NT / TPL;
    constexpr int LS = line_stride(L);
    constexpr int CS = L + 8;
    extern __shared__ float4 smz[];
    const int Kz = a.K + 1;
    float2 *tw = (float2 *)smz;
    float2 *Abuf = tw + L;
    float *acc = (float *)(Abuf + NG * LS);  // [16][CS], then zb
    const int b = blockIdx.y;
    const int tpa = L / 4;
    const int X0 = (blockIdx.x / tpa) * 4, Y0 = (blockIdx.x % tpa) * 4;
    float2 *T1 = a.out + (long long)b * a.out_bstride;
    {   // same zero-tile test as the spread (which wrote nothing for these tiles)
        const float dx = fmaxf(fmaxf((float)X0 - a.cx, a.cx - (float)(X0 + 3)), 0.f);
        const float dy = fmaxf(fmaxf((float)Y0 - a.cy, a.cy - (float)(Y0 + 3)), 0.f);
        if (dx * dx + dy * dy > a.zero_r2) {
            if (a.skip_zero) return;
            for (int e = threadIdx.x; e < SZ_COLS * Kz; e += NT) {
                const int col = e / Kz, k = e % Kz;
                T1[((long long)(X0 + (col >> 2)) * L + Y0 + (col & 3)) * Kz + k] = make_float2(0.f, 0.f);
            }
            return;
        }
    }
    const float *box = a.box + (long long)b * a.box_bstride;
    {   // the tile's columns: all loads issued before the stores, then the twiddle table
        constexpr int PER = SZ_COLS * L / 4 / NT;  // float4 per thread
        static_assert(SZ_COLS * L / 4 % NT == 0, "tile load");
        float4 v[PER];
#pragma unroll
        for (int u = 0; u < PER; u++) {
            const int e = threadIdx.x + NT * u, cc = e / (L / 4), z4 = e % (L / 4);
            v[u] = *reinterpret_cast<const float4 *>(box + ((long long)(X0 + (cc >> 2)) * L + Y0 + (cc & 3)) * L + 4 * z4);
        }
        load_twiddles<L>(tw, a.tw, threadIdx.x, NT);
#pragma unroll
        for (int u = 0; u < PER; u++) {
            const int e = threadIdx.x + NT * u, cc = e / (L / 4), z4 = e % (L / 4);
            *reinterpret_cast<float4 *>(acc + cc * CS + 4 * z4) = v[u];
        }
    }
    __syncthreads();
    tile_z_transform<L, NT, B4>(a, acc, Abuf, tw, T1, X0, Y0);
}

// real weights: the fused kernel or box + tile z transform (two-stage FFT plans); complex
// weights: box only (the z transform is the generic complex-row pass)
bool spread_z_supported(int L, int complex_w) { return complex_w ? (L == 128 || L == 256 || L == 384) : (L == 128 || L == 256); }

template <int L>
static void spread_z_launch(const SpreadZArgs &a, int batch, cudaStream_t s)
{
    constexpr int NG = 128 / Plan<L>::TPL;
    const int tpa = L / 4;
    if (a.box) {  // spread -> box, then the tile z transform
        const size_t sm1 = (size_t)a.phi_n * 32 + (size_t)SZ_COLS * (L + 8) * 4;
        cudaFuncSetAttribute(spread_z_kernel<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
        spread_z_kernel<L, true><<<dim3(tpa * tpa, batch), 128, sm1, s>>>(a);
        const size_t region = std::max({(size_t)SZ_COLS * (L + 8) * 4, (size_t)SZ_LINES * (2 * a.K + 1) * 8, L == 256 ? (size_t)SZ_LINES * 4 * ZB_RP * 8 : (size_t)0});
        const size_t sm2 = (size_t)L * 8 + (size_t)NG * line_stride(L) * 8 + region;
        if (L == 256 && a.c == 4 && a.G == 1024 && a.K == 255) {
            cudaFuncSetAttribute(pass_z_fast_kernel<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
            pass_z_fast_kernel<L, true><<<dim3(tpa * tpa, batch), 128, sm2, s>>>(a);
        } else {
            cudaFuncSetAttribute(pass_z_fast_kernel<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
            pass_z_fast_kernel<L, false><<<dim3(tpa * tpa, batch), 128, sm2, s>>>(a);
        }
        return;
    }
    const size_t region = std::max({(size_t)SZ_COLS * (L + 8) * 4, (size_t)SZ_LINES * (2 * a.K + 1) * 8, L == 256 ? (size_t)SZ_LINES * 4 * ZB_RP * 8 : (size_t)0});
    const size_t sm = (size_t)a.phi_n * 32 + (size_t)L * 8 + (size_t)NG * line_stride(L) * 8 + region;
    cudaFuncSetAttribute(spread_z_kernel<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    spread_z_kernel<L, false><<<dim3(tpa * tpa, batch), 128, sm, s>>>(a);
}

int spread_z_bins(int L) { return (L / SZ_BIN) * (L / SZ_BIN); }
int spread_z_bins_per_axis(int L) { return L / SZ_BIN; }
int spread_z_bins_per_ball(float rc_max) { const int t = (int)(2 * rc_max / SZ_BIN) + 2; return t * t; }

void launch_spread_z_bin(const SzBinArgs &a, int batch, cudaStream_t s)
{
    szb_rotate_kernel<<<dim3((a.n + 255) / 256, batch), 256, 0, s>>>(a);
    szb_count_kernel<<<dim3(a.nbins, batch), 256, 0, s>>>(a);
    szb_fill_kernel<<<dim3(a.nbins, batch), 256, 0, s>>>(a);
}

template <int L>
static void spread_z_launch_cplx(const SpreadZArgs &a, int batch, cudaStream_t s)
{
    const int tpa = L / 4;
    if (a.planar) {  // two real spreads at the real kernel's occupancy (half the accumulator)
        const size_t sm1 = (size_t)a.phi_n * 32 + (size_t)SZ_COLS * (L + 8) * 4;
        cudaFuncSetAttribute(spread_z_kernel<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
        SpreadZArgs im = a;
        im.recB = a.recBim;
        im.box = a.box + (long long)L * L * L;
        spread_z_kernel<L, true><<<dim3(tpa * tpa, batch), 128, sm1, s>>>(a);
        spread_z_kernel<L, true><<<dim3(tpa * tpa, batch), 128, sm1, s>>>(im);
        return;
    }
    const size_t sm = (size_t)a.phi_n * 32 + 2 * (size_t)SZ_COLS * (L + 8) * 4;
    cudaFuncSetAttribute(spread_z_kernel<L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    spread_z_kernel<L, true, true><<<dim3(tpa * tpa, batch), 128, sm, s>>>(a);
}

bool launch_spread_z(const SpreadZArgs &a, int batch, cudaStream_t s)
{
    if (a.phi_n != SZ_PHI_N || a.phi_U != SZ_PHI_U) return false;  // the table shape is compiled in
    if (a.cplx) {
        if (!a.box) return false;
        switch (a.L) {
        case 128: spread_z_launch_cplx<128>(a, batch, s); return true;
        case 256: spread_z_launch_cplx<256>(a, batch, s); return true;
        case 384: spread_z_launch_cplx<384>(a, batch, s); return true;
        default: return false;
        }
    }
    switch (a.L) {
    case 128: spread_z_launch<128>(a, batch, s); return true;
    case 256: spread_z_launch<256>(a, batch, s); return true;
    default: return false;
    }
}
