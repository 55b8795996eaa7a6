// dock_fast.cu -- the docking plan's per-rotation passes of R B with compile-time plan constants:
// box L = 384 fine cells, c = 2 cosets (G = 768), band |k_i| <= K = 191, fold period Np = 128,
// complex weights (sm_100a).
//
// Same quantities as the generic passes (passes.cu; PAPER.md L398-L419 eq_ccghat, the band
// spectrum of the relocated knots eq_rhoPhat, deconvolved by the blob window):
//   pass_z_dk   box[re|im][x][y][n] (spread_z planar)  -> T1[x][y][kz + 192]   (z transform)
//   pass_y_dk   T1                                      -> T2[x][kz + 192][ky + 192]
//   fold_dk     T2 -> x transform -> A''(k') B(-k') summed into F[k' mod 128]  (register-owned)
// What the plan shape makes compile-time (FFT384 lines of 32 threads, radices 4 x 8 x 12):
//  * thread tl of a line holds outputs q = tl + 32 m of coset p, k = 2 q + p (- 768 for the
//    negative half); the band keeps m in {0, 1, 2} (k = 2q + p <= 191) and m in {9, 10, 11}
//    (k = 2q + p - 768 >= -191), minus (p, q) = (0, 288);
//  * T1 rows hold kz at index kz + 192 (pitch 384): the two cosets' outputs of one q are
//    adjacent (k = 2q, 2q + 1), so a thread stores both with one 16-byte store;
//  * in the fold every in-band output lands on the fold target k mod 128 = 2 tl + 64 (m & 1) + p:
//    the thread owns its 4 targets, accumulated in registers (no shared-memory accumulator).
#include <algorithm>

#include "kernels.cuh"
#include "fft_ct.cuh"

using namespace fct;

namespace {

constexpr int DK_L = 384, DK_C = 2, DK_G = 768, DK_K = 191, DK_M = 2 * DK_K + 1, DK_NP = 128;
constexpr int DK_TPL = 32, DK_NL = 8, DK_NT = DK_TPL * DK_NL, DK_E = DK_L / DK_TPL;
constexpr int DK_P = 384;   // T1 / T2 row pitch: kz at index kz + 192
constexpr int DK_Z0 = 192;  // index of kz = 0
// line buffer strides: each line's A (stage-0 output, default pad) and B (mid-stage output,
// T3 padB) buffers.  64-bit shared stores are served a half-warp (128 bytes) at a time, so the
// transposes need each half-warp on 16 distinct 8-byte bank slots: = 4 mod 16 float2 for the
// passes' 4-line transposes (a half-warp stores 4 rows of 4 lines), = 2 mod 16 for the fold's
// 8-line ones (2 rows of 8 lines)
constexpr int DK_LSP = 436, DK_LSF = 434;
static_assert(DK_LSF >= T3<384>::BLEN && DK_LSF >= fct::pad(383) + 1 && DK_LSP % 16 == 4 && DK_LSF % 16 == 2, "dock strides");
constexpr int DK_TW = T3<DK_L>::SIZE;  // conflict-free twiddle tables (fft_regs_t3)
constexpr int DK_MS = cm_row_stride(DK_L, DK_C, DK_G, DK_K);  // A'' row stride (coset-major)
static_assert(Plan<DK_L>::TPL == DK_TPL && Plan<DK_L>::n == 3 && warp_local<DK_L>(), "dock plan");
static_assert(DK_E == 12, "outputs per thread");

// e^{-2 pi i m / 24} (coset twiddle step: e^{-2 pi i (tl + 32 m) / 768} = e^{-2 pi i tl / 768} W24^m)
__constant__ WTab<24, -1> c_w24 = WTab<24, -1>();

// in-band output m of coset p for lane tl (compile-time m after unrolling)
BC_DEV bool dk_in_band(int m, int p, int tl) { return (m < 3 || m >= 9) && !(m == 9 && p == 0 && tl == 0); }
BC_DEV int dk_k(int m, int p, int tl) { return 2 * (tl + DK_TPL * m) + p - (m >= 9 ? DK_G : 0); }

// x[m] *= e^{-2 pi i (tl + 32 m) / 768} (coset p = 1), from one L1 value and constant steps
BC_DEV void dk_coset(float2 (&y)[DK_E], const float2 (&x)[DK_E], const float2 *ctw, int p, int tl)
{
    if (p == 0) {
#pragma unroll
        for (int m = 0; m < DK_E; m++) y[m] = x[m];
        return;
    }
    const float2 u = __ldg(ctw + DK_L + tl);
#pragma unroll
    for (int m = 0; m < DK_E; m++) y[m] = m ? cmul(x[m], cmul(u, make_float2(c_w24.re[m], c_w24.im[m]))) : cmul(x[m], u);
}

// spread_z's zero-tile test (the 4 x 4-column tile of box row (x, y))
BC_DEV bool dk_zero_tile(int x, int y, float cx, float cy, float zero_r2)
{
    const int X0 = x & ~3, Y0 = y & ~3;
    const float dx = fmaxf(fmaxf((float)X0 - cx, cx - (float)(X0 + 3)), 0.f);
    const float dy = fmaxf(fmaxf((float)Y0 - cy, cy - (float)(Y0 + 3)), 0.f);
    return dx * dx + dy * dy > zero_r2;
}

// x planes of T2 written by pass_y_dk and read by fold_dk (one definition for both)
BC_DEV void dk_live_planes(float cx, float live_r2, int &xlo, int &xhi)
{
    const float hh = sqrtf(fmaxf(live_r2, 0.f));
    xlo = max(0, (int)ceilf(cx - hh));
    xhi = min(DK_L - 1, (int)floorf(cx + hh));
}

}  // namespace

// ============================================================================ z pass
// Block = 8 box rows (x, y0 .. y0 + 7).  Rows in tiles spread_z left unwritten read as zero; a
// block of only such rows writes nothing (the y pass loads only rows within live_r, all of
// them in written tiles).
template <int NL, bool MULT>
__global__ void __launch_bounds__(32 * NL, 20 / NL) pass_z_dk_kernel(DockPassArgs a)
{
    constexpr int NT = 32 * NL;
    extern __shared__ float2 smd[];
    float2 *tw = smd;
    float2 *A = tw + DK_TW;
    float2 *B = A + NL * DK_LSP;
    const int line = threadIdx.x / DK_TPL, tl = threadIdx.x % DK_TPL;
    const int b = blockIdx.y;
    const long long row0 = (long long)blockIdx.x * NL;
    const int x = (int)(row0 / DK_L), y0 = (int)(row0 % DK_L);
    if (dk_zero_tile(x, y0, a.cx, a.cy, a.zero_r2) && dk_zero_tile(x, y0 + NL - 1, a.cx, a.cy, a.zero_r2)) return;
    const bool live = !dk_zero_tile(x, y0 + line, a.cx, a.cy, a.zero_r2);
    // planar box: real plane, then the imaginary plane L^3 floats further
    const float *inr = reinterpret_cast<const float *>(a.in + (long long)b * a.in_bstride) + (row0 + line) * DK_L;
    const float *ini = inr + (long long)DK_L * DK_L * DK_L;
    float2 xv[DK_E];
#pragma unroll
    for (int m = 0; m < DK_E; m++) xv[m] = live ? make_float2(inr[tl + DK_TPL * m], ini[tl + DK_TPL * m]) : make_float2(0.f, 0.f);
    // the twiddle tables after the row loads are issued: both latencies overlap
    load_twiddles_t3<DK_L>(tw, a.tw, threadIdx.x, NT);
    __syncthreads();  // twiddle table
    float2 keep[6];
#pragma unroll 1
    for (int p = 0; p < DK_C; p++) {
        float2 yv[DK_E];
        dk_coset(yv, xv, a.ctw, p, tl);
        fft_regs_t3<DK_L, -1, true>(yv, A + line * DK_LSP, B + line * DK_LSP, tw, tl);
        __syncwarp();  // the next coset's FFT rewrites this line's buffers
        if (p == 0) {
#pragma unroll
            for (int u = 0; u < 6; u++) {
                const int m = u < 3 ? u : u + 6;
                keep[u] = dk_in_band(m, 0, tl) ? yv[m] : make_float2(0.f, 0.f);
            }
        } else {
            float2 *out = a.out + (long long)b * a.out_bstride + (row0 + line) * DK_P;
#pragma unroll
            for (int u = 0; u < 6; u++) {
                const int m = u < 3 ? u : u + 6;
                const int k0 = dk_k(m, 0, tl);  // even: k0, k0 + 1 adjacent at index k + 192
                float2 v0 = keep[u], v1 = yv[m];  // (keep: zero outside the band)
                if (MULT) {  // else the multipliers are folded into A'' (permute_cm_kernel)
                    const float2 m0 = k0 >= -DK_K ? __ldg(a.mult + k0 + DK_K) : make_float2(0.f, 0.f);
                    const float2 m1 = __ldg(a.mult + k0 + 1 + DK_K);
                    v0 = cmul(v0, m0);
                    v1 = cmul(v1, m1);
                }
                *reinterpret_cast<float4 *>(out + k0 + DK_Z0) = make_float4(v0.x, v0.y, v1.x, v1.y);
            }
        }
    }
}

// ============================================================================ y pass
// Block = one x plane, 8 consecutive T1 columns j0 .. j0 + 7 (kz = j - 192), one line each.
// Rows outside B's support cylinder at this x are not loaded; a plane outside it is not
// written (the fold does not read it).  T2 rows hold ky at index ky + 192, so, as in the z
// pass, a thread stores the two cosets' outputs of one q with one 16-byte store: no output
// staging (T2 = [x][j][ky + 192]).
template <int NL, bool MULT>
__global__ void __launch_bounds__(32 * NL, 20 / NL) pass_y_dk_kernel(DockPassArgs a)
{
    constexpr int NT = 32 * NL;
    extern __shared__ float2 smd[];
    float2 *tw = smd;
    float2 *A = tw + DK_TW;
    float2 *B = A + NL * DK_LSP;
    const int line = threadIdx.x / DK_TPL, tl = threadIdx.x % DK_TPL;
    const int b = blockIdx.y;
    constexpr int JT = DK_P / NL;  // 48 column tiles
    const int x = blockIdx.x / JT, j0 = (blockIdx.x % JT) * NL;
    const float2 *T1 = a.in + (long long)b * a.in_bstride + (long long)x * DK_L * DK_P + j0;
    float2 *T2 = a.out + (long long)b * a.out_bstride + ((long long)x * DK_P + j0) * DK_P;
    {   // planes the fold reads (dk_live_planes) but without a live row here are written as zero
        int xlo, xhi;
        dk_live_planes(a.cx, a.live_r2, xlo, xhi);
        if (x < xlo || x > xhi) return;
    }
    const float dxl = (float)x - a.cx;
    const float h2 = a.live_r2 - dxl * dxl;
    int ylo = 0, yhi = -1;
    if (h2 > 0.f) {
        const float hh = sqrtf(h2);
        ylo = max(0, (int)ceilf(a.cy - hh));
        yhi = min(DK_L - 1, (int)floorf(a.cy + hh));
    }
    if (ylo > yhi) {
        for (int e = threadIdx.x; e < NL * DK_P; e += NT) T2[e] = make_float2(0.f, 0.f);
        return;
    }
    float2 xv[DK_E];
    {
#pragma unroll
        for (int m = 0; m < DK_E; m++) {
            const int e = threadIdx.x + NT * m;
            const int n = e / NL, i = e % NL;
            xv[m] = (n >= ylo && n <= yhi) ? T1[(long long)n * DK_P + i] : make_float2(0.f, 0.f);
        }
        // the twiddle tables after the row loads are issued: both latencies overlap
        load_twiddles_t3<DK_L>(tw, a.tw, threadIdx.x, NT);
#pragma unroll
        for (int m = 0; m < DK_E; m++) {
            const int e = threadIdx.x + NT * m;
            A[(e % NL) * DK_LSP + pad(e / NL)] = xv[m];
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < DK_E; m++) xv[m] = A[line * DK_LSP + pad(tl + DK_TPL * m)];
        __syncthreads();
    }
    float2 keep[6];
#pragma unroll 1
    for (int p = 0; p < DK_C; p++) {
        float2 yv[DK_E];
        dk_coset(yv, xv, a.ctw, p, tl);
        fft_regs_t3<DK_L, -1, true>(yv, A + line * DK_LSP, B + line * DK_LSP, tw, tl);
        __syncwarp();
        if (p == 0) {
#pragma unroll
            for (int u = 0; u < 6; u++) {
                const int m = u < 3 ? u : u + 6;
                keep[u] = dk_in_band(m, 0, tl) ? yv[m] : make_float2(0.f, 0.f);
            }
        } else {
            float2 *out = T2 + (long long)line * DK_P;
#pragma unroll
            for (int u = 0; u < 6; u++) {
                const int m = u < 3 ? u : u + 6;
                const int k0 = dk_k(m, 0, tl);
                float2 v0 = keep[u], v1 = yv[m];  // (keep: zero outside the band)
                if (MULT) {  // else the multipliers are folded into A'' (permute_cm_kernel)
                    const float2 m0 = k0 >= -DK_K ? __ldg(a.mult + k0 + DK_K) : make_float2(0.f, 0.f);
                    const float2 m1 = __ldg(a.mult + k0 + 1 + DK_K);
                    v0 = cmul(v0, m0);
                    v1 = cmul(v1, m1);
                }
                *reinterpret_cast<float4 *>(out + k0 + DK_Z0) = make_float4(v0.x, v0.y, v1.x, v1.y);
            }
        }
    }
}

// ============================================================================ fold
// Persistent blocks over (target block, rotation) items, rotation-fastest (the batch's items
// share A'' rows through L2).  Item = target plane k'z, 8 targets k'y with labels
// 8 t + 1 .. 8 t + 8 (k'y = label mod 128: the lines' T2 rows -ky + 192 then start on a
// 16-byte boundary).  For each alias ky = label + 128 ny and kz = k'z + 128 nz in the band,
// the x transform of B's T2 line at (-ky, -kz) times A''(ky, kz) (= A'(k') mult_x(kx) at the
// coset-major position of the output kx, reading C-3: weights not conjugated,
// f_hat_A'(k') f_hat_RB(-k')), summed into the target k'x = -kx mod 128.
__global__ void __launch_bounds__(DK_NT, 2) fold_dk_kernel(DockFoldArgs a)
{
    extern __shared__ float2 smd[];
    float2 *tw = smd;
    float2 *A = tw + DK_TW;
    float2 *B = A + DK_NL * DK_LSF;
    const int line = threadIdx.x / DK_TPL, tl = threadIdx.x % DK_TPL;
    constexpr int YT = DK_NP / DK_NL;  // 16 target tiles per k'z plane
    const int n_items = DK_NP * YT * a.nb;
    load_twiddles_t3<DK_L>(tw, a.tw, threadIdx.x, DK_NT);
    __syncthreads();
    int xlo, xhi;  // x planes of T2 the y pass writes
    dk_live_planes(a.cx, a.live_r2, xlo, xhi);
#pragma unroll 1
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        const int b = w % a.nb;
        const int tb = w / a.nb;
        const int kzp = tb / YT, y1 = (tb % YT) * DK_NL + 1;  // labels y1 .. y1 + 7
        const float2 *T2 = a.T2 + (long long)b * a.t2_bstride;
        float2 acc[2][DK_C];
#pragma unroll
        for (int j = 0; j < 2; j++)
#pragma unroll
            for (int p = 0; p < DK_C; p++) acc[j][p] = make_float2(0.f, 0.f);
        // aliases within the band [-191, 191] of a label in [1, 128]: label - 256, - 128, + 0,
        // + 128; of k'z in [0, 128): k'z - 256 (k'z >= 65), - 128, + 0, + 128 (k'z <= 63)
#pragma unroll 1
        for (int nz = -2; nz <= 1; nz++) {
            const int kz = kzp + DK_NP * nz;
            if (kz < -DK_K || kz > DK_K) continue;
#pragma unroll 1
            for (int ny = -2; ny <= 1; ny++) {
                const int kylo = y1 + DK_NP * ny, kyhi = kylo + DK_NL - 1;
                if (kyhi < -DK_K || kylo > DK_K) continue;  // no line of the group in band
                // T2 lines (-ky_i, -kz), transposed through A for coalescing
                {
                    const int i = threadIdx.x % DK_NL, n0 = threadIdx.x / DK_NL;
                    const int kyi = kylo + i;
                    const bool ok = kyi >= -DK_K && kyi <= DK_K;
                    const float2 *src = T2 + (long long)(-kz + DK_Z0) * DK_P + (-kyi + DK_Z0);
                    float2 xv[DK_E];
#pragma unroll
                    for (int m = 0; m < DK_E; m++) {
                        const int n = n0 + (DK_NT / DK_NL) * m;
                        xv[m] = (ok && n >= xlo && n <= xhi) ? src[(long long)n * DK_P * DK_P] : make_float2(0.f, 0.f);
                    }
                    __syncthreads();  // previous group's FFTs are done with A
#pragma unroll
                    for (int m = 0; m < DK_E; m++) A[i * DK_LSF + pad(n0 + (DK_NT / DK_NL) * m)] = xv[m];
                }
                __syncthreads();
                float2 xv[DK_E];
#pragma unroll
                for (int m = 0; m < DK_E; m++) xv[m] = A[line * DK_LSF + pad(tl + DK_TPL * m)];
                __syncthreads();  // A is rewritten by the FFT below
                const int ky = kylo + line;
                const bool my_ok = ky >= -DK_K && ky <= DK_K;
                const float2 *arow = a.Ahat + ((long long)(my_ok ? ky + DK_K : 0) * DK_M + (kz + DK_K)) * DK_MS;
#pragma unroll 1
                for (int p = 0; p < DK_C; p++) {
                    const int pb = (p == 0 ? a.pos_base[0] : a.pos_base[1]) + tl;
                    float2 av[6];
#pragma unroll
                    for (int u = 0; u < 6; u++) {
                        const int m = u < 3 ? u : u + 6;
                        const int pos = pb + DK_TPL * m + (m < 3 ? DK_L : 0);
                        av[u] = (my_ok && dk_in_band(m, p, tl)) ? __ldg(arow + pos) : make_float2(0.f, 0.f);
                    }
                    float2 yv[DK_E];
                    dk_coset(yv, xv, a.ctw, p, tl);
                    fft_regs_t3<DK_L, -1, true>(yv, A + line * DK_LSF, B + line * DK_LSF, tw, tl);
                    __syncwarp();
                    // outputs m and m' with the same m & 1 share a target: (0, 2, 10) -> j = 0, (1, 9, 11) -> j = 1
                    const float2 s0 = cfma(av[0], yv[0], cfma(av[2], yv[2], cmul(av[4], yv[10])));
                    const float2 s1 = cfma(av[1], yv[1], cfma(av[3], yv[9], cmul(av[5], yv[11])));
                    if (p == 0) {
                        acc[0][0] = cadd(acc[0][0], s0);
                        acc[1][0] = cadd(acc[1][0], s1);
                    } else {
                        acc[0][1] = cadd(acc[0][1], s0);
                        acc[1][1] = cadd(acc[1][1], s1);
                    }
                }
            }
        }
        // targets k'x = -(2 tl + 64 j + p) mod 128 -> F[k'x][k'y][k'z]
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 2; j++)
#pragma unroll
            for (int p = 0; p < DK_C; p++) A[line * DK_LSF + ((DK_NP - (2 * tl + 64 * j + p)) & (DK_NP - 1))] = acc[j][p];
        __syncthreads();
        float2 *F = a.F + (long long)b * a.f_bstride;
        for (int e = threadIdx.x; e < DK_NL * DK_NP; e += DK_NT) {
            const int i = e % DK_NL, t = e / DK_NL;
            F[((long long)t * DK_NP + ((y1 + i) & (DK_NP - 1))) * DK_NP + kzp] = A[i * DK_LSF + t];
        }
    }
}

// ============================================================================ host side
bool dock_fast_supported(int L, int c, int G, int K, int Np, int complex_w)
{
    return L == DK_L && c == DK_C && G == DK_G && K == DK_K && Np == DK_NP && complex_w;
}

static size_t dk_smem(int nl, int ls) { return sizeof(float2) * ((size_t)DK_TW + 2 * nl * (size_t)ls); }

constexpr int DK_PASS_NL = 4;  // lines per block of the z / y passes (128 threads, 5 blocks per SM)

void launch_pass_z_dk(const DockPassArgs &a, int batch, cudaStream_t s)
{
    constexpr int NL = DK_PASS_NL;
    const size_t sm = dk_smem(NL, DK_LSP);
    const dim3 grid((unsigned)(DK_L * DK_L / NL), batch);
    if (a.mult) {
        cudaFuncSetAttribute(pass_z_dk_kernel<NL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        pass_z_dk_kernel<NL, true><<<grid, 32 * NL, sm, s>>>(a);
    } else {
        cudaFuncSetAttribute(pass_z_dk_kernel<NL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        pass_z_dk_kernel<NL, false><<<grid, 32 * NL, sm, s>>>(a);
    }
}

void launch_pass_y_dk(const DockPassArgs &a, int batch, cudaStream_t s)
{
    constexpr int NL = DK_PASS_NL;
    const size_t sm = dk_smem(NL, DK_LSP);
    const dim3 grid((unsigned)(DK_L * (DK_P / NL)), batch);
    if (a.mult) {
        cudaFuncSetAttribute(pass_y_dk_kernel<NL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        pass_y_dk_kernel<NL, true><<<grid, 32 * NL, sm, s>>>(a);
    } else {
        cudaFuncSetAttribute(pass_y_dk_kernel<NL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        pass_y_dk_kernel<NL, false><<<grid, 32 * NL, sm, s>>>(a);
    }
}

bool launch_fold_dk(const DockFoldArgs &a_in, int batch, cudaStream_t s)
{
    if (a_in.MS != DK_MS) return false;
    DockFoldArgs a = a_in;
    a.nb = batch;
    const size_t sm = dk_smem(DK_NL, DK_LSF);
    cudaFuncSetAttribute(fold_dk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long items = (long long)DK_NP * (DK_NP / DK_NL) * batch;
    const long long grid = std::min<long long>(items, (long long)sms * 2 * 4);
    fold_dk_kernel<<<(unsigned)grid, DK_NT, sm, s>>>(a);
    return true;
}

size_t dock_t_pitch() { return DK_P; }
