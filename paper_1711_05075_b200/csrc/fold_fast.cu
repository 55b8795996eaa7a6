// fold_fast.cu -- fused x-pass + spectral product + fold + inverse x for the plan shape
// L = Np = 256, c = 4 cosets, G = 4 (K + 1) (K = 255), real weights (sm_100a).
//
// Same arithmetic as fold_x_kernel<256, 256, false, true> (passes.cu; PAPER.md L398-L419
// eq_ccghat): for the targets (k'y, k'z in [z0, z0 + 8)) the x-transform of every alias
// line (ky, kz) of R B on the band, times A'' (A's spectrum with the origin phase and B's
// deconvolution folded in), summed into F[k mod Np] (conjugated at -k for the Hermitian
// partner half), then the inverse x-FFT of the folded lines, written as X1[mx][k'y][k'z].
// What this plan shape makes compile-time:
//  * thread tl of a line holds the FFT outputs q = tl + 16 m of coset p, k = 4 q + p;
//    the band |k| <= 255 keeps exactly m in {0..3} (k = 4q + p) and {12..15} (k = 4q + p - 1024),
//    minus (p, q) = (0, 192), and both land on the fold target t = 4 tl + 64 (m & 3) + p:
//    the thread OWNS its 16 targets, accumulated in registers (no shared-memory atomics);
//  * the Hermitian partner -t of a target owned by lane tl is owned by lane 15 - tl (p != 0)
//    or (16 - tl) & 15 (p = 0), in the same 16-lane line: conjugate-pass products move by
//    warp shuffles;
//  * A''s coset-major row positions are affine in (tl, m): coalesced 128-byte loads.
#include <algorithm>

#include "kernels.cuh"
#include "fft_ct.cuh"

using namespace fct;

namespace {

__constant__ WTab<64, -1> c_w64 = WTab<64, -1>();  // e^{-2 pi i e / 64}

constexpr int FF_L = 256, FF_C = 4, FF_TPL = 16, FF_NL = 8, FF_NT = FF_NL * FF_TPL;
constexpr int FF_G = FF_C * FF_L, FF_K = FF_G / 4 - 1, FF_M = 2 * FF_K + 1, FF_KZ = FF_K + 1;
constexpr int FF_NP = FF_L, FF_FZ = FF_NP / 2 + 1;
constexpr int FF_LS = line_stride(FF_L);
// the plan's strides as compile-time constants (the launcher refuses others)
constexpr int FF_MS = cm_row_stride(FF_L, FF_C, FF_G, FF_K);  // A'' row stride (coset-major)
constexpr int FF_X1P = (FF_FZ + 7) & ~7;                     // X1 row pitch (api.cu's zpitch)
static_assert(Plan<FF_L>::TPL == FF_TPL && Plan<FF_L>::n == 2, "fold_fast plan");

}  // namespace

__global__ void __launch_bounds__(FF_NT, 4) fold_fast_kernel(FoldFastArgs a)
{
    constexpr int E = FF_L / FF_TPL;  // 16
    extern __shared__ float2 smf[];
    float2 *tw = smf;                  // [L]
    float2 *ctw = tw + FF_L;           // [C][L]
    float2 *X = ctw + FF_C * FF_L;     // [NL][LS] input lines (x order)
    float2 *Ab = X + FF_NL * FF_LS;    // [NL][LS] FFT exchange / staging
    const int line = threadIdx.x / FF_TPL, tl = threadIdx.x % FF_TPL;
    const int lane = threadIdx.x & 31;
    // targets: 16 tiles of 8 k'z per k'y row cover k'z in [0, 128); the Nyquist plane k'z = 128
    // is done by 32 items whose 8 lines are 8 consecutive k'y rows (a 17th tile per row would
    // carry 1 valid line in 8)
    constexpr int ZT = (FF_FZ - 1) / FF_NL;            // 16
    constexpr int NREG = FF_NP * ZT, NNYQ = FF_NP / FF_NL;

    load_twiddles<FF_L>(tw, a.tw, threadIdx.x, FF_NT);
    for (int e = threadIdx.x; e < FF_C * FF_L; e += FF_NT) ctw[e] = a.ctw[e];

    // persistent blocks: work items w = (target block) * nb + rotation, rotation-fastest (the
    // nb items sharing A'' rows run together and share them through L2); the tables above are
    // loaded once per block
    const int n_items = (NREG + NNYQ) * a.nb;
#pragma unroll 1
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
    const int b = w % a.nb;
    const int tb = w / a.nb;
    const bool nyq = tb >= NREG;
    const int kyp = nyq ? FF_NL * (tb - NREG) : tb / ZT;   // k'y of line 0
    const int z0 = nyq ? FF_FZ - 1 : (tb % ZT) * FF_NL;     // k'z of line 0
    // line i: target (k'y, k'z) = (kyp + i, 128) on the Nyquist plane, (kyp, z0 + i) elsewhere
    auto line_kyp = [&](int i) { return nyq ? kyp + i : kyp; };
    auto line_kz = [&](int i) { return nyq ? z0 : z0 + i; };
    const float2 *T2 = a.T2 + (long long)b * a.t2_bstride;
    // the alias slots (pass, al): ky = +-k'y (+ 256 al); a slot is skipped when out of band for
    // the whole block (block-uniform); on the Nyquist plane validity is per line
    auto slot_ky = [&](int kp, int pass, int al) {
        return pass == 0 ? (al == 0 ? kp : kp - FF_NP) : (al == 0 ? -kp : FF_NP - kp);
    };
    unsigned slots = 0;
#pragma unroll
    for (int sidx = 0; sidx < 4; sidx++) {
        const int ky0 = slot_ky(kyp, sidx >> 1, sidx & 1), ky7 = slot_ky(kyp + FF_NL - 1, sidx >> 1, sidx & 1);
        const bool any = (ky0 >= -FF_K && ky0 <= FF_K) || (nyq && ky7 >= -FF_K && ky7 <= FF_K);
        if (any) slots |= 1u << sidx;
    }
    // L2 prefetch of a slot's T2 rows: 256 rows x 64 bytes, two rows per thread (regular items)
    auto prefetch_slot = [&](int sidx) {
        if (nyq) return;
        const int ky = slot_ky(kyp, sidx >> 1, sidx & 1), pass = sidx >> 1;
        const int kz = pass == 0 ? z0 : FF_NP - z0 - (FF_NL - 1);  // lowest kz of the 8 lines
        for (int n = threadIdx.x; n < FF_L; n += FF_NT) {
            const float2 *p = T2 + (n * FF_M + ky + FF_K) * FF_KZ + max(kz, 0);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        }
    };
    if (slots) prefetch_slot(__ffs(slots) - 1);

    // A'' row position of output (m, p) of lane tl: pos_base[p] + tl + 16 m (+ L for m < 4)
    float2 acc[4][FF_C];
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
        for (int p = 0; p < FF_C; p++) acc[j][p] = make_float2(0.f, 0.f);

    const int tz = line_kz(line);    // this line's target k'z
    const int tkyp = line_kyp(line); // and k'y
    // direct: kz = k'z in [0, 128], ky in {k'y, k'y - 256};  conjugate partner: kz = 256 - k'z
    // (k'z in [1, 128]), ky in {-k'y, 256 - k'y}; out-of-band ky / kz contribute nothing
#pragma unroll 1
    for (unsigned rest = slots; rest; rest &= rest - 1) {
        const int sidx = __ffs(rest) - 1;
        const int pass = sidx >> 1, al = sidx & 1;
        if (rest & (rest - 1)) prefetch_slot(__ffs(rest & (rest - 1)) - 1);
        const int ky = slot_ky(tkyp, pass, al);  // this thread's line
        {
            // ---- T2 lines (ky, kz(i)) -> X (transposed through registers for coalescing)
            // element m of this thread: row n = n0 + 16 m of line i (e = tid + 128 m, i = e % 8),
            // so the line's validity and source column are per-thread constants
            const int i = threadIdx.x % FF_NL, n0 = threadIdx.x / FF_NL;
            const int kt = line_kz(i);
            const int kyi = slot_ky(line_kyp(i), pass, al);
            const bool ok = (pass == 0 ? (kt < FF_FZ) : (kt >= 1 && kt < FF_FZ)) && kyi >= -FF_K && kyi <= FF_K;
            const float2 *src = T2 + (long long)(n0 * FF_M + kyi + FF_K) * FF_KZ + (pass == 0 ? kt : FF_NP - kt);
            float2 x[E];
#pragma unroll
            for (int m = 0; m < E; m++)
                x[m] = ok ? src[(long long)(FF_NT / FF_NL) * m * FF_M * FF_KZ] : make_float2(0.f, 0.f);
            __syncthreads();  // previous group's last reads of X / Ab are done
#pragma unroll
            for (int m = 0; m < E; m++) X[i * FF_LS + pad(n0 + (FF_NT / FF_NL) * m)] = x[m];
            __syncthreads();
            const bool my_ok = (pass == 0 ? (tz < FF_FZ) : (tz >= 1 && tz < FF_FZ)) && ky >= -FF_K && ky <= FF_K;
            const int my_kz = pass == 0 ? tz : FF_NP - tz;
            const float2 *arow = a.Ahat + (long long)((ky + FF_K) * FF_KZ + (my_ok ? my_kz : 0)) * FF_MS;
            // one copy of the FFT (runtime coset loop keeps the code in the instruction cache);
            // only the register-accumulator update is specialised per coset
#pragma unroll 1
            for (int p = 0; p < FF_C; p++) {
                // A'' values of the 8 in-band outputs (issued before the FFT to hide latency)
                // (select chain: a runtime index into the kernel-parameter array would force a
                // local-memory copy of the argument block)
                const int pb = (p == 0 ? a.pos_base[0] : p == 1 ? a.pos_base[1] : p == 2 ? a.pos_base[2] : a.pos_base[3]) + tl;
                float2 av[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int m = u < 4 ? u : u + 8;
                    const int pos = pb + 16 * m + (m < 4 ? FF_L : 0);
                    const bool in_band = my_ok && !(p == 0 && m == 12 && tl == 0);
                    av[u] = in_band ? __ldg(arow + pos) : make_float2(0.f, 0.f);
                }
                // (measured: absorbing the coset twiddle into per-coset last-stage tables or
                // generating the last stage's twiddles in registers cost more than the table
                // reads they save here)
                float2 y[E];
#pragma unroll
                for (int m = 0; m < E; m++) {
                    const int n = tl + FF_TPL * m;
                    const float2 v = X[line * FF_LS + pad(n)];
                    y[m] = p ? cmul(v, ctw[p * FF_L + n]) : v;
                }
                fft_regs<FF_L, -1, true, false>(y, Ab + line * FF_LS, Ab + line * FF_LS, tw, tl);
                // S[j] = sum of the products of outputs m = j and m = j + 12 (same target)
                float2 S[4];
#pragma unroll
                for (int j = 0; j < 4; j++) S[j] = cadd(cmulc(av[j], y[j]), cmulc(av[j + 4], y[j + 12]));
                __syncwarp();  // the next coset's FFT rewrites this line's Ab (fft_regs contract)
                if (pass == 0) {
                    switch (p) {
#define FF_DIRECT(P_)                                                               \
    case P_:                                                                        \
        _Pragma("unroll") for (int j = 0; j < 4; j++) acc[j][P_] = cadd(acc[j][P_], S[j]); \
        break;
                        FF_DIRECT(0) FF_DIRECT(1) FF_DIRECT(2) FF_DIRECT(3)
#undef FF_DIRECT
                    }
                } else {
                    const int src = (lane & 16) | (p == 0 ? ((16 - tl) & 15) : (15 - tl));
                    float2 Rv[4];
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        Rv[j].x = __shfl_sync(0xffffffffu, S[j].x, src);
                        Rv[j].y = __shfl_sync(0xffffffffu, S[j].y, src);
                    }
                    switch (p) {
                    case 0:
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const float2 v = tl == 0 ? Rv[(4 - j) & 3] : Rv[3 - j];
                            acc[j][0] = cadd(acc[j][0], cconj(v));
                        }
                        break;
#define FF_CONJ(P_)                                                                                          \
    case P_:                                                                                                 \
        _Pragma("unroll") for (int j = 0; j < 4; j++) acc[3 - j][4 - P_] = cadd(acc[3 - j][4 - P_], cconj(Rv[j])); \
        break;
                        FF_CONJ(1) FF_CONJ(2) FF_CONJ(3)
#undef FF_CONJ
                    }
                }
            }
        }
    }

    // ---- inverse x of the folded lines: F[t] (t = 4 tl + 64 j + p) -> X1[mx][k'y][k'z]
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
        for (int p = 0; p < FF_C; p++) X[line * FF_LS + pad(4 * tl + 64 * j + p)] = acc[j][p];
    __syncthreads();
    float2 v[E];
#pragma unroll
    for (int m = 0; m < E; m++) v[m] = X[line * FF_LS + pad(tl + FF_TPL * m)];
    fft_regs<FF_NP, +1, true, false>(v, Ab + line * FF_LS, Ab + line * FF_LS, tw, tl);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < E; m++) X[line * FF_LS + pad(tl + FF_TPL * m)] = v[m];
    __syncthreads();
    float2 *X1 = a.X1 + (long long)b * a.x1_bstride;
    for (int e = threadIdx.x; e < FF_NL * a.N; e += FF_NT) {
        const int i = e % FF_NL, q = e / FF_NL;
        X1[(q * FF_NP + line_kyp(i)) * FF_X1P + line_kz(i)] = X[i * FF_LS + pad(q)];
    }
    __syncthreads();  // X is rewritten by the next item's first group
    }
}

bool fold_fast_supported(int L, int c, int G, int K, int Np, int complex_w)
{
    return L == FF_L && c == FF_C && G == FF_G && K == FF_K && Np == FF_NP && !complex_w;
}

bool launch_fold_fast(const FoldFastArgs &a_in, int batch, cudaStream_t s)
{
    if (a_in.MS != FF_MS || a_in.x1_pitch != FF_X1P) return false;
    FoldFastArgs a = a_in;
    a.nb = batch;
    constexpr int ZT = (FF_FZ - 1) / FF_NL;
    const size_t sm = sizeof(float2) * ((size_t)FF_L + FF_C * FF_L + 2 * FF_NL * FF_LS);
    cudaFuncSetAttribute(fold_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long items = (long long)(FF_NP * ZT + FF_NP / FF_NL) * batch;
    const long long grid = std::min<long long>(items, (long long)sms * 4 * 4);  // 4 blocks / SM, 4 waves of items or more
    fold_fast_kernel<<<(unsigned)grid, FF_NT, sm, s>>>(a);
    return true;
}

// ============================================================================ forward y pass
// T1[ix][iy][kz] -> T2[ix][ky][kz] = mult_y(ky) sum_iy T1 exp(-2 pi i ky iy / G), |ky| <= K,
// for the same plan shape (the generic pass_kernel<256, -1, 2, 1> computes the same).
// Block = one ix, 8 consecutive kz.  Rows iy outside B's support cylinder at this ix are
// zero (spread_z writes them so) and are not loaded.  Per coset only the 128 in-band
// outputs (q < 64 or q >= 192) are staged and stored.
// MULT = false: mult_y is folded into A'' (permute_cm_kernel) and the outputs are stored as they are
template <bool MULT>
__global__ void __launch_bounds__(FF_NT, 5) pass_y_fast_kernel(PassYFastArgs a)
{
    constexpr int E = FF_L / FF_TPL;
    extern __shared__ float2 smf[];
    float2 *tw = smf;
    float2 *X = tw + FF_L;
    float2 *Ab = X;  // the input lines live in registers once read, so the FFT buffer reuses X
    const float2 *__restrict__ ctw = a.ctw;  // through L1
    const int line = threadIdx.x / FF_TPL, tl = threadIdx.x % FF_TPL;
    const int b = blockIdx.y;
    constexpr int ZT = FF_KZ / FF_NL;
    const int ix = blockIdx.x / ZT;
    const int kz0 = (blockIdx.x % ZT) * FF_NL;
    const float2 *T1 = a.T1 + (long long)b * a.t1_bstride + (long long)ix * FF_L * FF_KZ;
    float2 *T2 = a.T2 + (long long)b * a.t2_bstride + (long long)ix * FF_M * FF_KZ;

    // live rows at this ix: |(ix, iy) - (cx, cy)| <= r
    const float dxl = (float)ix - a.cx;
    const float h2 = a.live_r2 - dxl * dxl;
    int ylo = 0, yhi = -1;
    if (h2 > 0.f) {  // rows within live_r (spread_z writes every tile within live_r + 1)
        const float hh = sqrtf(h2);
        ylo = max(0, (int)ceilf(a.cy - hh));
        yhi = min(FF_L - 1, (int)floorf(a.cy + hh));
    }
    if (ylo > yhi) {  // x plane outside B's support cylinder: its T2 rows are zero, no transform
        for (int e = threadIdx.x; e < FF_M * FF_NL; e += FF_NT) T2[(e / FF_NL) * FF_KZ + kz0 + e % FF_NL] = make_float2(0.f, 0.f);
        return;
    }
    {
        float2 x[E];
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int e = threadIdx.x + FF_NT * m;
            const int n = e / FF_NL, i = e % FF_NL;
            x[m] = (n >= ylo && n <= yhi) ? T1[n * FF_KZ + kz0 + i] : make_float2(0.f, 0.f);
        }
        // the twiddle table after the row loads are issued: both latencies overlap
        load_twiddles<FF_L>(tw, a.tw, threadIdx.x, FF_NT);
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int e = threadIdx.x + FF_NT * m;
            X[(e % FF_NL) * FF_LS + pad(e / FF_NL)] = x[m];
        }
    }
    __syncthreads();
    float2 xr[E];  // the line stays in registers across the cosets: one shared-memory read
    //                (the kernel is L1/shared-bound; 5 blocks/SM at 96 registers)
#pragma unroll
    for (int m = 0; m < E; m++) xr[m] = X[line * FF_LS + pad(tl + FF_TPL * m)];
    __syncthreads();  // X is overwritten by the first FFT exchange below
#pragma unroll 1
    for (int p = 0; p < FF_C; p++) {  // runtime loop: one FFT copy in the instruction cache
        // coset twiddle e^{-2 pi i p (tl + 16 m) / 1024} = c1 W^m, W = e^{-2 pi i p / 64}: one L1
        // load per thread, then a 16-step recurrence (error ~16 ulp, far below the band error;
        // a per-element constant-bank index costed more than the extra multiply)
        // split as e^{-2 pi i p m / 64} (constant bank) x e^{-2 pi i p tl / 1024}, the latter on
        // the last stage's twiddle base (fft_regs_pow, as in fold_fast_kernel)
        const float2 u = __ldg(ctw + FF_L + 4 * tl + p);
        float2 y[E];
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int e = (p * m) & 63;
            y[m] = (p && m) ? cmul(xr[m], make_float2(c_w64.re[e], c_w64.im[e])) : xr[m];
        }
        fft_regs_pow<FF_L, -1, true>(y, Ab + line * FF_LS, u, tl);
        __syncwarp();
        // in-band outputs u = q (q < 64) or q - 128 (q >= 192), times mult_y(ky)
#pragma unroll
        for (int uu = 0; uu < 8; uu++) {
            const int m = uu < 4 ? uu : uu + 8;
            const int q = tl + FF_TPL * m;
            const int ky = FF_C * q + p - (m >= 12 ? FF_G : 0);
            const int u = m < 4 ? q : q - 128;
            if (MULT) {
                const float2 mu = (ky >= -FF_K) ? __ldg(a.mult + ky + FF_K) : make_float2(0.f, 0.f);
                Ab[line * FF_LS + u] = cmul(y[m], mu);
            } else {
                Ab[line * FF_LS + u] = y[m];  // (ky < -K: never stored below)
            }
        }
        __syncthreads();
        const int io = threadIdx.x % FF_NL, u0 = threadIdx.x / FF_NL;  // e = tid + 128 r
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const int u = u0 + (FF_NT / FF_NL) * r, i = io;
            const int q = u < 64 ? u : u + 128;
            const int ky = FF_C * q + p - (q >= 192 ? FF_G : 0);
            if (ky >= -FF_K) T2[(ky + FF_K) * FF_KZ + kz0 + i] = Ab[i * FF_LS + u];
        }
        __syncthreads();
    }
}

bool pass_y_fast_supported(int L, int c, int G, int K, int complex_w)
{
    return L == FF_L && c == FF_C && G == FF_G && K == FF_K && !complex_w;
}

void launch_pass_y_fast(const PassYFastArgs &a, int batch, cudaStream_t s)
{
    const size_t sm = sizeof(float2) * ((size_t)FF_L + FF_NL * FF_LS);
    const dim3 grid((unsigned)(FF_L * (FF_KZ / FF_NL)), batch);
    if (a.mult) {
        cudaFuncSetAttribute(pass_y_fast_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        pass_y_fast_kernel<true><<<grid, FF_NT, sm, s>>>(a);
    } else {
        cudaFuncSetAttribute(pass_y_fast_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        pass_y_fast_kernel<false><<<grid, FF_NT, sm, s>>>(a);
    }
}
