// api.cu -- the C ABI of libballcorr: contexts, validation, plans, orchestration.
//
// Every compute step runs in the kernels of spread*.cu / passes.cu / fold_fast.cu /
// exact.cu / query.cu / validate.cu; this file only validates, plans, allocates and
// launches.  There is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ballcorr.h"
#include "kernels.cuh"

namespace {

const double kPi = 3.14159265358979323846;

// Smoothing window of B in the fused path: the Kaiser-Bessel "blob"
//   phi(r) = C I0(alpha sqrt(1 - (r/W)^2)),  r < W (fine cells),  unit mass,
// whose 3D transform is phi_hat(nu) = F(alpha^2 - (2 pi W nu)^2) / F(alpha^2) with
// F(z^2) = (z cosh z - sinh z) / z^3 (= (sin y - y cos y) / y^3 for z = i y), nu in cycles
// per cell.  W = 4, alpha = 18.5: alias images at |nu| >= 0.75 are <= 6e-6 of the band
// (|nu_i| <= 1/4) and the band corner is damped only 22x (the Gaussian it replaces: 400x).
constexpr double kBlobW = 4.0, kBlobAlpha = 18.5;

struct ShapePlan {
    bool ok = false;
    bool blob = false;   // B smoothed with the KB blob (fused spread + z path), else the Gaussian
    int L = 0, c = 0, G = 0;
    int o[3] = {0, 0, 0};
    double hf = 0, tau = 0, cut = 0;
    float2 *d_mult[3] = {nullptr, nullptr, nullptr};  // axis x, y, z
    float2 *d_ctw = nullptr;                           // coset twiddles [c][L]
};

// One rotation batch in flight: workspaces, reduction keys, B's binning buffers and (for
// concurrent batches) an internal stream.
struct Slot {
    void *ws1 = nullptr, *ws2 = nullptr;
    size_t ws1_bytes = 0, ws2_bytes = 0;
    unsigned long long *keys = nullptr;
    int keys_cap = 0;
    float4 *recA = nullptr;
    int *szcnt = nullptr, *szoff = nullptr, *szlist = nullptr;
    int sz_cap = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
};

struct PendingEvent {
    const char *name;
    cudaEvent_t e0, e1;
};

}  // namespace

struct bc_ctx {
    int device = 0;
    bc_params p{};
    std::string err;

    // shapes (0 = A, 1 = B)
    bool have[2] = {false, false};
    int64_t n[2] = {0, 0};
    std::vector<double> hxyzr[2];
    std::vector<double> hw[2];  // interleaved (re, im)
    float4 *d_balls[2] = {nullptr, nullptr};
    float *d_wre[2] = {nullptr, nullptr};
    float *d_wim[2] = {nullptr, nullptr};
    double4 *d_balls64[2] = {nullptr, nullptr};
    double2 *d_w64[2] = {nullptr, nullptr};

    // spectral
    double P = 0;
    int K = 0, M = 0, Kz = 0, Fz = 0;
    ShapePlan plan[2];
    std::map<int, float2 *> d_tw;  // exp(-2 pi i m / L) per FFT length
    int *d_csr_off = nullptr, *d_csr_idx = nullptr;
    int64_t csr_lo = 0, csr_hi = -1;  // A's balls the per-tile candidate lists cover (hi < 0: all)
    float2 *d_Ahat_part = nullptr;    // partial band spectrum of a slice of A (bc_spectrum_A_partial)
    ResultPeers res_peers{};          // fused result exchange (bc_set_result_peers)
    void *d_res = nullptr;            // job-wide record buffer (bc_result_buffer)
    size_t res_bytes = 0;
    float4 *d_prof = nullptr;     // per-ball radial profile tables of B (cubic Hermite pieces)
    int *d_prof_off = nullptr;
    double dprof = 0;
    // fused spread + z transform of B (spread_z.cu): balls in cell units, per-ball series
    // constants, the universal (Phi1, Phi2) table, B's support radius
    float4 *d_bcells = nullptr;
    float2 *d_g02 = nullptr;
    float4 *d_recB = nullptr;      // (s, w, g0, g2) per ball of B (cells)
    float *d_recWi = nullptr;      // imaginary part of B's weights (complex weights)
    float4 *d_recBim = nullptr;    // (s, Im w, g0, g2) per ball of B (planar complex spread)
    double rc_max_B = 0;           // max (s + W) / hf over B

    float4 *d_phi = nullptr;
    float *d_dec = nullptr;        // 1 / phi_hat(|k| / G_B) indexed by |k|^2 (blob deconvolution)
    int phi_n = 0;
    double phi_U = 0, phi_D = 0;
    double live_r = 0;
    double spread_cells_B = 0;     // sum_j (4/3) pi (s_j / hf + W)^3: window-smoothed footprint cells of B
    int64_t live_tiles_B = 0;      // 4x4 column tiles of B's box inside its support cylinder
    float2 *d_Ahat = nullptr;      // A' = A_hat * origin phase, [ky][kz][kx] natural order
    float2 *d_Ahat_cm = nullptr;   // same, x axis in the coset-major order of B's plan
    size_t Ahat_cm_bytes = 0;
    bool cm_ready = false;
    int MS = 0;                    // row stride of d_Ahat_cm
    int *d_xtab = nullptr;         // fused-fold extraction table of B's x plan
    int2 *d_segs = nullptr;
    bool have_spec = false;

    // workspaces
    Slot slot[2];                  // batches in flight (slot 1 only with concurrent batches)
    cudaEvent_t ev_fork = nullptr;
    float *d_rot = nullptr;
    double *d_rot64 = nullptr;
    int64_t rot_cap = 0;
    void *d_out_stage = nullptr;
    size_t out_stage_bytes = 0;
    void *d_acc = nullptr;          // exact mode: fixed-point accumulators (exact.cu)
    size_t acc_bytes = 0;
    bool ex_ready = false;          // exact_plan() for the current shapes
    double ex_qscale = 1.0;
    bool ex_packed = false;         // fp32: packed 32-bit pair accumulators (exact.cu)
    bool ex_thread_per_knot = false;
    int *d_permB = nullptr;         // B's balls by radius (exact mode, thread-per-knot kernel)
    double *d_part = nullptr;
    long long *d_part_idx = nullptr;
    int part_cap = 0;
    int batch = 1;

    // single-configuration query: uniform grid of A's centres (built on first use)
    bool qgrid_ready = false;
    int *d_qstart = nullptr, *d_qidx = nullptr;
    int qn[3] = {0, 0, 0};
    double qg0[3] = {0, 0, 0}, qcs = 0;
    double *d_qR = nullptr, *d_qt = nullptr, *d_qpart = nullptr, *d_qout = nullptr;
    int64_t q_cap = 0;

    // deferred validation of device-resident inputs (validate.cu): mapped pinned status words
    unsigned *h_status = nullptr, *d_status = nullptr;
    // band-error probe (bc_params.tolerance): estimate for the current shapes, -1 = not run
    bool probe_done = false;
    double probe_err = -1.0;

    // spectral single-configuration query (query_spectral.cu): retained modes in radial-shell
    // order, their A', the shell table of B; rebuilt when m' grows or the shapes / spectrum change
    bool qs_ready = false;
    int64_t qs_m = 0;              // m' the current tables serve (modes counted with multiplicity)
    int qs_nm = 0, qs_nsh = 0;
    int4 *d_qs_modes = nullptr;
    int *d_qs_k2 = nullptr;
    float *d_qs_mult = nullptr;
    float2 *d_qs_Aq = nullptr, *d_qs_bv = nullptr, *d_qs_part = nullptr;
    double *d_qs_mpart = nullptr;
    size_t qs_part_bytes = 0, qs_mpart_bytes = 0;

    // spectral fp64 parity mode (spectral64.cu)
    bool sp64 = false;
    double2 *d_A64 = nullptr, *d_B64 = nullptr, *d_G64 = nullptr;
    double2 *d_sp64_w1 = nullptr, *d_sp64_w2 = nullptr;
    size_t sp64_ws_bytes = 0;
    std::map<long long, double2 *> d_tw64;  // e^{-2 pi i r / G} per period G

    int64_t launches = 0;
    bool prof = false;
    std::vector<PendingEvent> pending;
    std::vector<cudaEvent_t> event_pool;
    std::map<std::string, std::pair<double, int64_t>> stage_ms;
    std::vector<std::string> stage_order;
};

namespace {

bc_status fail(bc_ctx *ctx, bc_status st, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    return st;
}

#define CU(ctx, call)                                                                               \
    do {                                                                                            \
        cudaError_t _e = (call);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            return fail(ctx, _e == cudaErrorMemoryAllocation ? BC_ENOMEM : BC_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(_e), __FILE__, __LINE__);                         \
    } while (0)

#define TRY(expr)                      \
    do {                               \
        bc_status _s = (expr);         \
        if (_s != BC_OK) return _s;    \
    } while (0)

bool friendly(int L)
{
    if (L < 1) return false;
    for (int f : {2, 3, 5})
        while (L % f == 0) L /= f;
    return L == 1;
}

bool is_device_ptr(const void *ptr)
{
    if (!ptr) return false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Host copy of a caller array for the synchronous setup call bc_shape_upload.  A device array
// may have been produced on any of the caller's streams (including non-blocking ones that
// the legacy default stream does not order against), so the device is synchronised first.
bc_status fetch_host(bc_ctx *ctx, const double *src, size_t count, std::vector<double> &dst)
{
    dst.resize(count);
    if (count == 0) return BC_OK;
    if (is_device_ptr(src)) {
        CU(ctx, cudaDeviceSynchronize());
        CU(ctx, cudaMemcpy(dst.data(), src, count * sizeof(double), cudaMemcpyDeviceToHost));
    } else
        memcpy(dst.data(), src, count * sizeof(double));
    return BC_OK;
}

template <typename T>
bc_status dalloc(bc_ctx *ctx, T **ptr, size_t bytes)
{
    if (*ptr) {
        cudaFree(*ptr);
        *ptr = nullptr;
    }
    if (bytes == 0) bytes = 16;
    CU(ctx, cudaMalloc((void **)ptr, bytes));
    return BC_OK;
}

template <typename T>
void dfree(T *&ptr)
{
    if (ptr) cudaFree((void *)ptr);
    ptr = nullptr;
}

// ------------------------------------------------------------------ profiling helpers

cudaEvent_t take_event(bc_ctx *ctx)
{
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// One stage of the path: an NVTX range (header-only NVTX3; a no-op unless a tool such as ncu
// --nvtx attaches) and, with bc_set_profiling, a pair of CUDA events on the stage's stream.
struct StageScope {
    bc_ctx *ctx;
    cudaStream_t s;
    const char *name;
    cudaEvent_t e0 = nullptr;
    StageScope(bc_ctx *c, cudaStream_t st, const char *nm) : ctx(c), s(st), name(nm)
    {
        nvtxRangePushA(nm);
        if (ctx->prof) {
            e0 = take_event(ctx);
            cudaEventRecord(e0, s);
        }
    }
    ~StageScope()
    {
        if (ctx->prof) {
            cudaEvent_t e1 = take_event(ctx);
            cudaEventRecord(e1, s);
            ctx->pending.push_back({name, e0, e1});
        }
        nvtxRangePop();
    }
};

void collect_profile(bc_ctx *ctx)
{
    if (ctx->pending.empty()) return;
    cudaEventSynchronize(ctx->pending.back().e1);
    for (auto &pe : ctx->pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pe.e0, pe.e1);
        auto it = ctx->stage_ms.find(pe.name);
        if (it == ctx->stage_ms.end()) {
            ctx->stage_ms[pe.name] = {ms, 1};
            ctx->stage_order.push_back(pe.name);
        } else {
            it->second.first += ms;
            it->second.second += 1;
        }
        ctx->event_pool.push_back(pe.e0);
        ctx->event_pool.push_back(pe.e1);
    }
    ctx->pending.clear();
}

// ------------------------------------------------------------------ twiddle tables

bc_status ensure_twiddles(bc_ctx *ctx, int L)
{
    if (ctx->d_tw.count(L)) return BC_OK;
    std::vector<float2> t(L);
    for (int m = 0; m < L; m++) {
        const double ang = -2 * kPi * (double)m / L;
        t[m] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
    float2 *d = nullptr;
    CU(ctx, cudaMalloc(&d, sizeof(float2) * L));
    ctx->d_tw[L] = d;
    CU(ctx, cudaMemcpy(d, t.data(), sizeof(float2) * L, cudaMemcpyHostToDevice));
    return BC_OK;
}

// ------------------------------------------------------------------ spectral plan of one shape

// Choose (c, L, G, tau, cut, origin) so that the Gaussian-smoothed density of
// a shape whose centres lie in [lo, hi] (radii <= rmax) fits a box of L fine
// cells at spacing hf = P / G, with G = c L >= 4 (K + 1) (spread oversampling
// sigma_n ~ 2) and alias / truncation level eps.
bc_status plan_shape(bc_ctx *ctx, int which, const double lo[3], const double hi[3], double rmax)
{
    const double P = ctx->P;
    const int K = ctx->K;
    const double eps = ctx->p.spread_eps > 0 ? ctx->p.spread_eps : (ctx->sp64 ? 1e-15 : 1e-7);
    const double lg = std::log(1.0 / eps);
    const int Gmin = 4 * (K + 1);
    double extent = 0;
    for (int a = 0; a < 3; a++) extent = std::max(extent, hi[a] - lo[a]);
    extent += 2 * rmax;

    ShapePlan best;
    double best_cost = 1e300;
    // B with real weights: the fused spread + z kernel with the KB blob when a box size it
    // supports fits (G >= 4 (K + 1) as for the Gaussian: band |nu_i| <= 1/4 of the fine grid)
    // (complex weights: the blob spread to a complex box, then the generic complex-row z pass)
    const bool cplx_w = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    if (which == 1 && !ctx->p.generic_only && !ctx->sp64) {
        for (int c = 1; c <= 8; c++)
            for (int L : {128, 256, 384}) {
                if (!spread_z_supported(L, cplx_w) || c * L < Gmin) continue;
                const int G = c * L;
                const double hf = P / G;
                if (L * hf < extent + 2 * kBlobW * hf + 4 * hf) continue;
                const double cost = (double)G * ((double)L * L + (double)L * ctx->Kz + (double)ctx->M * ctx->Kz);
                if (cost < best_cost) {
                    best_cost = cost;
                    best = ShapePlan();
                    best.ok = true;
                    best.blob = true;
                    best.L = L;
                    best.c = c;
                    best.G = G;
                    best.hf = hf;
                    best.tau = 0;
                    best.cut = kBlobW * hf;
                }
            }
    }
    for (int c = 1; c <= 8 && !best.blob; c++) {
        int L = (Gmin + c - 1) / c;
        for (; L <= 1024; L++) {
            if (!fft_size_supported(L)) continue;
            const int G = c * L;
            const double hf = P / G;
            const double ke = (double)K / P, ka = (double)(G - K) / P;
            const double tau = std::sqrt(lg / (2 * kPi * kPi * (ka * ka - ke * ke)));
            const double cut = tau * std::sqrt(2 * lg);
            if (L * hf >= extent + 2 * cut + 4 * hf) {
                const double cost = (double)G * ((double)L * L + (double)L * ctx->Kz + (double)ctx->M * ctx->Kz);
                if (cost < best_cost) {
                    best_cost = cost;
                    best = ShapePlan();
                    best.ok = true;
                    best.L = L;
                    best.c = c;
                    best.G = G;
                    best.hf = hf;
                    best.tau = tau;
                    best.cut = cut;
                }
                break;
            }
        }
    }
    if (!best.ok)
        return fail(ctx, BC_ERANGE, "shape %c: no spreading box of <= 1024 cells fits extent %.6g with K=%d, P=%.6g",
                    which ? 'B' : 'A', extent, K, P);
    for (int a = 0; a < 3; a++) {
        best.o[a] = (int)std::floor((lo[a] - rmax - best.cut) / best.hf) - 2;
        if ((best.o[a] + best.L) * best.hf < hi[a] + rmax + best.cut + best.hf)
            return fail(ctx, BC_ERANGE, "internal: box does not cover shape %c on axis %d", which ? 'B' : 'A', a);
    }
    // multipliers: hf exp(-2 pi i k o / G) exp(+2 pi^2 tau^2 k^2 / P^2)   (shift + Gaussian deconvolution)
    // and, for A only, the origin phase exp(2 pi i k t0 / P) of the inverse transform
    ShapePlan &dst = ctx->plan[which];
    for (int a = 0; a < 3; a++) dfree(dst.d_mult[a]);
    dfree(dst.d_ctw);
    dst = best;
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    for (int a = 0; a < 3; a++) {
        const int klo = (a == 2 && !cplx) ? 0 : -K;
        const int nk = (a == 2) ? ctx->Kz : ctx->M;
        std::vector<float2> m(nk);
        for (int q = 0; q < nk; q++) {
            const long long k = klo + q;
            const long long num = ((k * dst.o[a]) % dst.G + dst.G) % dst.G;
            double ang = -2 * kPi * (double)num / dst.G;
            if (which == 0) {
                const double x = (double)k * ctx->p.t0[a] / P;
                ang += 2 * kPi * (x - std::floor(x));
            }
            // Gaussian window: separable deconvolution per axis; blob: radial, folded into A''
            const double amp = dst.blob ? dst.hf : dst.hf * std::exp(2 * kPi * kPi * dst.tau * dst.tau * (double)(k * k) / (P * P));
            m[q] = make_float2((float)(amp * std::cos(ang)), (float)(amp * std::sin(ang)));
        }
        TRY(dalloc(ctx, &dst.d_mult[a], sizeof(float2) * nk));
        CU(ctx, cudaMemcpy(dst.d_mult[a], m.data(), sizeof(float2) * nk, cudaMemcpyHostToDevice));
    }
    std::vector<float2> ct((size_t)dst.c * dst.L);
    for (int p = 0; p < dst.c; p++)
        for (int n = 0; n < dst.L; n++) {
            const double ang = -2 * kPi * (double)(((long long)p * n) % dst.G) / dst.G;
            ct[(size_t)p * dst.L + n] = make_float2((float)std::cos(ang), (float)std::sin(ang));
        }
    if (which == 1) {  // extraction table of the fused fold: per FFT output (p, q) of B's x pass
        std::vector<int> xt((size_t)dst.c * dst.L, -1);
        std::vector<int2> sg(8, make_int2(0, 0));
        for (int p = 0; p < dst.c; p++) {
            const CmSeg s = cm_segment(p, dst.L, dst.c, dst.G, K);
            sg[p] = make_int2(s.off, s.cnt);
            for (int q = 0; q < dst.L; q++) {
                int kx = dst.c * q + p;
                if (2 * kx > dst.G) kx -= dst.G;
                if (kx < -K || kx > K) continue;
                int t = (cplx ? -kx : kx) % ctx->p.Np;
                if (t < 0) t += ctx->p.Np;
                xt[(size_t)p * dst.L + q] = (q >= s.qn ? q - s.qn : q + (dst.L - s.qn)) | (t << 16);
            }
        }
        TRY(dalloc(ctx, &ctx->d_xtab, sizeof(int) * xt.size()));
        TRY(dalloc(ctx, &ctx->d_segs, sizeof(int2) * sg.size()));
        CU(ctx, cudaMemcpy(ctx->d_xtab, xt.data(), sizeof(int) * xt.size(), cudaMemcpyHostToDevice));
        CU(ctx, cudaMemcpy(ctx->d_segs, sg.data(), sizeof(int2) * sg.size(), cudaMemcpyHostToDevice));
    }
    TRY(dalloc(ctx, &dst.d_ctw, sizeof(float2) * ct.size()));
    CU(ctx, cudaMemcpy(dst.d_ctw, ct.data(), sizeof(float2) * ct.size(), cudaMemcpyHostToDevice));
    TRY(ensure_twiddles(ctx, dst.L));
    return BC_OK;
}

void shape_bounds(const bc_ctx *ctx, int which, double lo[3], double hi[3], double &rmax, double &rho)
{
    const std::vector<double> &x = ctx->hxyzr[which];
    for (int a = 0; a < 3; a++) {
        lo[a] = 1e300;
        hi[a] = -1e300;
    }
    rmax = 0;
    rho = 0;
    for (int64_t i = 0; i < ctx->n[which]; i++) {
        double nr = 0;
        for (int a = 0; a < 3; a++) {
            lo[a] = std::min(lo[a], x[4 * i + a]);
            hi[a] = std::max(hi[a], x[4 * i + a]);
            nr += x[4 * i + a] * x[4 * i + a];
        }
        rmax = std::max(rmax, x[4 * i + 3]);
        rho = std::max(rho, std::sqrt(nr));
    }
}

bc_status check_support(bc_ctx *ctx)
{
    if (ctx->p.mode != BC_MODE_SPECTRAL || !ctx->have[0] || !ctx->have[1]) return BC_OK;
    if (ctx->n[0] == 0 || ctx->n[1] == 0) return BC_OK;
    double loA[3], hiA[3], rA, rhoA, loB[3], hiB[3], rB, rhoB;
    shape_bounds(ctx, 0, loA, hiA, rA, rhoA);
    shape_bounds(ctx, 1, loB, hiB, rB, rhoB);
    for (int a = 0; a < 3; a++) {
        const double S = std::max(std::fabs(loA[a]), std::fabs(hiA[a])) + rhoB + rA + rB;
        const double need = std::max(S - ctx->p.t0[a], ctx->p.t0[a] + (ctx->p.N - 1) * ctx->p.h + S);
        if (ctx->P < need)
            return fail(ctx, BC_ERANGE,
                        "axis %d: support bound S=%.6g needs period P >= %.6g but P = Np*h = %.6g", a, S, need, ctx->P);
    }
    return BC_OK;
}

// (1_{B(0,s)} * G_tau)(d) in fp64, the same closed form as smoothed_ball() in spread.cu.
double smoothed_ball_host(double s, double d, double tau)
{
    const double a = (s - d) / (std::sqrt(2.0) * tau), b = (s + d) / (std::sqrt(2.0) * tau);
    const double t1 = a >= 0 ? 0.5 * (std::erf(a) + std::erf(b)) : 0.5 * (std::erfc(-a) - std::erfc(b));
    const double x = s * d / (tau * tau);
    double t2;
    if (x < 1e-2) {
        const double x2 = x * x;
        t2 = 2 * s / (tau * std::sqrt(2 * kPi)) * std::exp(-(s * s + d * d) / (2 * tau * tau)) *
             (1 + x2 / 6 + x2 * x2 / 120);
    } else {
        t2 = tau / (d * std::sqrt(2 * kPi)) *
             (std::exp(-(s - d) * (s - d) / (2 * tau * tau)) - std::exp(-(s + d) * (s + d) / (2 * tau * tau)));
    }
    return t1 - t2;
}

// Per-ball cubic-Hermite tables of the smoothed radial profile of shape B on
// intervals of width tau/16 out to s + cut (max interpolation error ~2e-8).
bc_status build_profiles_B(bc_ctx *ctx)
{
    const ShapePlan &pl = ctx->plan[1];
    const double D = pl.tau / 16.0;
    ctx->dprof = D;
    std::vector<float4> tab;
    std::vector<int> off((size_t)std::max<int64_t>(ctx->n[1], 1), 0);
    for (int64_t j = 0; j < ctx->n[1]; j++) {
        const double s = ctx->hxyzr[1][4 * j + 3];
        const int nint = (int)std::ceil((s + pl.cut) / D) + 2;
        off[j] = (int)tab.size();
        std::vector<double> v(nint + 1), dv(nint + 1);
        for (int k = 0; k <= nint; k++) {
            const double d = k * D, h = 1e-4 * D;
            v[k] = smoothed_ball_host(s, d, pl.tau);
            dv[k] = (smoothed_ball_host(s, d + h, pl.tau) - smoothed_ball_host(s, std::fabs(d - h), pl.tau)) / (2 * h) * D;
        }
        for (int k = 0; k < nint; k++) {
            const double p0 = v[k], p1 = v[k + 1], m0 = dv[k], m1 = dv[k + 1];
            tab.push_back(make_float4((float)p0, (float)m0, (float)(-3 * p0 - 2 * m0 + 3 * p1 - m1),
                                      (float)(2 * p0 + m0 - 2 * p1 + m1)));
        }
        if (tab.size() > (size_t)1 << 30) return fail(ctx, BC_ENOMEM, "profile tables too large");
    }
    if (tab.empty()) tab.push_back(make_float4(0, 0, 0, 0));
    TRY(dalloc(ctx, &ctx->d_prof, sizeof(float4) * tab.size()));
    TRY(dalloc(ctx, &ctx->d_prof_off, sizeof(int) * off.size()));
    CU(ctx, cudaMemcpy(ctx->d_prof, tab.data(), sizeof(float4) * tab.size(), cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(ctx->d_prof_off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
    return BC_OK;
}

// ---- KB blob helpers (fp64, host)
double blob_F(double z2)
{
    if (std::fabs(z2) < 1e-3) return 1.0 / 3 + z2 / 30 + z2 * z2 / 840;
    if (z2 > 0) {
        const double z = std::sqrt(z2);
        return (z * std::cosh(z) - std::sinh(z)) / (z * z * z);
    }
    const double y = std::sqrt(-z2);
    return (std::sin(y) - y * std::cos(y)) / (y * y * y);
}
double blob_hat(double nu)  // unit-mass blob transform, nu in cycles per cell
{
    const double t = 2 * kPi * kBlobW * nu;
    return blob_F(kBlobAlpha * kBlobAlpha - t * t) / blob_F(kBlobAlpha * kBlobAlpha);
}
double blob_C() { return 1.0 / (4 * kPi * std::pow(kBlobW, 3) * blob_F(kBlobAlpha * kBlobAlpha)); }
double blob_phi(double r)
{
    if (r >= kBlobW) return 0;
    return blob_C() * std::cyl_bessel_i(0.0, kBlobAlpha * std::sqrt(1 - (r / kBlobW) * (r / kBlobW)));
}
double blob_dphi(double r)
{
    if (r >= kBlobW || r <= 0) return 0;
    const double q = std::sqrt(1 - (r / kBlobW) * (r / kBlobW));
    return blob_C() * std::cyl_bessel_i(1.0, kBlobAlpha * q) * kBlobAlpha * (-r / (kBlobW * kBlobW)) / q;
}
// composite 16-point Gauss-Legendre on [a, b] (the integrands below are smooth on [0, W])
struct GL16 {
    double x[16], w[16];
    GL16()
    {
        for (int i = 0; i < 16; i++) {
            double z = std::cos(kPi * (i + 0.75) / 16.5), pp = 0;
            for (int it = 0; it < 100; it++) {
                double p1 = 1, p2 = 0;
                for (int j = 1; j <= 16; j++) {
                    const double p3 = p2;
                    p2 = p1;
                    p1 = ((2 * j - 1) * z * p2 - (j - 1) * p3) / j;
                }
                pp = 16 * (z * p1 - p2) / (z * z - 1);
                const double dz = p1 / pp;
                z -= dz;
                if (std::fabs(dz) < 1e-16) break;
            }
            x[i] = z;
            w[i] = 2 / ((1 - z * z) * pp * pp);
        }
    }
};
template <typename Fn>
double gl_integrate(Fn f, double a, double b, int panels = 16)
{
    static const GL16 gl;  // thread-safe one-time initialisation (C++11 static)
    const double *x = gl.x, *w = gl.w;
    double sum = 0;
    const double hp = (b - a) / panels;
    for (int p = 0; p < panels; p++) {
        const double m = a + (p + 0.5) * hp, r = 0.5 * hp;
        for (int i = 0; i < 16; i++) sum += w[i] * r * f(m + r * x[i]);
    }
    return sum;
}

// Tables of the fused spread + z kernel (cell units).  For a radial window phi of
// support W, the window-smoothed ball profile is exactly
//   g(s, d) = Phi1(s-d) + Phi1(s+d) - (Phi2(s-d) - Phi2(s+d)) / d,
//   Phi1(u) = sgn(u) 2 pi [int_0^|u| t^2 phi + |u| Q(|u|)],   Phi2(u) = pi int_|u|^W t (t^2 - u^2) phi,
//   Q(a) = int_a^W t phi,  Phi1 = +-1/2 and Phi2 = 0 for |u| >= W;
// cubic Hermite pieces of width W/48 on [-W, W] (fp64 -> fp32), and per ball the d -> 0
// series g = g0 + g2 d^2 with g0(s) = 2 Phi1(s) - 4 pi s Q(s), g2(s) = (2 pi / 3) s^2 phi'(s).
bc_status build_spread_z_tables(bc_ctx *ctx)
{
    const ShapePlan &pl = ctx->plan[1];
    const double U = kBlobW, D = kBlobW / 48;  // cubic Hermite error ~2e-7 of the unit density
    auto Q = [&](double a) { return a >= U ? 0.0 : gl_integrate([](double t) { return t * blob_phi(t); }, a, U); };
    auto M2 = [&](double a) { return gl_integrate([](double t) { return t * t * blob_phi(t); }, 0, std::min(a, U)); };
    auto phi1 = [&](double u) {
        const double a = std::fabs(u);
        if (a >= U) return u > 0 ? 0.5 : -0.5;
        const double v = 2 * kPi * (M2(a) + a * Q(a));
        return u >= 0 ? v : -v;
    };
    auto dphi1 = [&](double u) { return 2 * kPi * Q(std::fabs(u)); };
    auto phi2 = [&](double u) {
        const double a = std::fabs(u);
        if (a >= U) return 0.0;
        return kPi * gl_integrate([a](double t) { return t * (t * t - a * a) * blob_phi(t); }, a, U);
    };
    auto dphi2 = [&](double u) { return -2 * kPi * u * Q(std::fabs(u)); };
    const int n = (int)std::lround(2 * U / D);
    std::vector<float4> tab((size_t)2 * n);
    auto herm = [&](double p0, double m0, double p1, double m1) {
        return make_float4((float)p0, (float)m0, (float)(-3 * p0 - 2 * m0 + 3 * p1 - m1), (float)(2 * p0 + m0 - 2 * p1 + m1));
    };
    std::vector<double> v1(n + 1), d1(n + 1), v2(n + 1), d2(n + 1);
    for (int i = 0; i <= n; i++) {
        const double u = -U + i * D;
        v1[i] = phi1(u);
        d1[i] = dphi1(u) * D;
        v2[i] = phi2(u);
        d2[i] = dphi2(u) * D;
    }
    for (int i = 0; i < n; i++) {  // [n] Phi1 pieces, then [n] Phi2 pieces
        tab[i] = herm(v1[i], d1[i], v1[i + 1], d1[i + 1]);
        tab[n + i] = herm(v2[i], d2[i], v2[i + 1], d2[i + 1]);
    }
    const int64_t nb = ctx->n[1];
    const size_t cnt = (size_t)std::max<int64_t>(nb, 1);
    std::vector<float4> bc(cnt, make_float4(0, 0, 0, 1));
    std::vector<float2> g(cnt, make_float2(0, 0));
    for (int64_t j = 0; j < nb; j++) {
        const double *x = &ctx->hxyzr[1][4 * j];
        const double sc = x[3] / pl.hf;
        bc[j] = make_float4((float)(x[0] / pl.hf), (float)(x[1] / pl.hf), (float)(x[2] / pl.hf), (float)sc);
        g[j] = make_float2((float)(2 * phi1(sc) - 4 * kPi * sc * Q(sc)), (float)(2 * kPi / 3 * sc * sc * blob_dphi(sc)));
    }
    // radial deconvolution 1 / phi_hat(|k| / G) for every |k|^2 of the cube band
    const size_t nk2 = (size_t)3 * ctx->K * ctx->K + 1;
    std::vector<float> dec(nk2);
    for (size_t q = 0; q < nk2; q++) dec[q] = (float)(1.0 / blob_hat(std::sqrt((double)q) / pl.G));
    std::vector<float4> rb(cnt, make_float4(0, 0, 0, 0));
    ctx->rc_max_B = 0;
    for (int64_t j = 0; j < nb; j++) {
        rb[j] = make_float4(bc[j].w, (float)ctx->hw[1][2 * j], g[j].x, g[j].y);
        ctx->rc_max_B = std::max(ctx->rc_max_B, ctx->hxyzr[1][4 * j + 3] / pl.hf + kBlobW);
    }
    TRY(dalloc(ctx, &ctx->d_recB, sizeof(float4) * cnt));
    CU(ctx, cudaMemcpy(ctx->d_recB, rb.data(), sizeof(float4) * cnt, cudaMemcpyHostToDevice));
    std::vector<float> wi(cnt, 0.f);
    for (int64_t j = 0; j < nb; j++) wi[j] = (float)ctx->hw[1][2 * j + 1];
    TRY(dalloc(ctx, &ctx->d_recWi, sizeof(float) * cnt));
    CU(ctx, cudaMemcpy(ctx->d_recWi, wi.data(), sizeof(float) * cnt, cudaMemcpyHostToDevice));
    for (int64_t j = 0; j < nb; j++) rb[j].y = wi[j];  // (s, Im w, g0, g2) for the planar spread
    TRY(dalloc(ctx, &ctx->d_recBim, sizeof(float4) * cnt));
    CU(ctx, cudaMemcpy(ctx->d_recBim, rb.data(), sizeof(float4) * cnt, cudaMemcpyHostToDevice));
    ctx->slot[0].sz_cap = ctx->slot[1].sz_cap = 0;  // binning workspace resized at the next correlate
    TRY(dalloc(ctx, &ctx->d_phi, sizeof(float4) * tab.size()));
    TRY(dalloc(ctx, &ctx->d_bcells, sizeof(float4) * cnt));
    TRY(dalloc(ctx, &ctx->d_g02, sizeof(float2) * cnt));
    TRY(dalloc(ctx, &ctx->d_dec, sizeof(float) * nk2));
    CU(ctx, cudaMemcpy(ctx->d_phi, tab.data(), sizeof(float4) * tab.size(), cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(ctx->d_bcells, bc.data(), sizeof(float4) * cnt, cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(ctx->d_g02, g.data(), sizeof(float2) * cnt, cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(ctx->d_dec, dec.data(), sizeof(float) * nk2, cudaMemcpyHostToDevice));
    ctx->phi_n = n;
    ctx->phi_U = U;
    ctx->phi_D = D;
    return BC_OK;
}

// Generic (Gaussian) plan of B: cell-unit balls and the footprint radius for the per-rotation
// 16 x 16-column binning (the spread_z binning kernels), so that each 16^3 spread tile scans
// only the balls listed in its column bin instead of all of B (boxes of 16-multiple edge).
bool generic_bins_B(const bc_ctx *ctx) { return !ctx->plan[1].blob && ctx->plan[1].L % 16 == 0 && !ctx->sp64; }

bc_status build_generic_bins_B(bc_ctx *ctx)
{
    if (!generic_bins_B(ctx)) return BC_OK;
    const ShapePlan &pl = ctx->plan[1];
    const int64_t nb = ctx->n[1];
    const size_t cnt = (size_t)std::max<int64_t>(nb, 1);
    std::vector<float4> bc(cnt, make_float4(0, 0, 0, 1));
    ctx->rc_max_B = 0;
    for (int64_t j = 0; j < nb; j++) {
        const double *x = &ctx->hxyzr[1][4 * j];
        bc[j] = make_float4((float)(x[0] / pl.hf), (float)(x[1] / pl.hf), (float)(x[2] / pl.hf), (float)(x[3] / pl.hf));
        ctx->rc_max_B = std::max(ctx->rc_max_B, (x[3] + pl.cut) / pl.hf);
    }
    TRY(dalloc(ctx, &ctx->d_bcells, sizeof(float4) * cnt));
    CU(ctx, cudaMemcpy(ctx->d_bcells, bc.data(), sizeof(float4) * cnt, cudaMemcpyHostToDevice));
    ctx->slot[0].sz_cap = ctx->slot[1].sz_cap = 0;  // binning workspace resized at the next correlate
    return BC_OK;
}

bool use_spread_z(const bc_ctx *ctx) { return ctx->plan[1].ok && ctx->plan[1].blob; }


// the docking plan shape on dock_fast.cu's kernels (blob spread to a complex box, then the
// compile-time z / y passes and fold)
bool use_dock_fast(const bc_ctx *ctx)
{
    const ShapePlan &pb = ctx->plan[1];
    return use_spread_z(ctx) && !ctx->p.generic_only &&
           dock_fast_supported(pb.L, pb.c, pb.G, ctx->K, ctx->p.Np, ctx->p.weights == BC_WEIGHTS_COMPLEX);
}

// Real-weight blob plans (spread_z -> z unpack -> y pass -> fold, every fold variant reading A''
// mode by mode) and the docking plan (dock_fast.cu): B's y and z multipliers are folded into A''
// with the x ones, so the z unpack and B's y / z passes store their outputs without them (sweep
// y pass 0.124 -> 0.099 ms per rotation).  generic_only keeps them in the passes (the reference
// path of the fused-vs-generic tests).
bool yz_in_A(const bc_ctx *ctx)
{
#ifdef BC_NO_YZ_FOLD
    return false;
#endif
    return (use_spread_z(ctx) && !ctx->p.generic_only && ctx->p.weights != BC_WEIGHTS_COMPLEX) || use_dock_fast(ctx);
}

// Uniform grid of A's centres for bc_evaluate_points: cell size cs >= max r_A + max s_B, so
// every A ball overlapping a B ball centred at c lies in the 27 cells around c.  CSR, ball
// order within each cell (deterministic sums).  At most 128 cells per axis.
bc_status build_query_grid(bc_ctx *ctx)
{
    const std::vector<double> &x = ctx->hxyzr[0];
    const int64_t nA = ctx->n[0];
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300}, ra = 0, sb = 0;
    for (int64_t i = 0; i < nA; i++) {
        for (int d = 0; d < 3; d++) {
            lo[d] = std::min(lo[d], x[4 * i + d]);
            hi[d] = std::max(hi[d], x[4 * i + d]);
        }
        ra = std::max(ra, x[4 * i + 3]);
    }
    for (int64_t j = 0; j < ctx->n[1]; j++) sb = std::max(sb, ctx->hxyzr[1][4 * j + 3]);
    double cs = ra + sb;
    for (int d = 0; d < 3; d++) cs = std::max(cs, (hi[d] - lo[d]) / 127.0);
    cs *= 1.0 + 1e-9;
    int nc = 1;
    for (int d = 0; d < 3; d++) {
        ctx->qg0[d] = lo[d];
        ctx->qn[d] = std::max(1, (int)std::floor((hi[d] - lo[d]) / cs) + 1);
        nc *= ctx->qn[d];
    }
    ctx->qcs = cs;
    std::vector<int> cell((size_t)nA), start((size_t)nc + 1, 0), idx((size_t)std::max<int64_t>(nA, 1));
    for (int64_t i = 0; i < nA; i++) {
        int g[3];
        for (int d = 0; d < 3; d++)
            g[d] = std::min(ctx->qn[d] - 1, std::max(0, (int)std::floor((x[4 * i + d] - lo[d]) / cs)));
        cell[i] = (g[0] * ctx->qn[1] + g[1]) * ctx->qn[2] + g[2];
        start[cell[i] + 1]++;
    }
    for (int c = 0; c < nc; c++) start[c + 1] += start[c];
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (int64_t i = 0; i < nA; i++) idx[fill[cell[i]]++] = (int)i;
    TRY(dalloc(ctx, &ctx->d_qstart, sizeof(int) * start.size()));
    TRY(dalloc(ctx, &ctx->d_qidx, sizeof(int) * idx.size()));
    CU(ctx, cudaMemcpy(ctx->d_qstart, start.data(), sizeof(int) * start.size(), cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(ctx->d_qidx, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice));
    ctx->qgrid_ready = true;
    return BC_OK;
}

bc_status build_csr_A(bc_ctx *ctx, int64_t lo = 0, int64_t hi = -1)
{
    if (hi < 0) hi = ctx->n[0];
    ctx->csr_lo = lo;
    ctx->csr_hi = hi == ctx->n[0] ? -1 : hi;
    const ShapePlan &pl = ctx->plan[0];
    const int tpa = (pl.L + 15) / 16;
    const int ntiles = tpa * tpa * tpa;
    std::vector<std::vector<int>> lists(ntiles);
    const std::vector<double> &x = ctx->hxyzr[0];
    for (int64_t i = lo; i < hi; i++) {
        double u[3];
        int t0[3], t1[3];
        const double rc = (x[4 * i + 3] + pl.cut) / pl.hf;
        for (int a = 0; a < 3; a++) {
            u[a] = x[4 * i + a] / pl.hf - pl.o[a];
            t0[a] = std::max(0, (int)std::floor((u[a] - rc - 1) / 16));
            t1[a] = std::min(tpa - 1, (int)std::floor((u[a] + rc + 1) / 16));
        }
        for (int tx = t0[0]; tx <= t1[0]; tx++)
            for (int ty = t0[1]; ty <= t1[1]; ty++)
                for (int tz = t0[2]; tz <= t1[2]; tz++) lists[(tx * tpa + ty) * tpa + tz].push_back((int)i);
    }
    std::vector<int> off(ntiles + 1, 0), idx;
    for (int t = 0; t < ntiles; t++) off[t + 1] = off[t] + (int)lists[t].size();
    idx.reserve(off[ntiles]);
    for (int t = 0; t < ntiles; t++) idx.insert(idx.end(), lists[t].begin(), lists[t].end());
    TRY(dalloc(ctx, &ctx->d_csr_off, sizeof(int) * off.size()));
    TRY(dalloc(ctx, &ctx->d_csr_idx, sizeof(int) * std::max<size_t>(1, idx.size())));
    CU(ctx, cudaMemcpy(ctx->d_csr_off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
    if (!idx.empty()) CU(ctx, cudaMemcpy(ctx->d_csr_idx, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice));
    return BC_OK;
}

bc_status ensure_ws(bc_ctx *ctx, void **ptr, size_t &cur, size_t need)
{
    if (need <= cur && *ptr) return BC_OK;
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    cur = 0;
    CU(ctx, cudaMalloc(ptr, need));
    cur = need;
    return BC_OK;
}

// per-rotation sizes (bytes) of the two ping-pong spectral workspaces of a shape
//   ws1: box -> T2 -> X1        ws2: T1 -> F (B) or A_hat staging -> Y1
void spectral_ws_sizes(const bc_ctx *ctx, int which, size_t &s1, size_t &s2)
{
    const ShapePlan &pl = ctx->plan[which];
    const size_t L = pl.L, Kz = ctx->Kz, M = ctx->M, Np = ctx->p.Np, N = ctx->p.N, Fz = ctx->Fz;
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    const size_t box = L * L * L * (cplx ? 8 : 4);
    // (the docking kernels keep T1 / T2 rows at pitch dock_t_pitch() >= Kz)
    const size_t Pk = (which == 1 && use_dock_fast(ctx)) ? std::max(Kz, dock_t_pitch()) : Kz;
    const size_t T1 = L * L * Pk * 8, T2 = L * std::max(M, Pk) * Pk * 8;
    const size_t Fzp = (Fz + 7) & ~(size_t)7;  // padded row pitch of X1 / Y1 on the fast plan
    const size_t F = Np * Np * Fz * 8, X1 = N * Np * Fzp * 8, Y1 = N * N * Fzp * 8;
    s1 = std::max(std::max(box, T2), X1);
    s2 = std::max(std::max(std::max(T1, F), Y1), X1);  // X1 sits in ws2 when the inverse x is fused
    s1 = (s1 + 255) / 256 * 256;
    s2 = (s2 + 255) / 256 * 256;
}

// spread + z + y passes of one shape; for A also the x pass into A_hat.
bc_status shape_spectrum(bc_ctx *ctx, int which, const float *d_rot, int nb, void *ws1, void *ws2,
                         size_t s1_per, size_t s2_per, cudaStream_t s, Slot &sl)
{
    const ShapePlan &pl = ctx->plan[which];
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    const int L = pl.L;
    const float2 *tw = ctx->d_tw[L];
    if (which == 1 && use_spread_z(ctx)) {
        const int n = (int)ctx->n[1];
        const int nbins = spread_z_bins(L);
        const long long lstride = (long long)n * spread_z_bins_per_ball((float)ctx->rc_max_B);
        if (sl.sz_cap < nb) {
            TRY(dalloc(ctx, &sl.recA, sizeof(float4) * (size_t)n * nb));
            TRY(dalloc(ctx, &sl.szcnt, sizeof(int) * (size_t)nbins * nb));
            TRY(dalloc(ctx, &sl.szoff, sizeof(int) * (size_t)nbins * nb));
            TRY(dalloc(ctx, &sl.szlist, sizeof(int) * (size_t)lstride * nb));
            sl.sz_cap = nb;
        }
        {
            SzBinArgs bn{};
            bn.n = n;
            bn.balls = ctx->d_bcells;
            bn.rot = d_rot;
            bn.ox = (float)pl.o[0];
            bn.oy = (float)pl.o[1];
            bn.oz = (float)pl.o[2];
            bn.cut = (float)(pl.cut / pl.hf);
            bn.recA = sl.recA;
            bn.bpa = spread_z_bins_per_axis(L);
            bn.nbins = nbins;
            bn.counts = sl.szcnt;
            bn.offs = sl.szoff;
            bn.lists = sl.szlist;
            bn.list_stride = lstride;
            StageScope sc(ctx, s, "bin_B");
            launch_spread_z_bin(bn, nb, s);
            ctx->launches += 3;
        }
        SpreadZArgs a{};
        a.L = L;
        a.K = ctx->K;
        a.c = pl.c;
        a.G = pl.G;
        a.n_balls = n;
        a.recA = sl.recA;
        a.recB = ctx->d_recB;
        a.recWi = ctx->d_recWi;
        a.recBim = ctx->d_recBim;
        a.cplx = cplx ? 1 : 0;
        a.planar = (cplx && use_dock_fast(ctx)) ? 1 : 0;  // pass_z_dk reads the planar box
        a.counts = sl.szcnt;
        a.offs = sl.szoff;
        a.lists = sl.szlist;
        a.nbins = nbins;
        a.list_stride = lstride;
        a.phi = ctx->d_phi;
        a.phi_n = ctx->phi_n;
        a.phi_U = (float)ctx->phi_U;
        a.phi_invD = (float)(1.0 / ctx->phi_D);
        a.cx = (float)(-pl.o[0]);
        a.cy = (float)(-pl.o[1]);
        a.live_r2 = (float)(ctx->live_r * ctx->live_r);
        a.zero_r2 = (float)((ctx->live_r + 1) * (ctx->live_r + 1));
        // complex weights: the complex box, its unwritten zero tiles skipped by the z pass below
        a.skip_zero = (cplx || pass_y_fast_supported(L, pl.c, pl.G, ctx->K, cplx)) ? 1 : 0;
        // spread to the box (ws1, free until the y pass writes T2 there) and transform it in a
        // second kernel -- the spread alone runs at twice the occupancy (sweep 0.694 -> 0.671,
        // torus 0.130 -> 0.122 ms per rotation); complex weights always take the box
        if (a.skip_zero || !cplx) {
            a.box = (float *)ws1;
            a.box_bstride = (long long)(s1_per / 4);
        }
        a.mult_z = yz_in_A(ctx) ? nullptr : pl.d_mult[2];
        a.tw = tw;
        a.ctw = pl.d_ctw;
        a.out = (float2 *)ws2;
        a.out_bstride = (long long)(s2_per / 8);
        StageScope sc(ctx, s, "spread_z_B");
        if (!launch_spread_z(a, nb, s))
            return fail(ctx, BC_EUNSUPPORTED, "spread_z: profile table (n = %d, U = %g) or box L = %d not compiled in",
                        a.phi_n, (double)a.phi_U, a.L);
        ctx->launches += ((a.box && !cplx) || a.planar) ? 2 : 1;
    } else {
        SpreadArgs a{};
        if (which == 1 && generic_bins_B(ctx)) {  // per-rotation column bins (spread_z.cu kernels)
            const int n = (int)ctx->n[1];
            const int nbins = spread_z_bins(L);
            const long long lstride = (long long)n * spread_z_bins_per_ball((float)ctx->rc_max_B);
            if (sl.sz_cap < nb) {
                TRY(dalloc(ctx, &sl.recA, sizeof(float4) * (size_t)n * nb));
                TRY(dalloc(ctx, &sl.szcnt, sizeof(int) * (size_t)nbins * nb));
                TRY(dalloc(ctx, &sl.szoff, sizeof(int) * (size_t)nbins * nb));
                TRY(dalloc(ctx, &sl.szlist, sizeof(int) * (size_t)lstride * nb));
                sl.sz_cap = nb;
            }
            SzBinArgs bn{};
            bn.n = n;
            bn.balls = ctx->d_bcells;
            bn.rot = d_rot;
            bn.ox = (float)pl.o[0];
            bn.oy = (float)pl.o[1];
            bn.oz = (float)pl.o[2];
            bn.cut = (float)(pl.cut / pl.hf);
            bn.recA = sl.recA;
            bn.bpa = spread_z_bins_per_axis(L);
            bn.nbins = nbins;
            bn.counts = sl.szcnt;
            bn.offs = sl.szoff;
            bn.lists = sl.szlist;
            bn.list_stride = lstride;
            StageScope sc(ctx, s, "bin_B");
            launch_spread_z_bin(bn, nb, s);
            ctx->launches += 3;
            a.bin_counts = sl.szcnt;
            a.bin_offs = sl.szoff;
            a.bin_lists = sl.szlist;
            a.bin_stride = lstride;
            a.nbins = nbins;
            a.bpa = bn.bpa;
        }
        a.L = L;
        a.ox = pl.o[0];
        a.oy = pl.o[1];
        a.oz = pl.o[2];
        a.hf = (float)pl.hf;
        a.inv_hf = (float)(1.0 / pl.hf);
        a.tau = (float)pl.tau;
        a.cut = (float)pl.cut;
        a.n_balls = (int)ctx->n[which];
        a.balls = ctx->d_balls[which];
        a.w_re = ctx->d_wre[which];
        a.w_im = ctx->d_wim[which];
        a.csr_off = which == 0 ? ctx->d_csr_off : nullptr;
        a.csr_idx = which == 0 ? ctx->d_csr_idx : nullptr;
        a.rot = d_rot;
        a.complex_w = cplx;
        a.out = ws1;
        a.out_batch_stride = (long long)(s1_per / (cplx ? 8 : 4));
        a.tiles_per_axis = (L + 15) / 16;
        if (which == 1) {
            a.prof = ctx->d_prof;
            a.prof_off = ctx->d_prof_off;
            a.inv_dprof = (float)(1.0 / ctx->dprof);
        }
        StageScope sc(ctx, s, which ? "spread_B" : "spread_A");
        launch_spread(a, nb, s);
        ctx->launches++;
    }
    PassArgs base{};
    base.L = L;
    base.c = pl.c;
    base.G = pl.G;
    base.signed_k = 1;
    base.tw = tw;
    base.ctw = pl.d_ctw;
    if (which == 1 && use_dock_fast(ctx)) {
        DockPassArgs a{};
        a.tw = tw;
        a.ctw = pl.d_ctw;
        a.cx = (float)(-pl.o[0]);
        a.cy = (float)(-pl.o[1]);
        a.live_r2 = (float)(ctx->live_r * ctx->live_r);
        a.zero_r2 = (float)((ctx->live_r + 1) * (ctx->live_r + 1));
        {
            DockPassArgs z = a;
            z.mult = yz_in_A(ctx) ? nullptr : pl.d_mult[2];
            z.in = (const float2 *)ws1;
            z.in_bstride = (long long)(s1_per / 8);
            z.out = (float2 *)ws2;
            z.out_bstride = (long long)(s2_per / 8);
            StageScope sc(ctx, s, "pass_z_dk");
            launch_pass_z_dk(z, nb, s);
            ctx->launches++;
        }
        {
            DockPassArgs y = a;
            y.mult = yz_in_A(ctx) ? nullptr : pl.d_mult[1];
            y.in = (const float2 *)ws2;
            y.in_bstride = (long long)(s2_per / 8);
            y.out = (float2 *)ws1;
            y.out_bstride = (long long)(s1_per / 8);
            StageScope sc(ctx, s, "pass_y_dk");
            launch_pass_y_dk(y, nb, s);
            ctx->launches++;
        }
        CU(ctx, cudaGetLastError());
        return BC_OK;
    }
    if (!(which == 1 && use_spread_z(ctx)) || (which == 1 && cplx)) {
        PassArgs a = base;
        a.klo = cplx ? -ctx->K : 0;
        a.nk = ctx->Kz;
        a.mult = pl.d_mult[2];
        a.lines = (long long)L * L;
        a.in = ws1;
        a.in_real = !cplx;
        a.in_bstride = (long long)(s1_per / (cplx ? 8 : 4));
        a.out = (float2 *)ws2;
        a.out_bstride = (long long)(s2_per / 8);
        if (which == 1 && use_spread_z(ctx)) {  // the complex box of spread_z: skip its zero tiles
            a.zskip = 2;                          // (the y pass below reads only live rows)
            a.zcx = (float)(-pl.o[0]);
            a.zcy = (float)(-pl.o[1]);
            a.zero_r2 = (float)((ctx->live_r + 1) * (ctx->live_r + 1));
        }
        StageScope sc(ctx, s, which ? "pass_z_B" : "pass_z_A");
        launch_pass(a, 0, nb, s);
        ctx->launches++;
    }
    if (which == 1 && use_spread_z(ctx) && pass_y_fast_supported(L, pl.c, pl.G, ctx->K, cplx)) {
        PassYFastArgs a{};
        a.tw = tw;
        a.ctw = pl.d_ctw;
        a.mult = yz_in_A(ctx) ? nullptr : pl.d_mult[1];
        a.T1 = (const float2 *)ws2;
        a.t1_bstride = (long long)(s2_per / 8);
        a.T2 = (float2 *)ws1;
        a.t2_bstride = (long long)(s1_per / 8);
        a.cx = (float)(-pl.o[0]);
        a.cy = (float)(-pl.o[1]);
        a.live_r2 = (float)(ctx->live_r * ctx->live_r);
        StageScope sc(ctx, s, "pass_y_fast");
        launch_pass_y_fast(a, nb, s);
        ctx->launches++;
    } else {
        PassArgs a = base;
        a.klo = -ctx->K;
        a.nk = ctx->M;
        a.mult = (which == 1 && yz_in_A(ctx)) ? nullptr : pl.d_mult[1];
        a.O = L;
        a.I = ctx->Kz;
        a.in = ws2;
        a.in_bstride = (long long)(s2_per / 8);
        a.out = (float2 *)ws1;
        a.out_bstride = (long long)(s1_per / 8);
        if (which == 1 && use_spread_z(ctx)) {  // T1 of the complex box: live rows only
            a.ylive = 1;
            a.zcx = (float)(-pl.o[0]);
            a.zcy = (float)(-pl.o[1]);
            a.live_r2 = (float)(ctx->live_r * ctx->live_r);
        }
        StageScope sc(ctx, s, which ? "pass_y_B" : "pass_y_A");
        launch_pass(a, 1, nb, s);
        ctx->launches++;
    }
    if (which == 0) {
        PassArgs a = base;
        a.klo = -ctx->K;
        a.nk = ctx->M;
        a.mult = pl.d_mult[0];
        a.O = 1;
        a.I = ctx->M * ctx->Kz;
        a.in = ws1;
        a.in_bstride = (long long)(s1_per / 8);
        a.out = ctx->d_Ahat;
        a.out_bstride = 0;
        StageScope sc(ctx, s, "pass_x_A");
        launch_pass(a, 2, nb, s);
        ctx->launches++;
    }
    CU(ctx, cudaGetLastError());
    return BC_OK;
}

bc_status upload_shape_device(bc_ctx *ctx, int which)
{
    const int64_t n = ctx->n[which];
    const size_t cnt = (size_t)std::max<int64_t>(n, 1);
    std::vector<float4> b(cnt);
    std::vector<float> wr(cnt), wi(cnt);
    std::vector<double4> b64(cnt);
    std::vector<double2> w64(cnt);
    for (int64_t i = 0; i < n; i++) {
        const double *x = &ctx->hxyzr[which][4 * i];
        b[i] = make_float4((float)x[0], (float)x[1], (float)x[2], (float)x[3]);
        b64[i] = make_double4(x[0], x[1], x[2], x[3]);
        wr[i] = (float)ctx->hw[which][2 * i];
        wi[i] = (float)ctx->hw[which][2 * i + 1];
        w64[i] = make_double2(ctx->hw[which][2 * i], ctx->hw[which][2 * i + 1]);
    }
    TRY(dalloc(ctx, &ctx->d_balls[which], sizeof(float4) * cnt));
    TRY(dalloc(ctx, &ctx->d_wre[which], sizeof(float) * cnt));
    TRY(dalloc(ctx, &ctx->d_wim[which], sizeof(float) * cnt));
    TRY(dalloc(ctx, &ctx->d_balls64[which], sizeof(double4) * cnt));
    TRY(dalloc(ctx, &ctx->d_w64[which], sizeof(double2) * cnt));
    CU(ctx, cudaMemcpy(ctx->d_balls[which], b.data(), sizeof(float4) * cnt, cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(ctx->d_wre[which], wr.data(), sizeof(float) * cnt, cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(ctx->d_wim[which], wi.data(), sizeof(float) * cnt, cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(ctx->d_balls64[which], b64.data(), sizeof(double4) * cnt, cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(ctx->d_w64[which], w64.data(), sizeof(double2) * cnt, cudaMemcpyHostToDevice));
    return BC_OK;
}

// Tolerance on |R R^T - I| entries: 1e-5 for the fp32 path, 1e-12 for fp64.
double rot_tol(const bc_ctx *ctx) { return ctx->p.precision == BC_FP64 ? 1e-12 : 1e-5; }

// A violation recorded on the device by validate.cu (deferred BC_EINVAL); resets the words.
bc_status check_deferred(bc_ctx *ctx)
{
    if (!ctx->h_status) return BC_OK;
    volatile unsigned *st = ctx->h_status;
    const unsigned flags = st[0];
    if (!flags) return BC_OK;
    const unsigned idx = st[1];
    st[0] = 0;
    st[1] = 0xffffffffu;
    return fail(ctx, BC_EINVAL, "deferred (device-resident input of an earlier call): entry %u: %s%s%s%s", idx,
                (flags & BC_DEFER_NONFINITE_R) ? "non-finite R " : "",
                (flags & BC_DEFER_NOT_ORTHONORMAL) ? "R R^T deviates from I " : "",
                (flags & BC_DEFER_DET) ? "det R <= 0 " : "", (flags & BC_DEFER_NONFINITE_T) ? "non-finite t" : "");
}

bc_status validate_rotations(bc_ctx *ctx, const double *R, int64_t n_rot)
{
    const double tol = rot_tol(ctx);
    for (int64_t r = 0; r < n_rot; r++) {
        const double *m = &R[9 * r];
        for (int q = 0; q < 9; q++)
            if (!std::isfinite(m[q])) return fail(ctx, BC_EINVAL, "rotation %lld has a non-finite entry", (long long)r);
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) {
                double d = 0;
                for (int k = 0; k < 3; k++) d += m[3 * i + k] * m[3 * j + k];
                if (std::fabs(d - (i == j ? 1.0 : 0.0)) > tol)
                    return fail(ctx, BC_EINVAL, "rotation %lld: R R^T deviates from I by %.3g", (long long)r,
                                std::fabs(d - (i == j ? 1.0 : 0.0)));
            }
        const double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                           m[2] * (m[3] * m[7] - m[4] * m[6]);
        if (det <= 0) return fail(ctx, BC_EINVAL, "rotation %lld has det %.6g <= 0", (long long)r, det);
    }
    return BC_OK;
}

bc_status ensure_deferred_status(bc_ctx *ctx)
{
    if (ctx->h_status) return BC_OK;
    unsigned *h = nullptr;
    CU(ctx, cudaHostAlloc((void **)&h, 2 * sizeof(unsigned), cudaHostAllocMapped));
    h[0] = 0;
    h[1] = 0xffffffffu;
    unsigned *d = nullptr;
    cudaError_t e = cudaHostGetDevicePointer((void **)&d, h, 0);
    if (e != cudaSuccess) {
        cudaFreeHost(h);
        return fail(ctx, BC_ECUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
    }
    ctx->h_status = h;
    ctx->d_status = d;
    return BC_OK;
}

// Rotations of the call into ctx->d_rot (fp32, spectral path) and ctx->d_rot64 (fp64, exact
// mode), on `s`.  Host R was validated by the caller and is copied; device R is validated
// and converted by validate.cu with no host round trip (violations: deferred BC_EINVAL).
bc_status prepare_rotations(bc_ctx *ctx, const double *R, bool dev_R, int64_t n_rot, cudaStream_t s)
{
    TRY(ensure_deferred_status(ctx));
    if (n_rot > ctx->rot_cap) {
        TRY(dalloc(ctx, &ctx->d_rot, sizeof(float) * 9 * n_rot));
        TRY(dalloc(ctx, &ctx->d_rot64, sizeof(double) * 9 * n_rot));
        ctx->rot_cap = n_rot;
    }
    RotPrepArgs a{};
    a.n = n_rot;
    a.tol = rot_tol(ctx);
    a.r32 = ctx->d_rot;
    a.status = ctx->d_status;
    if (dev_R) {
        a.R = R;
        a.r64 = ctx->d_rot64;
    } else {
        CU(ctx, cudaMemcpyAsync(ctx->d_rot64, R, sizeof(double) * 9 * n_rot, cudaMemcpyHostToDevice, s));
        a.R = ctx->d_rot64;
    }
    launch_rot_prep(a, s);
    ctx->launches++;
    CU(ctx, cudaGetLastError());
    return BC_OK;
}

bc_status ensure_query_ws(bc_ctx *ctx, int64_t chunk)
{
    if (ctx->q_cap >= chunk) return BC_OK;
    const int nblk = query_blocks((int)ctx->n[1]);
    TRY(dalloc(ctx, &ctx->d_qR, sizeof(double) * 9 * chunk));
    TRY(dalloc(ctx, &ctx->d_qt, sizeof(double) * 3 * chunk));
    TRY(dalloc(ctx, &ctx->d_qpart, sizeof(double) * 2 * nblk * chunk));
    TRY(dalloc(ctx, &ctx->d_qout, sizeof(double) * 2 * chunk));
    ctx->q_cap = chunk;
    return BC_OK;
}

// Exact pair-lens query of the nq configurations in ctx->d_qR / ctx->d_qt (query.cu).
bc_status run_query(bc_ctx *ctx, int nq, double *dst, cudaStream_t s)
{
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    QueryArgs qa{};
    qa.nq = nq;
    qa.nB = (int)ctx->n[1];
    qa.R = ctx->d_qR;
    qa.t = ctx->d_qt;
    qa.A = ctx->d_balls64[0];
    qa.B = ctx->d_balls64[1];
    qa.wA = ctx->d_w64[0];
    qa.wB = ctx->d_w64[1];
    qa.start = ctx->d_qstart;
    qa.idx = ctx->d_qidx;
    qa.nx = ctx->qn[0];
    qa.ny = ctx->qn[1];
    qa.nz = ctx->qn[2];
    qa.gx0 = ctx->qg0[0];
    qa.gy0 = ctx->qg0[1];
    qa.gz0 = ctx->qg0[2];
    qa.inv_cs = 1.0 / ctx->qcs;
    qa.partial = ctx->d_qpart;
    qa.out = dst;
    qa.complex_w = cplx;
    {
        StageScope sc(ctx, s, "evaluate_points");
        launch_query(qa, s);
        ctx->launches += 2;
    }
    CU(ctx, cudaGetLastError());
    return BC_OK;
}

// Exact mode's fixed-point scale (exact.cu): 2^61 / B with B = min(|A|_inf |B|_1, |A|_1 |B|_inf)
// >= max |f| (|f| <= |rho_A|_inf |rho_B|_1 and symmetrically; |rho|_inf <= sum |w|, |rho|_1 =
// sum |w| vol), so no partial sum can overflow int64.
bc_status exact_plan(bc_ctx *ctx)
{
    if (ctx->ex_ready) return BC_OK;
    double sAi = 0, sA1 = 0, sBi = 0, sB1 = 0;
    for (int w = 0; w < 2; w++)
        for (int64_t i = 0; i < ctx->n[w]; i++) {
            const double m = std::hypot(ctx->hw[w][2 * i], ctx->hw[w][2 * i + 1]), r = ctx->hxyzr[w][4 * i + 3];
            (w ? sBi : sAi) += m;
            (w ? sB1 : sA1) += m * 4.0 / 3.0 * kPi * r * r * r;
        }
    const double bound = std::min(sAi * sB1, sA1 * sBi);
    ctx->ex_qscale = bound > 0 ? std::ldexp(1.0, 61) / bound : 1.0;
    // kernel choice (measured, Tiny / Single): a thread per knot walking its ball (B by radius)
    // when there are enough knots to fill the GPU (>= 2^18) and footprints are small (mean box
    // <= 1000 points): Single 0.60 -> 0.45 ms; else a warp per knot (Tiny: 1,024 knots, 0.034 ms
    // vs 0.20 ms with a thread per knot)
    double mr = 0, ms = 0;
    for (int64_t i = 0; i < ctx->n[0]; i++) mr += ctx->hxyzr[0][4 * i + 3];
    for (int64_t j = 0; j < ctx->n[1]; j++) ms += ctx->hxyzr[1][4 * j + 3];
    mr /= std::max<int64_t>(ctx->n[0], 1);
    ms /= std::max<int64_t>(ctx->n[1], 1);
    const double side = 2 * (mr + ms) / ctx->p.h + 1;
    ctx->ex_thread_per_knot = side * side * side <= 1000.0 && (double)ctx->n[0] * ctx->n[1] >= 262144.0;
    // fp32 thread-per-knot with even N: packed pair accumulators, scale 2^30 / B' with the tight
    // bound B' = min(inf'_A |B|_1, |A|_1 inf'_B) >= sum |terms| at any point, where
    // inf'_S = max_i sum_{i' : |c_i - c_i'| < r_i + r_i'} |w_i'| >= |rho_S|_inf (a point of
    // density is inside some ball i, and every ball containing it meets ball i); O(n^2), so only
    // for n <= 16384
    ctx->ex_packed = false;
    if (ctx->p.precision == BC_FP32 && ctx->ex_thread_per_knot && ctx->p.N % 2 == 0 && ctx->n[0] <= 16384 &&
        ctx->n[1] <= 16384) {
        double inf[2] = {0, 0};
        for (int w = 0; w < 2; w++) {
            const std::vector<double> &x = ctx->hxyzr[w];
            for (int64_t i = 0; i < ctx->n[w]; i++) {
                double acc = 0;
                for (int64_t k = 0; k < ctx->n[w]; k++) {
                    const double dx = x[4 * i] - x[4 * k], dy = x[4 * i + 1] - x[4 * k + 1], dz = x[4 * i + 2] - x[4 * k + 2];
                    const double rr = x[4 * i + 3] + x[4 * k + 3];
                    if (dx * dx + dy * dy + dz * dz < rr * rr) acc += std::hypot(ctx->hw[w][2 * k], ctx->hw[w][2 * k + 1]);
                }
                inf[w] = std::max(inf[w], acc);
            }
        }
        const double tight = std::min(inf[0] * sB1, sA1 * inf[1]);
        if (tight > 0) {
            ctx->ex_packed = true;
            ctx->ex_qscale = std::ldexp(1.0, 30) / tight;
        }
    }
    std::vector<int> perm((size_t)std::max<int64_t>(ctx->n[1], 1), 0);
    for (int64_t j = 0; j < ctx->n[1]; j++) perm[j] = (int)j;
    std::stable_sort(perm.begin(), perm.begin() + ctx->n[1],
                     [&](int x, int y) { return ctx->hxyzr[1][4 * x + 3] < ctx->hxyzr[1][4 * y + 3]; });
    TRY(dalloc(ctx, &ctx->d_permB, sizeof(int) * perm.size()));
    CU(ctx, cudaMemcpy(ctx->d_permB, perm.data(), sizeof(int) * perm.size(), cudaMemcpyHostToDevice));
    ctx->ex_ready = true;
    return BC_OK;
}

// Retained modes of the spectral query for m' (query_spectral.cu): the band's modes |k_i| <= K
// sorted by (|k|^2, kx, ky, kz) -- the radial-shell ("spiral") order of PAPER.md L436 -- with a
// mode and its mirror kept together for real weights (half space kz > 0 | kz = 0, ky > 0 |
// kz = ky = 0, kx > 0, counted twice; k = 0 once).  The first modes whose multiplicities add up
// to at most m' are retained.  Built on the host once per (shapes, spectrum, larger m').
bc_status qs_prepare(bc_ctx *ctx, int64_t m_prime, cudaStream_t s)
{
    if (ctx->qs_ready && m_prime <= ctx->qs_m) return BC_OK;
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    const int K = ctx->K;
    // enumerate a ball |k| <= Rk (grown until it holds m' modes or the whole cube band)
    struct Mode {
        int k2, x, y, z;
    };
    std::vector<Mode> modes;
    double Rk = std::cbrt(3.0 * (double)m_prime / (4 * kPi)) + 2;
    for (;;) {
        modes.clear();
        const int lim = std::min(K, (int)std::ceil(Rk));
        const long long R2 = (long long)(Rk * Rk);
        for (int x = -lim; x <= lim; x++)
            for (int y = -lim; y <= lim; y++)
                for (int z = cplx ? -lim : 0; z <= lim; z++) {
                    const long long k2 = (long long)x * x + (long long)y * y + (long long)z * z;
                    if (k2 > R2) continue;
                    if (!cplx && (z == 0 && (y < 0 || (y == 0 && x < 0)))) continue;  // the mirror half
                    modes.push_back({(int)k2, x, y, z});
                }
        int64_t cnt = 0;
        for (const Mode &m : modes) cnt += (cplx || m.k2 == 0) ? 1 : 2;
        if (cnt >= m_prime || R2 >= 3LL * K * K) break;  // enough modes, or the whole cube band
        Rk *= 1.25;
    }
    std::sort(modes.begin(), modes.end(), [](const Mode &a, const Mode &b) {
        if (a.k2 != b.k2) return a.k2 < b.k2;
        if (a.x != b.x) return a.x < b.x;
        if (a.y != b.y) return a.y < b.y;
        return a.z < b.z;
    });
    std::vector<int4> hm;
    std::vector<float> hmult;
    std::vector<int> k2s;
    int64_t cnt = 0;
    for (const Mode &m : modes) {
        const int mu = (cplx || m.k2 == 0) ? 1 : 2;
        if (cnt + mu > m_prime) break;
        cnt += mu;
        if (k2s.empty() || k2s.back() != m.k2) k2s.push_back(m.k2);
        hm.push_back(make_int4(m.x, m.y, m.z, (int)k2s.size() - 1));
        hmult.push_back((float)mu);
    }
    ctx->qs_nm = (int)hm.size();
    ctx->qs_nsh = (int)k2s.size();
    ctx->qs_m = m_prime;  // serves every m' <= this (a real-weight pair may leave cnt = m' - 1)
    const int nB = (int)ctx->n[1];
    TRY(dalloc(ctx, &ctx->d_qs_modes, sizeof(int4) * hm.size()));
    TRY(dalloc(ctx, &ctx->d_qs_mult, sizeof(float) * hm.size()));
    TRY(dalloc(ctx, &ctx->d_qs_k2, sizeof(int) * k2s.size()));
    TRY(dalloc(ctx, &ctx->d_qs_Aq, sizeof(float2) * hm.size()));
    TRY(dalloc(ctx, &ctx->d_qs_bv, sizeof(float2) * (size_t)std::max(nB, 1) * k2s.size()));
    CU(ctx, cudaMemcpyAsync(ctx->d_qs_modes, hm.data(), sizeof(int4) * hm.size(), cudaMemcpyHostToDevice, s));
    CU(ctx, cudaMemcpyAsync(ctx->d_qs_mult, hmult.data(), sizeof(float) * hmult.size(), cudaMemcpyHostToDevice, s));
    CU(ctx, cudaMemcpyAsync(ctx->d_qs_k2, k2s.data(), sizeof(int) * k2s.size(), cudaMemcpyHostToDevice, s));
    QsTableArgs t{};
    t.B = ctx->d_balls64[1];
    t.wB = ctx->d_w64[1];
    t.nB = nB;
    t.k2 = ctx->d_qs_k2;
    t.nsh = ctx->qs_nsh;
    t.P = ctx->P;
    t.complex_w = cplx;
    t.bv = ctx->d_qs_bv;
    t.Ahat = ctx->d_Ahat;
    t.modes = ctx->d_qs_modes;
    t.nm = ctx->qs_nm;
    t.K = K;
    t.Kz = ctx->Kz;
    t.Aq = ctx->d_qs_Aq;
    launch_qs_tables(t, s);
    ctx->launches += 2;
    CU(ctx, cudaStreamSynchronize(s));  // host vectors above go out of scope (pageable copies)
    CU(ctx, cudaGetLastError());
    ctx->qs_ready = true;
    return BC_OK;
}

// ------------------------------------------------------------------ spectral fp64 parity mode

bc_status sp64_twiddles(bc_ctx *ctx, long long G, double2 **out)
{
    auto it = ctx->d_tw64.find(G);
    if (it != ctx->d_tw64.end()) {
        *out = it->second;
        return BC_OK;
    }
    std::vector<double2> t((size_t)G);
    for (long long r = 0; r < G; r++) {
        const double ang = -2 * kPi * (double)r / (double)G;
        t[r] = make_double2(std::cos(ang), std::sin(ang));
    }
    double2 *d = nullptr;
    CU(ctx, cudaMalloc(&d, sizeof(double2) * G));
    CU(ctx, cudaMemcpy(d, t.data(), sizeof(double2) * G, cudaMemcpyHostToDevice));
    ctx->d_tw64[G] = d;
    *out = d;
    return BC_OK;
}

// The band spectrum of shape `which` (rotated by the device matrix `rot` for B) into `band`
// [kx][ky][kz] (full band, each axis k in [-K, K]): spread, then z, y, x axis DFTs.
bc_status sp64_shape_spectrum(bc_ctx *ctx, int which, const double *rot, double2 *band, cudaStream_t s)
{
    const ShapePlan &pl = ctx->plan[which];
    const int L = pl.L, M = ctx->M, K = ctx->K;
    if (L > 160 || M > 129)
        return fail(ctx, BC_EUNSUPPORTED, "spectral fp64 is a parity mode: box L = %d (<= 160), band M = %d (<= 129)", L,
                    M);
    const size_t N = ctx->p.N;
    const size_t need = sizeof(double2) * std::max({(size_t)L * L * L, (size_t)L * L * M, N * M * M, N * N * M,
                                                    N * N * N});
    if (ctx->sp64_ws_bytes < need) {
        TRY(dalloc(ctx, &ctx->d_sp64_w1, need));
        TRY(dalloc(ctx, &ctx->d_sp64_w2, need));
        ctx->sp64_ws_bytes = need;
    }
    double2 *tw = nullptr;
    TRY(sp64_twiddles(ctx, pl.G, &tw));
    Sp64SpreadArgs sa{};
    sa.L = L;
    for (int a = 0; a < 3; a++) sa.o[a] = pl.o[a];
    sa.hf = pl.hf;
    sa.tau = pl.tau;
    sa.cut = pl.cut;
    sa.balls = ctx->d_balls64[which];
    sa.w = ctx->d_w64[which];
    sa.n = (int)ctx->n[which];
    sa.rot = rot;
    sa.out = ctx->d_sp64_w1;
    {
        StageScope sc(ctx, s, which ? "sp64_spread_B" : "sp64_spread_A");
        launch_sp64_spread(sa, s);
        ctx->launches++;
    }
    Sp64DftArgs d{};
    d.qlo = -K;
    d.nlo = 0;
    d.G = pl.G;
    d.sign = -1;
    d.tw = tw;
    d.mult = 1;
    d.hf = pl.hf;
    d.tau = pl.tau;
    d.P = ctx->P;
    d.origin = which == 0;
    d.nq = M;
    d.Lin = L;
    // z: box [ix][iy][iz] -> [ix][iy][kz]
    d.in = ctx->d_sp64_w1;
    d.out = ctx->d_sp64_w2;
    d.O = L * L;
    d.I = 1;
    d.off = pl.o[2];
    d.t0 = ctx->p.t0[2];
    launch_sp64_dft(d, s);
    // y: [ix][iy][kz] -> [ix][ky][kz]
    d.in = ctx->d_sp64_w2;
    d.out = ctx->d_sp64_w1;
    d.O = L;
    d.I = M;
    d.off = pl.o[1];
    d.t0 = ctx->p.t0[1];
    launch_sp64_dft(d, s);
    // x: [ix][ky][kz] -> band [kx][ky][kz]
    d.in = ctx->d_sp64_w1;
    d.out = band;
    d.O = 1;
    d.I = M * M;
    d.off = pl.o[0];
    d.t0 = ctx->p.t0[0];
    launch_sp64_dft(d, s);
    ctx->launches += 3;
    CU(ctx, cudaGetLastError());
    return BC_OK;
}

bc_status sp64_spectrum_A(bc_ctx *ctx, cudaStream_t s)
{
    const size_t M3 = (size_t)ctx->M * ctx->M * ctx->M;
    if (!ctx->d_A64) TRY(dalloc(ctx, &ctx->d_A64, sizeof(double2) * M3));
    if (ctx->n[0] == 0) {
        CU(ctx, cudaMemsetAsync(ctx->d_A64, 0, sizeof(double2) * M3, s));
        return BC_OK;
    }
    return sp64_shape_spectrum(ctx, 0, nullptr, ctx->d_A64, s);
}

// f for n_rot rotations (ctx->d_rot64), F_FULL only: B's band, G = A' B(-k), inverse x, y, z.
bc_status sp64_run_rotations(bc_ctx *ctx, int64_t n_rot, int out_kind, char *dout, size_t out_per, cudaStream_t s)
{
    if (out_kind != BC_OUT_F_FULL)
        return fail(ctx, BC_EUNSUPPORTED, "spectral fp64 (parity mode) returns the full field only");
    const int M = ctx->M, K = ctx->K, N = ctx->p.N, Np = ctx->p.Np;
    const size_t M3 = (size_t)M * M * M;
    if (!ctx->d_B64) TRY(dalloc(ctx, &ctx->d_B64, sizeof(double2) * M3));
    if (!ctx->d_G64) TRY(dalloc(ctx, &ctx->d_G64, sizeof(double2) * M3));
    double2 *twN = nullptr;
    TRY(sp64_twiddles(ctx, Np, &twN));
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    for (int64_t r = 0; r < n_rot; r++) {
        TRY(sp64_shape_spectrum(ctx, 1, ctx->d_rot64 + 9 * r, ctx->d_B64, s));
        launch_sp64_product(ctx->d_A64, ctx->d_B64, ctx->d_G64, M, s);
        Sp64DftArgs d{};
        d.qlo = 0;
        d.nlo = -K;
        d.G = Np;
        d.sign = +1;
        d.tw = twN;
        d.mult = 0;
        d.nq = N;
        d.Lin = M;
        // inverse x: [kx][ky][kz] -> [mx][ky][kz]   (workspaces hold N M M <= L L M doubles)
        d.in = ctx->d_G64;
        d.out = ctx->d_sp64_w1;
        d.O = 1;
        d.I = M * M;
        launch_sp64_dft(d, s);
        // inverse y: [mx][ky][kz] -> [mx][my][kz]
        d.in = ctx->d_sp64_w1;
        d.out = ctx->d_sp64_w2;
        d.O = N;
        d.I = M;
        launch_sp64_dft(d, s);
        // inverse z: [mx][my][kz] -> [mx][my][mz]
        d.in = ctx->d_sp64_w2;
        d.out = ctx->d_sp64_w1;
        d.O = N * N;
        d.I = 1;
        launch_sp64_dft(d, s);
        launch_sp64_output(ctx->d_sp64_w1, (long long)N * N * N, 1.0 / (ctx->P * ctx->P * ctx->P), cplx,
                           (double *)(dout + out_per * r), s);
        ctx->launches += 5;
        CU(ctx, cudaGetLastError());
    }
    return BC_OK;
}

// The per-rotation path for n_rot rotations already prepared in ctx->d_rot (fp32) and
// ctx->d_rot64 (fp64), written to the device buffer dout (out_per bytes per rotation).
bc_status run_rotations(bc_ctx *ctx, int64_t n_rot, int out_kind, char *dout, size_t out_per, cudaStream_t s)
{
    if (ctx->sp64) return sp64_run_rotations(ctx, n_rot, out_kind, dout, out_per, s);
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    const long long N = ctx->p.N, N3 = N * N * N;
    if (ctx->p.mode == BC_MODE_EXACT) {
        TRY(exact_plan(ctx));
        int nb = ctx->p.max_batch > 0 ? ctx->p.max_batch : 8;
        const size_t per = (size_t)N3 * (cplx ? 2 : 1) * sizeof(long long);
        while (nb > 1 && per * nb > ((size_t)4 << 30)) nb /= 2;
        nb = (int)std::min<int64_t>(nb, n_rot);
        if (ctx->acc_bytes < per * nb) {
            TRY(dalloc(ctx, &ctx->d_acc, per * nb));
            ctx->acc_bytes = per * nb;
        }
        if (ctx->part_cap < nb * 64 * 2) {
            TRY(dalloc(ctx, &ctx->d_part, sizeof(double) * nb * 64 * 2));
            TRY(dalloc(ctx, &ctx->d_part_idx, sizeof(long long) * nb * 64 * 2));
            ctx->part_cap = nb * 64 * 2;
        }
        for (int64_t r0 = 0; r0 < n_rot; r0 += nb) {
            const int b = (int)std::min<int64_t>(nb, n_rot - r0);
            CU(ctx, cudaMemsetAsync(ctx->d_acc, 0, per * b, s));
            ExactArgs a{};
            a.nA = (int)ctx->n[0];
            a.nB = (int)ctx->n[1];
            a.N = (int)N;
            a.h = ctx->p.h;
            a.inv_h = 1.0 / ctx->p.h;
            a.t0x = ctx->p.t0[0];
            a.t0y = ctx->p.t0[1];
            a.t0z = ctx->p.t0[2];
            a.A = ctx->d_balls64[0];
            a.B = ctx->d_balls64[1];
            a.wA = ctx->d_w64[0];
            a.wB = ctx->d_w64[1];
            a.rot = ctx->d_rot64 + 9 * r0;
            a.complex_w = cplx;
            a.fp64 = ctx->p.precision == BC_FP64;
            a.iacc = (long long *)ctx->d_acc;
            a.acc_bstride = (long long)(per / sizeof(long long));
            a.qscale = ctx->ex_qscale;
            a.thread_per_knot = ctx->ex_thread_per_knot ? 1 : 0;
            a.permB = ctx->d_permB;
            a.packed = ctx->ex_packed ? 1 : 0;
            {
                StageScope sc(ctx, s, "exact_pairs");
                launch_exact_scatter(a, b, s);
                ctx->launches++;
            }
            ExactOutArgs o{};
            o.N = (int)N;
            o.complex_w = cplx;
            o.fp64 = a.fp64;
            o.iacc = a.iacc;
            o.acc_bstride = a.acc_bstride;
            o.inv_qscale = 1.0 / ctx->ex_qscale;
            o.packed = a.packed;
            o.out_kind = out_kind;
            o.out = dout + out_per * r0;
            o.partials = ctx->d_part;
            o.partial_idx = ctx->d_part_idx;
            {
                StageScope sc(ctx, s, "exact_out");
                int nl = 0;
                launch_exact_out(o, b, s, &nl);
                ctx->launches += nl;
            }
            CU(ctx, cudaGetLastError());
        }
    } else {
        size_t s1, s2;
        spectral_ws_sizes(ctx, 1, s1, s2);
        int nb = ctx->p.max_batch > 0 ? ctx->p.max_batch : 16;
        while (nb > 1 && (s1 + s2) * nb > ((size_t)12 << 30)) nb /= 2;
        nb = (int)std::min<int64_t>(nb, n_rot);
        ctx->batch = nb;
        // concurrent batches (opt-in, concurrency = 2): two slots on internal streams forked
        // from / joined to `s`, so that blocks of different kernels (the spread of one batch,
        // the fold of the other) share the SMs.  Measured 3.6 % slower on the sweep (L1 / L2
        // contention), hence off by default.  Not while profiling (stage times would overlap).
        const int64_t n_batches = (n_rot + nb - 1) / nb;
        const int nslots = (!ctx->prof && n_batches > 1 && ctx->p.concurrency == 2) ? 2 : 1;
        for (int q = 0; q < nslots; q++) {
            Slot &sl = ctx->slot[q];
            TRY(ensure_ws(ctx, &sl.ws1, sl.ws1_bytes, s1 * nb));
            TRY(ensure_ws(ctx, &sl.ws2, sl.ws2_bytes, s2 * nb));
            if (sl.keys_cap < 2 * nb) {
                TRY(dalloc(ctx, &sl.keys, sizeof(unsigned long long) * 2 * nb));
                sl.keys_cap = 2 * nb;
            }
            if (nslots > 1 && !sl.stream) {
                CU(ctx, cudaStreamCreateWithFlags(&sl.stream, cudaStreamNonBlocking));
                CU(ctx, cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
            }
        }
        const int Np = ctx->p.Np;
        const ShapePlan &pB = ctx->plan[1];
        const bool fast_fold = !ctx->p.generic_only && fold_fast_supported(pB.L, pB.c, pB.G, ctx->K, Np, cplx);
        const bool dock_fold = use_dock_fast(ctx);
        const bool fused_inv = fast_fold || (!ctx->p.generic_only && !dock_fold && fold_fuses_inverse(pB.L, Np));
        // row pitch of X1 / Y1: padded to 8 modes on the fast plan (64-byte row pieces stay
        // 32-byte-sector aligned), the stored count elsewhere
        const int zpitch = fast_fold ? (ctx->Fz + 7) & ~7 : ctx->Fz;
        if (!ctx->cm_ready) {  // A' into the coset-major x order of B's plan (once per A / B plan)
            const ShapePlan &pb = ctx->plan[1];
            ctx->MS = cm_row_stride(pb.L, pb.c, pb.G, ctx->K);
            const size_t nspec = (size_t)ctx->MS * ctx->M * ctx->Kz;
            // grown only (a cudaFree would synchronise the device: the call stays asynchronous)
            if (ctx->Ahat_cm_bytes < sizeof(float2) * nspec) {
                TRY(dalloc(ctx, &ctx->d_Ahat_cm, sizeof(float2) * nspec));
                ctx->Ahat_cm_bytes = sizeof(float2) * nspec;
            }
            launch_permute_cm(ctx->d_Ahat, pb.d_mult[0], ctx->d_Ahat_cm, (long long)ctx->M * ctx->Kz, ctx->K, pb.L, pb.c,
                              pb.G, cplx, ctx->MS, ctx->Kz, ctx->p.band_radius, pb.blob ? ctx->d_dec : nullptr, s,
                              yz_in_A(ctx) ? pb.d_mult[1] : nullptr, yz_in_A(ctx) ? pb.d_mult[2] : nullptr);
            ctx->launches++;
            CU(ctx, cudaGetLastError());
            ctx->cm_ready = true;
        }
        if (nslots > 1) {  // fork: the slots' streams wait for the uploads / A'' on `s`
            if (!ctx->ev_fork) CU(ctx, cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
            CU(ctx, cudaEventRecord(ctx->ev_fork, s));
            for (int q = 0; q < nslots; q++) CU(ctx, cudaStreamWaitEvent(ctx->slot[q].stream, ctx->ev_fork, 0));
        }
        const cudaStream_t s_user = s;
        for (int64_t r0 = 0; r0 < n_rot; r0 += nb) {
            const int b = (int)std::min<int64_t>(nb, n_rot - r0);
            Slot &sl = ctx->slot[nslots > 1 ? (int)((r0 / nb) % nslots) : 0];
            const cudaStream_t s = nslots > 1 ? sl.stream : s_user;
            void *const ws1 = sl.ws1, *const ws2 = sl.ws2;
            unsigned long long *const keys = sl.keys;
            // 1-3: spread R B, z and y passes of its box DFT
            TRY(shape_spectrum(ctx, 1, ctx->d_rot + 9 * r0, b, ws1, ws2, s1, s2, s, sl));
            const ShapePlan &pb = ctx->plan[1];
            // 4: x pass fused with the spectral product (A' conj(RB)) and the fold onto Np^3
            if (dock_fold) {
                DockFoldArgs a{};
                a.tw = ctx->d_tw[pb.L];
                a.ctw = pb.d_ctw;
                a.T2 = (const float2 *)ws1;
                a.t2_bstride = (long long)(s1 / 8);
                a.Ahat = ctx->d_Ahat_cm;
                a.MS = ctx->MS;
                for (int p = 0; p < 2; p++) {
                    const CmSeg sg = cm_segment(p, pb.L, pb.c, pb.G, ctx->K);
                    a.pos_base[p] = sg.off - sg.qn;
                }
                a.F = (float2 *)ws2;
                a.f_bstride = (long long)(s2 / 8);
                a.cx = (float)(-pb.o[0]);
                a.live_r2 = (float)(ctx->live_r * ctx->live_r);
                StageScope sc(ctx, s, "fold_dk");
                if (!launch_fold_dk(a, b, s))
                    return fail(ctx, BC_EUNSUPPORTED, "fold_dk: A'' row stride MS = %d not the compiled plan's", a.MS);
                ctx->launches++;
            } else if (fast_fold) {
                FoldFastArgs a{};
                a.tw = ctx->d_tw[pb.L];
                a.ctw = pb.d_ctw;
                a.T2 = (const float2 *)ws1;
                a.t2_bstride = (long long)(s1 / 8);
                a.Ahat = ctx->d_Ahat_cm;
                a.MS = ctx->MS;
                for (int p = 0; p < 4; p++) {
                    const CmSeg sg = cm_segment(p, pb.L, pb.c, pb.G, ctx->K);
                    a.pos_base[p] = sg.off - sg.qn;
                }
                a.X1 = (float2 *)ws2;
                a.x1_bstride = (long long)(s2 / 8);
                a.x1_pitch = zpitch;
                a.N = (int)N;
                StageScope sc(ctx, s, "fold_fast");
                if (!launch_fold_fast(a, b, s))
                    return fail(ctx, BC_EUNSUPPORTED, "fold_fast: strides (MS = %d, X1 pitch = %d) not the compiled plan's",
                                a.MS, a.x1_pitch);
                ctx->launches++;
            } else {
                FoldXArgs a{};
                a.L = pb.L;
                a.c = pb.c;
                a.G = pb.G;
                a.K = ctx->K;
                a.M = ctx->M;
                a.Kz = ctx->Kz;
                a.Np = Np;
                a.Fz = ctx->Fz;
                a.complex_w = cplx;
                a.mult = nullptr;
                a.MS = ctx->MS;
                a.xtab = ctx->d_xtab;
                a.segs = ctx->d_segs;
                a.tw = ctx->d_tw[pb.L];
                a.ctw = pb.d_ctw;
                a.T2 = (const float2 *)ws1;
                a.t2_bstride = (long long)(s1 / 8);
                a.Ahat = ctx->d_Ahat_cm;
                a.F = (float2 *)ws2;  // F, or X1 when the inverse x pass is fused
                a.f_bstride = (long long)(s2 / 8);
                a.N = (int)N;
                a.fuse_inv = fused_inv;
                a.tw_inv = ctx->d_tw[Np];
                StageScope sc(ctx, s, fused_inv ? "fold_x_inv" : "fold_x");
                launch_fold_x(a, b, s);
                ctx->launches++;
            }
            // 5-6: inverse transforms along x and y (only the N output rows)
            PassArgs inv{};
            inv.L = Np;
            inv.c = 1;
            inv.G = Np;
            inv.klo = 0;
            inv.nk = (int)N;
            inv.signed_k = 0;
            inv.tw = ctx->d_tw[Np];
            // X1 lives in ws1 after a separate inverse x pass, in ws2 when it is fused
            if (!fused_inv) {
                PassArgs a = inv;
                a.O = 1;
                a.I = Np * ctx->Fz;
                a.in = ws2;
                a.in_bstride = (long long)(s2 / 8);
                a.out = (float2 *)ws1;
                a.out_bstride = (long long)(s1 / 8);
                StageScope sc(ctx, s, "inv_x");
                launch_pass(a, 3, b, s);
                ctx->launches++;
            }
            void *y1 = fused_inv ? ws1 : ws2;
            const long long y1_bstride = (long long)((fused_inv ? s1 : s2) / 8);
            {
                PassArgs a = inv;
                a.O = (int)N;
                a.I = ctx->Fz;
                a.in = fused_inv ? ws2 : ws1;
                a.in_bstride = (long long)((fused_inv ? s2 : s1) / 8);
                a.out = (float2 *)y1;
                a.out_bstride = y1_bstride;
                a.pitch_in = a.pitch_out = zpitch;
                StageScope sc(ctx, s, "inv_y");
                launch_pass(a, 3, b, s);
                ctx->launches++;
            }
            // 8: inverse along z (C2R / C2C), 1/P^3, full output or reduction keys
            if (out_kind != BC_OUT_F_FULL) {
                launch_keys_init(keys, 2 * b, s);
                ctx->launches++;
            }
            {
                LastArgs a{};
                a.Np = Np;
                a.N = (int)N;
                a.Fz = ctx->Fz;
                a.hermitian = !cplx;
                a.scale = (float)(1.0 / (ctx->P * ctx->P * ctx->P));
                a.tw = ctx->d_tw[Np];
                a.in = (const float2 *)y1;
                a.in_bstride = y1_bstride;
                a.pitch = zpitch;
                a.out_kind = out_kind;
                a.out_full = dout + out_per * r0;
                a.full_bstride = N3;
                a.keys = keys;
                StageScope sc(ctx, s, "inv_z_reduce");
                launch_last(a, b, s);
                ctx->launches++;
            }
            if (out_kind != BC_OUT_F_FULL) {
                StageScope sc(ctx, s, "finalize");
                ResultPeers rp = ctx->res_peers;
                rp.base += r0;
                launch_keys_finalize(keys, b, out_kind, dout + out_per * r0, rp, s);
                ctx->launches++;
            }
            CU(ctx, cudaGetLastError());
        }
        if (nslots > 1) {  // join
            for (int q = 0; q < nslots; q++) {
                CU(ctx, cudaEventRecord(ctx->slot[q].done, ctx->slot[q].stream));
                CU(ctx, cudaStreamWaitEvent(s_user, ctx->slot[q].done, 0));
            }
        }
    }
    return BC_OK;
}

size_t out_elem_bytes(const bc_ctx *ctx, int kind)
{
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    const bool f64 = ctx->p.precision == BC_FP64;
    if (kind == BC_OUT_F_FULL) {
        const size_t N3 = (size_t)ctx->p.N * ctx->p.N * ctx->p.N;
        return N3 * (f64 ? 8 : 4) * (cplx ? 2 : 1);
    }
    return sizeof(bc_extremum) * (kind == BC_OUT_MINMAX ? 2 : 1);
}

// Band-error guard (bc_params.tolerance > 0, spectral mode).  The spectral result is the
// band-limited f (include/ballcorr.h); how far it is from the exact f depends on the shapes
// (few or small balls need a wider band).  Once per pair of uploaded shapes,
// before the first correlation, the library correlates two probe rotations (the identity
// and a fixed generic one) on the full grid, evaluates the EXACT f (query.cu, fp64
// pair-lens sum) at a 12^3 block of translations around each probe's max|f| and at 2,048
// pseudo-random translations, and estimates the relative error max|f_spec - f_exact| /
// max|f_exact| over those samples.  Above the tolerance: BC_ERANGE (raise K).  The estimate
// is a sampled lower bound of the true grid maximum, kept by bc_query("band_error").
// Synchronous (setup-time work).
bc_status band_probe(bc_ctx *ctx, cudaStream_t s)
{
    if (ctx->p.mode != BC_MODE_SPECTRAL || !(ctx->p.tolerance > 0) || ctx->probe_done) return BC_OK;
    if (ctx->n[0] == 0 || ctx->n[1] == 0) {
        ctx->probe_done = true;
        ctx->probe_err = 0.0;
        return BC_OK;
    }
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    const int64_t N = ctx->p.N, N3 = N * N * N;
    double Rp[18] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    {  // unit quaternion (w, x, y, z) ~ (0.8, 0.2, -0.4, 0.4), normalised
        double q[4] = {0.8, 0.2, -0.4, 0.4}, nq = 0;
        for (double v : q) nq += v * v;
        nq = std::sqrt(nq);
        for (double &v : q) v /= nq;
        const double w = q[0], x = q[1], y = q[2], z = q[3];
        const double m[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
                             2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
                             2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)};
        for (int i = 0; i < 9; i++) Rp[9 + i] = m[i];
    }
    TRY(prepare_rotations(ctx, Rp, false, 2, s));
    const size_t out_per = out_elem_bytes(ctx, BC_OUT_F_FULL);
    void *d = nullptr;
    CU(ctx, cudaMalloc(&d, out_per * 2));
    bc_status st = run_rotations(ctx, 2, BC_OUT_F_FULL, (char *)d, out_per, s);
    std::vector<float> f(out_per * 2 / sizeof(float));
    if (st == BC_OK) {
        cudaError_t e = cudaMemcpyAsync(f.data(), d, out_per * 2, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = fail(ctx, BC_ECUDA, "band probe: %s", cudaGetErrorString(e));
    }
    cudaFree(d);
    if (st != BC_OK) return st;
    if (!ctx->qgrid_ready) TRY(build_query_grid(ctx));
    const int cw = cplx ? 2 : 1;
    double err = 0.0, scale = 0.0;
    for (int r = 0; r < 2; r++) {
        const float *fr = f.data() + (size_t)r * N3 * cw;
        int64_t am = 0;
        double best = -1;
        for (int64_t i = 0; i < N3; i++) {
            const double v = cplx ? std::hypot((double)fr[2 * i], (double)fr[2 * i + 1]) : std::fabs((double)fr[i]);
            if (v > best) {
                best = v;
                am = i;
            }
        }
        std::vector<int64_t> idx;
        const int64_t ax = am / (N * N), ay = (am / N) % N, az = am % N;
        const int64_t B = std::min<int64_t>(12, N);
        auto lo = [&](int64_t c) { return std::min(std::max<int64_t>(c - B / 2, 0), N - B); };
        for (int64_t i = lo(ax); i < lo(ax) + B; i++)
            for (int64_t j = lo(ay); j < lo(ay) + B; j++)
                for (int64_t k = lo(az); k < lo(az) + B; k++) idx.push_back((i * N + j) * N + k);
        uint64_t x = 0x9e3779b97f4a7c15ull + (uint64_t)r;
        for (int q = 0; q < 2048; q++) {  // splitmix64
            x += 0x9e3779b97f4a7c15ull;
            uint64_t z = x;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            z ^= z >> 31;
            idx.push_back((int64_t)(z % (uint64_t)N3));
        }
        const int64_t nq = (int64_t)idx.size();
        TRY(ensure_query_ws(ctx, nq));
        std::vector<double> hR((size_t)9 * nq), ht((size_t)3 * nq), ex((size_t)2 * nq);
        for (int64_t q = 0; q < nq; q++) {
            for (int i = 0; i < 9; i++) hR[9 * q + i] = Rp[9 * r + i];
            const int64_t m[3] = {idx[q] / (N * N), (idx[q] / N) % N, idx[q] % N};
            for (int a = 0; a < 3; a++) ht[3 * q + a] = ctx->p.t0[a] + (double)m[a] * ctx->p.h;
        }
        CU(ctx, cudaMemcpyAsync(ctx->d_qR, hR.data(), sizeof(double) * hR.size(), cudaMemcpyHostToDevice, s));
        CU(ctx, cudaMemcpyAsync(ctx->d_qt, ht.data(), sizeof(double) * ht.size(), cudaMemcpyHostToDevice, s));
        TRY(run_query(ctx, (int)nq, ctx->d_qout, s));
        CU(ctx, cudaMemcpyAsync(ex.data(), ctx->d_qout, sizeof(double) * cw * nq, cudaMemcpyDeviceToHost, s));
        CU(ctx, cudaStreamSynchronize(s));
        for (int64_t q = 0; q < nq; q++) {
            const int64_t i = idx[q];
            double dv, sv;
            if (cplx) {
                dv = std::hypot((double)fr[2 * i] - ex[2 * q], (double)fr[2 * i + 1] - ex[2 * q + 1]);
                sv = std::hypot(ex[2 * q], ex[2 * q + 1]);
            } else {
                dv = std::fabs((double)fr[i] - ex[q]);
                sv = std::fabs(ex[q]);
            }
            err = std::max(err, dv);
            scale = std::max(scale, sv);
        }
    }
    ctx->probe_done = true;
    ctx->probe_err = scale > 0 ? err / scale : 0.0;
    if (ctx->probe_err > ctx->p.tolerance)
        return fail(ctx, BC_ERANGE,
                    "band K=%d too narrow for these shapes: estimated max relative error %.3g > tolerance %.3g "
                    "(probe rotations vs the exact pair-lens sum; raise K)",
                    ctx->K, ctx->probe_err, ctx->p.tolerance);
    return BC_OK;
}


}  // namespace

// ============================================================================ public API

extern "C" {

const char *bc_status_string(int st)
{
    switch (st) {
    case BC_OK: return "BC_OK";
    case BC_EINVAL: return "BC_EINVAL";
    case BC_ERANGE: return "BC_ERANGE";
    case BC_ENOMEM: return "BC_ENOMEM";
    case BC_ESTATE: return "BC_ESTATE";
    case BC_EUNSUPPORTED: return "BC_EUNSUPPORTED";
    case BC_ECUDA: return "BC_ECUDA";
    default: return "BC_UNKNOWN";
    }
}

const char *bc_last_error(const bc_ctx *ctx)
{
    if (!ctx) return "no context";
    return ctx->err.c_str();
}

bc_status bc_create(int device, const bc_params *p, bc_ctx **out)
{
    if (!p || !out) return BC_EINVAL;
    *out = nullptr;
    if (p->N < 1 || !(p->h > 0) || !std::isfinite(p->h)) return BC_EINVAL;
    for (int a = 0; a < 3; a++)
        if (!std::isfinite(p->t0[a])) return BC_EINVAL;
    if (p->mode != BC_MODE_SPECTRAL && p->mode != BC_MODE_EXACT) return BC_EINVAL;
    if (p->precision != BC_FP32 && p->precision != BC_FP64) return BC_EINVAL;
    if (p->weights != BC_WEIGHTS_REAL && p->weights != BC_WEIGHTS_COMPLEX) return BC_EINVAL;
    if (p->max_batch < 0) return BC_EINVAL;
    if (p->concurrency < 0 || p->concurrency > 2) return BC_EINVAL;
    if (!(p->tolerance >= 0) || !std::isfinite(p->tolerance)) return BC_EINVAL;
    if (p->mode == BC_MODE_SPECTRAL && p->precision == BC_FP64 && p->tolerance > 0) return BC_EUNSUPPORTED;
    if (p->mode == BC_MODE_SPECTRAL) {
        // fp64: the parity mode of spectral64.cu (small problems, F_FULL output)
        if (p->precision == BC_FP64 && (p->K > 64 || p->Np > 256)) return BC_EUNSUPPORTED;
        if (p->Np < p->N || p->Np < 2 || (p->Np % 2) != 0 || !friendly(p->Np) || p->Np > 1024) return BC_EINVAL;
        if (p->K < 1 || p->K > 2047) return BC_EINVAL;
        if (!(p->band_radius >= 0) || !std::isfinite(p->band_radius)) return BC_EINVAL;
        if (p->precision != BC_FP64 && !fft_size_supported(p->Np)) return BC_EUNSUPPORTED;  // fp64: direct DFTs
        if (p->N > 1625) return BC_EUNSUPPORTED;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return BC_ECUDA;
    }
    if (cudaSetDevice(device) != cudaSuccess) return BC_ECUDA;
    bc_ctx *ctx = new bc_ctx();
    ctx->device = device;
    ctx->p = *p;
    if (p->mode == BC_MODE_SPECTRAL) {
        const bool cplx = p->weights == BC_WEIGHTS_COMPLEX;
        ctx->P = p->Np * p->h;
        ctx->K = p->K;
        ctx->M = 2 * p->K + 1;
        ctx->Kz = cplx ? ctx->M : p->K + 1;
        ctx->Fz = cplx ? p->Np : p->Np / 2 + 1;
        ctx->sp64 = p->precision == BC_FP64;
        if (ensure_twiddles(ctx, p->Np) != BC_OK) {
            bc_destroy(ctx);
            return BC_ENOMEM;
        }
    }
    *out = ctx;
    return BC_OK;
}

bc_status bc_destroy(bc_ctx *ctx)
{
    if (!ctx) return BC_OK;
    cudaSetDevice(ctx->device);
    for (int w = 0; w < 2; w++) {
        dfree(ctx->d_balls[w]);
        dfree(ctx->d_wre[w]);
        dfree(ctx->d_wim[w]);
        dfree(ctx->d_balls64[w]);
        dfree(ctx->d_w64[w]);
        for (int a = 0; a < 3; a++) dfree(ctx->plan[w].d_mult[a]);
        dfree(ctx->plan[w].d_ctw);
    }
    for (auto &kv : ctx->d_tw) cudaFree(kv.second);
    dfree(ctx->d_csr_off);
    dfree(ctx->d_csr_idx);
    dfree(ctx->d_prof);
    dfree(ctx->d_prof_off);
    dfree(ctx->d_bcells);
    dfree(ctx->d_g02);
    dfree(ctx->d_phi);
    dfree(ctx->d_dec);
    dfree(ctx->d_recB);
    dfree(ctx->d_recWi);
    dfree(ctx->d_recBim);
    for (Slot &sl : ctx->slot) {
        if (sl.ws1) cudaFree(sl.ws1);
        if (sl.ws2) cudaFree(sl.ws2);
        dfree(sl.keys);
        dfree(sl.recA);
        dfree(sl.szcnt);
        dfree(sl.szoff);
        dfree(sl.szlist);
        if (sl.stream) cudaStreamDestroy(sl.stream);
        if (sl.done) cudaEventDestroy(sl.done);
    }
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    dfree(ctx->d_A64);
    dfree(ctx->d_B64);
    dfree(ctx->d_G64);
    dfree(ctx->d_sp64_w1);
    dfree(ctx->d_sp64_w2);
    for (auto &kv : ctx->d_tw64) cudaFree(kv.second);
    dfree(ctx->d_qs_modes);
    dfree(ctx->d_qs_k2);
    dfree(ctx->d_qs_mult);
    dfree(ctx->d_qs_Aq);
    dfree(ctx->d_qs_bv);
    dfree(ctx->d_qs_part);
    dfree(ctx->d_qs_mpart);
    dfree(ctx->d_qstart);
    dfree(ctx->d_qidx);
    dfree(ctx->d_qR);
    dfree(ctx->d_qt);
    dfree(ctx->d_qpart);
    dfree(ctx->d_qout);
    dfree(ctx->d_Ahat);
    dfree(ctx->d_Ahat_cm);
    dfree(ctx->d_Ahat_part);
    dfree(ctx->d_res);
    dfree(ctx->d_xtab);
    dfree(ctx->d_segs);

    dfree(ctx->d_rot);
    dfree(ctx->d_rot64);
    if (ctx->d_out_stage) cudaFree(ctx->d_out_stage);
    dfree(ctx->d_acc);
    dfree(ctx->d_permB);
    dfree(ctx->d_part);
    dfree(ctx->d_part_idx);
    for (auto &pe : ctx->pending) {
        cudaEventDestroy(pe.e0);
        cudaEventDestroy(pe.e1);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->h_status) cudaFreeHost(ctx->h_status);
    delete ctx;
    return BC_OK;
}

bc_status bc_shape_upload(bc_ctx *ctx, int which, const double *xyzr, const double *w, int64_t n)
{
    if (!ctx) return BC_EINVAL;
    TRY(check_deferred(ctx));
    if (which != 0 && which != 1) return fail(ctx, BC_EINVAL, "which must be 0 (A) or 1 (B)");
    if (n < 0 || (n > 0 && !xyzr)) return fail(ctx, BC_EINVAL, "bad shape size or NULL xyzr");
    if (n > (1ll << 30)) return fail(ctx, BC_EINVAL, "too many balls");
    CU(ctx, cudaSetDevice(ctx->device));
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    std::vector<double> x, wv;
    TRY(fetch_host(ctx, xyzr, (size_t)n * 4, x));
    if (w) TRY(fetch_host(ctx, w, (size_t)n * (cplx ? 2 : 1), wv));
    for (int64_t i = 0; i < n; i++) {
        for (int q = 0; q < 4; q++)
            if (!std::isfinite(x[4 * i + q])) return fail(ctx, BC_EINVAL, "ball %lld has a non-finite entry", (long long)i);
        if (!(x[4 * i + 3] > 0)) return fail(ctx, BC_EINVAL, "ball %lld has radius <= 0", (long long)i);
    }
    for (double v : wv)
        if (!std::isfinite(v)) return fail(ctx, BC_EINVAL, "non-finite weight");
    ctx->hxyzr[which] = x;
    ctx->hw[which].assign((size_t)n * 2, 0.0);
    for (int64_t i = 0; i < n; i++) {
        if (!w) {
            ctx->hw[which][2 * i] = 1.0;
        } else if (cplx) {
            ctx->hw[which][2 * i] = wv[2 * i];
            ctx->hw[which][2 * i + 1] = wv[2 * i + 1];
        } else {
            ctx->hw[which][2 * i] = wv[i];
        }
    }
    ctx->n[which] = n;
    ctx->have[which] = true;
    ctx->qgrid_ready = false;
    ctx->probe_done = false;
    ctx->probe_err = -1.0;
    ctx->ex_ready = false;
    ctx->qs_ready = false;
    if (which == 0) ctx->have_spec = false;
    ctx->cm_ready = false;
    TRY(upload_shape_device(ctx, which));
    if (ctx->p.mode == BC_MODE_SPECTRAL && n > 0) {
        double lo[3], hi[3], rmax, rho;
        shape_bounds(ctx, which, lo, hi, rmax, rho);
        if (which == 1)
            for (int a = 0; a < 3; a++) {  // any rotation keeps B inside the ball of radius max|b_j|
                lo[a] = -rho;
                hi[a] = rho;
            }
        TRY(plan_shape(ctx, which, lo, hi, rmax));
        if (which == 0) TRY(build_csr_A(ctx));
        if (which == 1 && !ctx->plan[1].blob) TRY(build_profiles_B(ctx));
        if (which == 1) {
            const ShapePlan &pb = ctx->plan[1];
            ctx->live_r = (rho + rmax + pb.cut) / pb.hf + 2.0;
            ctx->spread_cells_B = 0;
            for (int64_t j = 0; j < n; j++) {
                const double rc = (ctx->hxyzr[1][4 * j + 3] + pb.cut) / pb.hf;
                ctx->spread_cells_B += 4.0 / 3.0 * kPi * rc * rc * rc;
            }
            ctx->live_tiles_B = 0;  // same test as spread_z_kernel's zero-tile exit
            for (int X0 = 0; X0 < pb.L; X0 += 4)
                for (int Y0 = 0; Y0 < pb.L; Y0 += 4) {
                    const double cx = -pb.o[0], cy = -pb.o[1];
                    const double dx = std::max(std::max(X0 - cx, cx - (X0 + 3)), 0.0);
                    const double dy = std::max(std::max(Y0 - cy, cy - (Y0 + 3)), 0.0);
                    if (dx * dx + dy * dy <= (ctx->live_r + 1) * (ctx->live_r + 1)) ctx->live_tiles_B++;
                }
            if (ctx->plan[1].blob) TRY(build_spread_z_tables(ctx));
            else TRY(build_generic_bins_B(ctx));
        }
    }
    TRY(check_support(ctx));
    return BC_OK;
}

bc_status bc_spectrum_A(bc_ctx *ctx, void *stream)
{
    if (!ctx) return BC_EINVAL;
    TRY(check_deferred(ctx));
    if (!ctx->have[0]) return fail(ctx, BC_ESTATE, "shape A has not been uploaded");
    if (ctx->p.mode != BC_MODE_SPECTRAL || ctx->have_spec) {
        ctx->have_spec = true;
        return BC_OK;
    }
    CU(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t nspec = (size_t)ctx->M * ctx->M * ctx->Kz;
    if (!ctx->d_Ahat) TRY(dalloc(ctx, &ctx->d_Ahat, sizeof(float2) * nspec));  // fixed size per context
    ctx->cm_ready = false;
    ctx->probe_done = false;
    ctx->qs_ready = false;
    if (ctx->n[0] == 0) {
        CU(ctx, cudaMemsetAsync(ctx->d_Ahat, 0, sizeof(float2) * nspec, s));
        ctx->have_spec = true;
        return BC_OK;
    }
    if (ctx->sp64) {
        TRY(sp64_spectrum_A(ctx, s));
        ctx->have_spec = true;
        return BC_OK;
    }
    if (ctx->csr_lo != 0 || ctx->csr_hi >= 0) TRY(build_csr_A(ctx));  // after a partial spectrum
    // A's spread / z / y passes run in the context's batch workspaces (slot 0; kept, grown
    // when A's plan needs more): no allocation and no synchronisation per call
    size_t s1, s2;
    spectral_ws_sizes(ctx, 0, s1, s2);
    Slot &sl = ctx->slot[0];
    TRY(ensure_ws(ctx, &sl.ws1, sl.ws1_bytes, s1));
    TRY(ensure_ws(ctx, &sl.ws2, sl.ws2_bytes, s2));
    TRY(shape_spectrum(ctx, 0, nullptr, 1, sl.ws1, sl.ws2, s1, s2, s, sl));
    if (ctx->prof) collect_profile(ctx);
    ctx->have_spec = true;
    return BC_OK;
}

bc_status bc_spectrum_A_buffer(bc_ctx *ctx, void **dev_ptr, int64_t *bytes)
{
    if (!ctx) return BC_EINVAL;
    if (ctx->sp64) return fail(ctx, BC_EUNSUPPORTED, "the fp64 spectral parity mode keeps its spectrum private");
    if (!dev_ptr || !bytes) return fail(ctx, BC_EINVAL, "NULL dev_ptr/bytes");
    if (ctx->p.mode != BC_MODE_SPECTRAL) return fail(ctx, BC_EUNSUPPORTED, "exact mode has no spectrum of A");
    CU(ctx, cudaSetDevice(ctx->device));
    const size_t nspec = (size_t)ctx->M * ctx->M * ctx->Kz;
    if (!ctx->d_Ahat) TRY(dalloc(ctx, &ctx->d_Ahat, sizeof(float2) * nspec));
    *dev_ptr = ctx->d_Ahat;
    *bytes = (int64_t)(sizeof(float2) * nspec);
    return BC_OK;
}

bc_status bc_spectrum_A_import(bc_ctx *ctx)
{
    if (!ctx) return BC_EINVAL;
    if (ctx->sp64) return fail(ctx, BC_EUNSUPPORTED, "the fp64 spectral parity mode keeps its spectrum private");
    if (ctx->p.mode != BC_MODE_SPECTRAL) return fail(ctx, BC_EUNSUPPORTED, "exact mode has no spectrum of A");
    if (!ctx->have[0]) return fail(ctx, BC_ESTATE, "shape A has not been uploaded");
    if (!ctx->d_Ahat) return fail(ctx, BC_ESTATE, "bc_spectrum_A_buffer has not been called");
    ctx->cm_ready = false;  // A'' (coset-major, B's multipliers) is rebuilt from the new contents
    ctx->probe_done = false;
    ctx->qs_ready = false;
    ctx->have_spec = true;
    return BC_OK;
}

bc_status bc_correlate_rotations(bc_ctx *ctx, const double *R, int64_t n_rot, int out_kind, void *out, void *stream)
{
    if (!ctx) return BC_EINVAL;
    TRY(check_deferred(ctx));
    if (!R || !out || n_rot < 1) return fail(ctx, BC_EINVAL, "NULL R/out or n_rot < 1");
    if (out_kind < BC_OUT_F_FULL || out_kind > BC_OUT_MAX_REAL) return fail(ctx, BC_EINVAL, "bad out_kind");
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    if (cplx && out_kind != BC_OUT_F_FULL && out_kind != BC_OUT_MAX_REAL)
        return fail(ctx, BC_EINVAL, "complex weights support F_FULL and MAX_REAL only");
    if (!ctx->have[0] || !ctx->have[1]) return fail(ctx, BC_ESTATE, "upload both shapes first");
    if (ctx->p.mode == BC_MODE_SPECTRAL && !ctx->have_spec && ctx->n[0] > 0 && ctx->n[1] > 0)
        return fail(ctx, BC_ESTATE, "call bc_spectrum_A first");
    CU(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    const bool dev_R = is_device_ptr(R);
    if (!dev_R) TRY(validate_rotations(ctx, R, n_rot));  // host R: immediate BC_EINVAL
    // band-error guard (bc_params.tolerance): once per pair of uploaded shapes
    TRY(band_probe(ctx, s));

    const size_t out_per = out_elem_bytes(ctx, out_kind);
    const bool host_out = !is_device_ptr(out);
    char *dout = (char *)out;
    if (host_out) {
        TRY(ensure_ws(ctx, &ctx->d_out_stage, ctx->out_stage_bytes, out_per * n_rot));
        dout = (char *)ctx->d_out_stage;
    }
    TRY(prepare_rotations(ctx, R, dev_R, n_rot, s));

    if (ctx->n[0] == 0 || ctx->n[1] == 0) {
        // empty shape: f == 0 identically; a bc_extremum {0.0, 0} is all-zero bytes too
        CU(ctx, cudaMemsetAsync(dout, 0, out_per * n_rot, s));
    } else {
        TRY(run_rotations(ctx, n_rot, out_kind, dout, out_per, s));
    }
    if (host_out) {
        CU(ctx, cudaMemcpyAsync(out, dout, out_per * n_rot, cudaMemcpyDeviceToHost, s));
        CU(ctx, cudaStreamSynchronize(s));
        TRY(check_deferred(ctx));
    }
    if (ctx->prof) collect_profile(ctx);
    return BC_OK;
}

bc_status bc_evaluate_points(bc_ctx *ctx, const double *R, const double *t, int64_t n, double *out, void *stream)
{
    if (!ctx) return BC_EINVAL;
    TRY(check_deferred(ctx));
    if (!R || !t || !out || n < 1) return fail(ctx, BC_EINVAL, "NULL R/t/out or n < 1");
    if (!ctx->have[0] || !ctx->have[1]) return fail(ctx, BC_ESTATE, "upload both shapes first");
    CU(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    const bool dev_R = is_device_ptr(R), dev_t = is_device_ptr(t);
    if (!dev_R) TRY(validate_rotations(ctx, R, n));
    if (!dev_t)
        for (int64_t q = 0; q < 3 * n; q++)
            if (!std::isfinite(t[q])) return fail(ctx, BC_EINVAL, "non-finite translation");
    TRY(ensure_deferred_status(ctx));
    const size_t out_per = cplx ? 2 : 1;
    const bool host_out = !is_device_ptr(out);
    if (ctx->n[0] == 0 || ctx->n[1] == 0) {
        if (host_out)
            std::fill(out, out + out_per * n, 0.0);
        else
            CU(ctx, cudaMemsetAsync(out, 0, sizeof(double) * out_per * n, s));
        return BC_OK;
    }
    if (!ctx->qgrid_ready) TRY(build_query_grid(ctx));
    const int64_t chunk = std::min<int64_t>(n, 65535);
    TRY(ensure_query_ws(ctx, chunk));
    for (int64_t q0 = 0; q0 < n; q0 += chunk) {
        const int nq = (int)std::min<int64_t>(chunk, n - q0);
        // R and t into the query buffers: host arrays are copied (validated above), device
        // arrays are validated and copied on the device (deferred BC_EINVAL, no host round trip)
        RotPrepArgs ra{};
        ra.R = dev_R ? R + 9 * q0 : ctx->d_qR;
        ra.t = dev_t ? t + 3 * q0 : nullptr;
        ra.n = nq;
        ra.index_base = q0;
        ra.tol = rot_tol(ctx);
        ra.r64 = dev_R ? ctx->d_qR : nullptr;
        ra.t64 = dev_t ? ctx->d_qt : nullptr;
        ra.status = ctx->d_status;
        if (!dev_R) CU(ctx, cudaMemcpyAsync(ctx->d_qR, R + 9 * q0, sizeof(double) * 9 * nq, cudaMemcpyHostToDevice, s));
        if (!dev_t) CU(ctx, cudaMemcpyAsync(ctx->d_qt, t + 3 * q0, sizeof(double) * 3 * nq, cudaMemcpyHostToDevice, s));
        if (dev_R || dev_t) {
            launch_rot_prep(ra, s);
            ctx->launches++;
        }
        double *dst = host_out ? ctx->d_qout : out + out_per * q0;
        TRY(run_query(ctx, nq, dst, s));
        if (host_out) {
            CU(ctx, cudaMemcpyAsync(out + out_per * q0, ctx->d_qout, sizeof(double) * out_per * nq, cudaMemcpyDeviceToHost, s));
            CU(ctx, cudaStreamSynchronize(s));
        }
    }
    if (host_out) TRY(check_deferred(ctx));
    return BC_OK;
}

bc_status bc_evaluate_points_spectral(bc_ctx *ctx, const double *R, const double *t, int64_t n, int64_t m_prime,
                                      double *out, void *stream)
{
    if (!ctx) return BC_EINVAL;
    TRY(check_deferred(ctx));
    if (!R || !t || !out || n < 1) return fail(ctx, BC_EINVAL, "NULL R/t/out or n < 1");
    if (ctx->p.mode != BC_MODE_SPECTRAL || ctx->sp64)
        return fail(ctx, BC_EUNSUPPORTED, "the spectral query needs spectral mode in fp32");
    if (!ctx->have[0] || !ctx->have[1]) return fail(ctx, BC_ESTATE, "upload both shapes first");
    if (!ctx->have_spec) return fail(ctx, BC_ESTATE, "call bc_spectrum_A first");
    const int64_t band = (int64_t)ctx->M * ctx->M * ctx->M;
    if (m_prime < 1 || m_prime > std::min<int64_t>(band, (int64_t)1 << 22))
        return fail(ctx, BC_ERANGE, "m' = %lld outside [1, min(band modes %lld, 2^22)]", (long long)m_prime,
                    (long long)band);
    CU(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    const bool dev_R = is_device_ptr(R), dev_t = is_device_ptr(t);
    if (!dev_R) TRY(validate_rotations(ctx, R, n));
    if (!dev_t)
        for (int64_t q = 0; q < 3 * n; q++)
            if (!std::isfinite(t[q])) return fail(ctx, BC_EINVAL, "non-finite translation");
    TRY(ensure_deferred_status(ctx));
    const size_t out_per = cplx ? 2 : 1;
    const bool host_out = !is_device_ptr(out);
    if (ctx->n[0] == 0 || ctx->n[1] == 0) {
        if (host_out)
            std::fill(out, out + out_per * n, 0.0);
        else
            CU(ctx, cudaMemsetAsync(out, 0, sizeof(double) * out_per * n, s));
        return BC_OK;
    }
    TRY(qs_prepare(ctx, m_prime, s));
    // the retained modes for THIS m' (a prefix of the prepared list)
    QsArgs a{};
    a.nB = (int)ctx->n[1];
    {
        // prefix length: modes whose multiplicities add up to <= m'
        int64_t cnt = 0;
        int nm = 0;
        // the list is sorted; k = 0 first, multiplicity 1, the rest 2 (real) or 1 (complex)
        for (; nm < ctx->qs_nm; nm++) {
            const int mu = (cplx || nm == 0) ? 1 : 2;
            if (cnt + mu > m_prime) break;
            cnt += mu;
        }
        a.nm = nm;
    }
    a.nsh = ctx->qs_nsh;
    a.B = ctx->d_balls64[1];
    a.t0x = ctx->p.t0[0];
    a.t0y = ctx->p.t0[1];
    a.t0z = ctx->p.t0[2];
    a.invP = 1.0 / ctx->P;
    a.modes = ctx->d_qs_modes;
    a.bv = ctx->d_qs_bv;
    a.Aq = ctx->d_qs_Aq;
    a.mult = ctx->d_qs_mult;
    a.scale = 1.0 / (ctx->P * ctx->P * ctx->P);
    a.complex_w = cplx;
    const int nbc = qs_ball_chunks(a.nB), nmb = qs_mode_blocks(a.nm);
    const size_t per_q = (size_t)nbc * a.nm * sizeof(float2);
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>({n, 65535, (int64_t)((size_t)512 << 20) / (int64_t)per_q}));
    TRY(ensure_query_ws(ctx, chunk));
    TRY(ensure_ws(ctx, (void **)&ctx->d_qs_part, ctx->qs_part_bytes, per_q * chunk));
    TRY(ensure_ws(ctx, (void **)&ctx->d_qs_mpart, ctx->qs_mpart_bytes, sizeof(double) * 2 * nmb * chunk));
    a.part = ctx->d_qs_part;
    a.mpart = ctx->d_qs_mpart;
    for (int64_t q0 = 0; q0 < n; q0 += chunk) {
        const int nq = (int)std::min<int64_t>(chunk, n - q0);
        RotPrepArgs ra{};
        ra.R = dev_R ? R + 9 * q0 : ctx->d_qR;
        ra.t = dev_t ? t + 3 * q0 : nullptr;
        ra.n = nq;
        ra.index_base = q0;
        ra.tol = rot_tol(ctx);
        ra.r64 = dev_R ? ctx->d_qR : nullptr;
        ra.t64 = dev_t ? ctx->d_qt : nullptr;
        ra.status = ctx->d_status;
        if (!dev_R) CU(ctx, cudaMemcpyAsync(ctx->d_qR, R + 9 * q0, sizeof(double) * 9 * nq, cudaMemcpyHostToDevice, s));
        if (!dev_t) CU(ctx, cudaMemcpyAsync(ctx->d_qt, t + 3 * q0, sizeof(double) * 3 * nq, cudaMemcpyHostToDevice, s));
        if (dev_R || dev_t) {
            launch_rot_prep(ra, s);
            ctx->launches++;
        }
        a.nq = nq;
        a.R = ctx->d_qR;
        a.t = ctx->d_qt;
        a.out = host_out ? ctx->d_qout : out + out_per * q0;
        {
            StageScope sc(ctx, s, "evaluate_points_spectral");
            launch_qs(a, s);
            ctx->launches += 3;
        }
        CU(ctx, cudaGetLastError());
        if (host_out) {
            CU(ctx, cudaMemcpyAsync(out + out_per * q0, ctx->d_qout, sizeof(double) * out_per * nq, cudaMemcpyDeviceToHost, s));
            CU(ctx, cudaStreamSynchronize(s));
        }
    }
    if (host_out) TRY(check_deferred(ctx));
    return BC_OK;
}

// ------------------------------------------------------------------ fused exchanges (collectives.cu)

bc_status bc_ipc_handle(bc_ctx *ctx, const void *dev_ptr, void *handle)
{
    if (!ctx) return BC_EINVAL;
    if (!dev_ptr || !handle) return fail(ctx, BC_EINVAL, "NULL dev_ptr/handle");
    CU(ctx, cudaSetDevice(ctx->device));
    {
        // a handle maps the whole allocation: a pointer inside a larger one (e.g. a caching
        // allocator's sub-block) would open at the allocation's base on the peer
        typedef int (*range_fn)(unsigned long long *, size_t *, unsigned long long);
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess && fn &&
            q == cudaDriverEntryPointSuccess) {
            unsigned long long base = 0;
            size_t size = 0;
            if (((range_fn)fn)(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) == 0 &&
                base != (unsigned long long)(uintptr_t)dev_ptr)
                return fail(ctx, BC_EINVAL, "dev_ptr is not the base of its allocation (offset %llu)",
                            (unsigned long long)(uintptr_t)dev_ptr - base);
        }
        cudaGetLastError();
    }
    cudaIpcMemHandle_t h;
    CU(ctx, cudaIpcGetMemHandle(&h, (void *)dev_ptr));
    static_assert(sizeof(h) == BC_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle, &h, sizeof(h));
    return BC_OK;
}

bc_status bc_ipc_open(bc_ctx *ctx, const void *handle, void **dev_ptr)
{
    if (!ctx) return BC_EINVAL;
    if (!dev_ptr || !handle) return fail(ctx, BC_EINVAL, "NULL dev_ptr/handle");
    CU(ctx, cudaSetDevice(ctx->device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    CU(ctx, cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return BC_OK;
}

bc_status bc_ipc_close(bc_ctx *ctx, void *dev_ptr)
{
    if (!ctx) return BC_EINVAL;
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, cudaIpcCloseMemHandle(dev_ptr));
    return BC_OK;
}

bc_status bc_spectrum_A_partial_buffer(bc_ctx *ctx, void **dev_ptr, int64_t *bytes)
{
    if (!ctx) return BC_EINVAL;
    if (ctx->sp64) return fail(ctx, BC_EUNSUPPORTED, "the fp64 spectral parity mode keeps its spectrum private");
    if (!dev_ptr || !bytes) return fail(ctx, BC_EINVAL, "NULL dev_ptr/bytes");
    if (ctx->p.mode != BC_MODE_SPECTRAL) return fail(ctx, BC_EUNSUPPORTED, "exact mode has no spectrum of A");
    CU(ctx, cudaSetDevice(ctx->device));
    const size_t nspec = (size_t)ctx->M * ctx->M * ctx->Kz;
    if (!ctx->d_Ahat_part) TRY(dalloc(ctx, &ctx->d_Ahat_part, sizeof(float2) * nspec));
    *dev_ptr = ctx->d_Ahat_part;
    *bytes = (int64_t)(sizeof(float2) * nspec);
    return BC_OK;
}

bc_status bc_spectrum_A_partial(bc_ctx *ctx, int64_t lo, int64_t hi, void *stream)
{
    if (!ctx) return BC_EINVAL;
    TRY(check_deferred(ctx));
    if (!ctx->have[0]) return fail(ctx, BC_ESTATE, "shape A has not been uploaded");
    if (ctx->p.mode != BC_MODE_SPECTRAL) return fail(ctx, BC_EUNSUPPORTED, "exact mode has no spectrum of A");
    if (lo < 0 || hi < lo || hi > ctx->n[0]) return fail(ctx, BC_EINVAL, "ball slice [%lld, %lld) outside [0, %lld)",
                                                         (long long)lo, (long long)hi, (long long)ctx->n[0]);
    CU(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    void *part = nullptr;
    int64_t bytes = 0;
    TRY(bc_spectrum_A_partial_buffer(ctx, &part, &bytes));
    if (hi == lo) {
        CU(ctx, cudaMemsetAsync(part, 0, (size_t)bytes, s));
        return BC_OK;
    }
    CU(ctx, cudaStreamSynchronize(s));  // the candidate lists below are rebuilt on the host
    TRY(build_csr_A(ctx, lo, hi));
    size_t s1, s2;
    spectral_ws_sizes(ctx, 0, s1, s2);
    Slot &sl = ctx->slot[0];
    TRY(ensure_ws(ctx, &sl.ws1, sl.ws1_bytes, s1));
    TRY(ensure_ws(ctx, &sl.ws2, sl.ws2_bytes, s2));
    float2 *full = ctx->d_Ahat;
    ctx->d_Ahat = (float2 *)part;  // shape_spectrum's x pass writes d_Ahat
    const bc_status st = shape_spectrum(ctx, 0, nullptr, 1, sl.ws1, sl.ws2, s1, s2, s, sl);
    ctx->d_Ahat = full;
    TRY(st);
    if (ctx->prof) collect_profile(ctx);
    return BC_OK;
}

bc_status bc_spectrum_A_reduce(bc_ctx *ctx, const void *const *partials, int n, void *stream)
{
    if (!ctx) return BC_EINVAL;
    if (ctx->sp64) return fail(ctx, BC_EUNSUPPORTED, "the fp64 spectral parity mode keeps its spectrum private");
    TRY(check_deferred(ctx));
    if (!partials || n < 1 || n > BC_MAX_PEERS) return fail(ctx, BC_EINVAL, "need 1..%d partial spectra", BC_MAX_PEERS);
    for (int r = 0; r < n; r++)
        if (!partials[r]) return fail(ctx, BC_EINVAL, "partial spectrum %d is NULL", r);
    if (ctx->p.mode != BC_MODE_SPECTRAL) return fail(ctx, BC_EUNSUPPORTED, "exact mode has no spectrum of A");
    if (!ctx->have[0] || !ctx->have[1]) return fail(ctx, BC_ESTATE, "upload both shapes first (A'' needs B's plan)");
    if (!ctx->plan[1].ok) return fail(ctx, BC_ESTATE, "shape B has no spectral plan (empty B)");
    CU(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t nspec = (size_t)ctx->M * ctx->M * ctx->Kz;
    if (!ctx->d_Ahat) TRY(dalloc(ctx, &ctx->d_Ahat, sizeof(float2) * nspec));
    const bool cplx = ctx->p.weights == BC_WEIGHTS_COMPLEX;
    const ShapePlan &pb = ctx->plan[1];
    ctx->MS = cm_row_stride(pb.L, pb.c, pb.G, ctx->K);
    const size_t ncm = (size_t)ctx->MS * ctx->M * ctx->Kz;
    if (ctx->Ahat_cm_bytes < sizeof(float2) * ncm) {
        TRY(dalloc(ctx, &ctx->d_Ahat_cm, sizeof(float2) * ncm));
        ctx->Ahat_cm_bytes = sizeof(float2) * ncm;
    }
    ReducePermuteArgs a{};
    for (int r = 0; r < n; r++) a.parts[r] = (const float2 *)partials[r];
    a.n_parts = n;
    a.Ahat = ctx->d_Ahat;
    a.mult = pb.d_mult[0];
    a.mult_y = yz_in_A(ctx) ? pb.d_mult[1] : nullptr;
    a.mult_z = yz_in_A(ctx) ? pb.d_mult[2] : nullptr;
    a.out = ctx->d_Ahat_cm;
    a.rows = (long long)ctx->M * ctx->Kz;
    a.K = ctx->K;
    a.L = pb.L;
    a.c = pb.c;
    a.G = pb.G;
    a.neg = cplx;
    a.MS = ctx->MS;
    a.Kz = ctx->Kz;
    a.R2 = ctx->p.band_radius > 0 ? ctx->p.band_radius * ctx->p.band_radius : 0.0;
    a.dec = pb.blob ? ctx->d_dec : nullptr;
    {
        StageScope sc(ctx, s, "reduce_permute");
        launch_reduce_permute(a, s);
        ctx->launches++;
    }
    CU(ctx, cudaGetLastError());
    ctx->cm_ready = true;
    ctx->have_spec = true;
    ctx->probe_done = false;
    ctx->qs_ready = false;
    return BC_OK;
}

bc_status bc_result_buffer(bc_ctx *ctx, int64_t bytes, void **dev_ptr)
{
    if (!ctx) return BC_EINVAL;
    if (!dev_ptr || bytes < 1) return fail(ctx, BC_EINVAL, "NULL dev_ptr or bytes < 1");
    CU(ctx, cudaSetDevice(ctx->device));
    if (ctx->res_bytes < (size_t)bytes) {
        TRY(dalloc(ctx, &ctx->d_res, (size_t)bytes));
        ctx->res_bytes = (size_t)bytes;
        CU(ctx, cudaMemset(ctx->d_res, 0, (size_t)bytes));
    }
    *dev_ptr = ctx->d_res;
    return BC_OK;
}

bc_status bc_set_result_peers(bc_ctx *ctx, void *const *buffers, int n, int64_t base)
{
    if (!ctx) return BC_EINVAL;
    if (n < 0 || n > BC_MAX_PEERS || (n > 0 && !buffers) || base < 0)
        return fail(ctx, BC_EINVAL, "need 0..%d result buffers and base >= 0", BC_MAX_PEERS);
    for (int r = 0; r < n; r++)
        if (!buffers[r]) return fail(ctx, BC_EINVAL, "result buffer %d is NULL", r);
    ctx->res_peers = ResultPeers{};
    for (int r = 0; r < n; r++) ctx->res_peers.buf[r] = buffers[r];
    ctx->res_peers.n = n;
    ctx->res_peers.base = base;
    return BC_OK;
}

bc_status bc_sync(bc_ctx *ctx, void *stream)
{
    if (!ctx) return BC_EINVAL;
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, cudaStreamSynchronize((cudaStream_t)stream));
    TRY(check_deferred(ctx));
    return BC_OK;
}

bc_status bc_query(const bc_ctx *ctx, const char *key, double *value)
{
    if (!ctx || !key || !value) return BC_EINVAL;
    const std::string k(key);
    const ShapePlan &A = ctx->plan[0], &B = ctx->plan[1];
    if (k == "P") *value = ctx->P;
    else if (k == "tau_A") *value = A.tau;
    else if (k == "tau_B") *value = B.tau;
    else if (k == "G_A") *value = A.G;
    else if (k == "G_B") *value = B.G;
    else if (k == "L_A") *value = A.L;
    else if (k == "L_B") *value = B.L;
    else if (k == "c_A") *value = A.c;
    else if (k == "c_B") *value = B.c;
    else if (k == "cut_A") *value = A.cut;
    else if (k == "cut_B") *value = B.cut;
    else if (k == "band_modes") *value = (double)ctx->M * ctx->M * ctx->Kz;
    else if (k == "batch") *value = ctx->batch;
    else if (k == "bytes_workspace")
        *value = (double)(ctx->slot[0].ws1_bytes + ctx->slot[0].ws2_bytes + ctx->slot[1].ws1_bytes + ctx->slot[1].ws2_bytes);
    else if (k == "fused_spread_z") *value = use_spread_z(ctx) ? 1 : 0;
    else if (k == "blob_B") *value = B.blob ? 1 : 0;
    else if (k == "spread_cells_B") *value = ctx->spread_cells_B;
    else if (k == "live_tiles_B") *value = (double)ctx->live_tiles_B;
    else if (k == "K") *value = ctx->K;
    else if (k == "band_error") *value = ctx->probe_done ? ctx->probe_err : -1.0;
    else if (k == "query_modes") *value = (double)ctx->qs_m;
    else if (k == "Np") *value = ctx->p.Np;
    else if (k == "fused_fold_inv") *value = (!ctx->p.generic_only && fold_fuses_inverse(B.L, ctx->p.Np)) ? 1 : 0;
    else if (k == "fold_fast")
        *value = (!ctx->p.generic_only && fold_fast_supported(B.L, B.c, B.G, ctx->K, ctx->p.Np,
                                                             ctx->p.weights == BC_WEIGHTS_COMPLEX)) ? 1 : 0;
    else if (k == "dock_fast") *value = use_dock_fast(ctx) ? 1 : 0;
    else return BC_EINVAL;
    return BC_OK;
}

int64_t bc_launch_count(const bc_ctx *ctx) { return ctx ? ctx->launches : 0; }

bc_status bc_set_profiling(bc_ctx *ctx, int enabled)
{
    if (!ctx) return BC_EINVAL;
    ctx->prof = enabled != 0;
    return BC_OK;
}

int bc_stage_times(bc_ctx *ctx, const char **names, double *total_ms, int64_t *launches, int cap)
{
    if (!ctx) return 0;
    collect_profile(ctx);
    int n = 0;
    for (const std::string &nm : ctx->stage_order) {
        if (n < cap) {
            auto &v = ctx->stage_ms[nm];
            if (names) names[n] = ctx->stage_ms.find(nm)->first.c_str();
            if (total_ms) total_ms[n] = v.first;
            if (launches) launches[n] = v.second;
        }
        n++;
    }
    return n;
}

bc_status bc_reset_stage_times(bc_ctx *ctx)
{
    if (!ctx) return BC_EINVAL;
    collect_profile(ctx);
    ctx->stage_ms.clear();
    ctx->stage_order.clear();
    return BC_OK;
}

}  // extern "C"
