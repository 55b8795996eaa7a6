// kernels.cuh -- launch-parameter structs and kernel declarations of libballcorr.
#pragma once

#include "common.cuh"

#include "ballcorr.h"  // BC_MAX_PEERS: ranks of one NVLink / NVSwitch domain (one box)

// ----------------------------------------------------------------- spreading
// Gaussian-smoothed ball density on a box of the fine lattice (spacing hf):
//   rho_s(x_n) = sum_j v_j (1_{B(c_j, s_j)} * G_tau)(x_n),  x_n = (o + n) hf,  n in [0, L)^3
// (the knot density rho_P of PAPER.md L150 eq_rhoP convolved with the ball
// primitive, eq_ballconv, and with an isotropic Gaussian G_tau that the
// spectral deconvolution removes exactly).
struct SpreadArgs {
    int L;            // box edge (cells)
    int ox, oy, oz;   // box origin in fine cells
    float hf;         // fine spacing
    float inv_hf;
    float tau;        // Gaussian sigma (length units)
    float cut;        // footprint radius beyond the ball radius (length units)
    int n_balls;      // candidate count when csr == nullptr
    const float4 *balls;    // (x, y, z, s) fp32
    const float *w_re;      // weights (real part), nullptr => 1
    const float *w_im;      // imaginary parts (complex mode), nullptr => 0
    const int *csr_off;     // per-tile candidate offsets (A) or nullptr (all balls)
    const int *csr_idx;
    const float *rot;       // per batch element 9 floats (row-major R) or nullptr (identity)
    int complex_w;
    void *out;              // float [b][L][L][L] (real) or float2 (complex)
    long long out_batch_stride;  // elements
    int tiles_per_axis;
    // optional per-ball radial profile tables: cubic pieces c0 + t c1 + t^2 c2 + t^3 c3 on
    // intervals of width dprof (length units); ball j's pieces start at prof[prof_off[j]]
    const float4 *prof;
    const int *prof_off;
    float inv_dprof;
    // optional per-rotation candidate lists of B (16 x 16-column bins of spread_z.cu's binning):
    // tile (tx, ty, tz) scans bin tx * bpa + ty of its rotation
    const int *bin_counts, *bin_offs, *bin_lists;
    long long bin_stride;
    int nbins, bpa;
};

// fused spreading + z transform of R B (spread_z.cu), real weights.  Cell units throughout:
// ball (x, y, z, s) / hf in B's frame; the box origin o (cells); cut = footprint beyond s.
// per-rotation binning of B's balls for spread_z (16 x 16-column bins, ball order)
struct SzBinArgs {
    int n;                  // balls
    const float4 *balls;    // (x, y, z, s) / hf, B frame
    const float *rot;       // [b][9]
    float ox, oy, oz, cut;  // box origin (cells), window support W (cells)
    float4 *recA;           // [b][n] (u_x, u_y, u_z, (s + W)^2), box cells
    int bpa, nbins;         // bins per axis, bins
    int *counts, *offs;     // [b][nbins]
    int *lists;             // [b][list_stride] ball indices
    long long list_stride;
};
int spread_z_bins(int L);
int spread_z_bins_per_axis(int L);
int spread_z_bins_per_ball(float rc_max);
void launch_spread_z_bin(const SzBinArgs &a, int batch, cudaStream_t s);

struct SpreadZArgs {
    int L, K, c, G;
    int n_balls;
    const float4 *recA;     // [b][n] rotated balls (SzBinArgs)
    const float4 *recB;     // [n] (s, w, g0, g2): radius (cells), weight (real part), d -> 0 series g0 + g2 d^2
    const float *recWi;     // [n] imaginary part of the weight (complex weights: BOX mode only)
    const float4 *recBim;   // [n] (s, Im w, g0, g2) (complex weights, planar box)
    int cplx;               // complex weights: the box holds float2 cells
    int planar;             // complex weights: two real spreads (Re w, then Im w) into the planes
                            // box[b][0 .. L^3) (real parts) and box[b][L^3 .. 2 L^3) (imaginary)
    const int *counts, *offs, *lists;  // the bins (SzBinArgs)
    int nbins;
    long long list_stride;
    const float4 *phi;      // cubic pieces on [-U, U]: [phi_n] of Phi1, then [phi_n] of Phi2
    int phi_n;
    float phi_U, phi_invD;
    float cx, cy, live_r2;  // support cylinder of R B (any R): centre (cells) and radius^2
    float zero_r2;          // tiles farther than sqrt(zero_r2) from the axis are zero
    int skip_zero;          // 1: do not write the zero tiles (the y pass never reads them)
    const float2 *mult_z;   // [K + 1]
    const float2 *tw;       // exp(-2 pi i m / L)
    const float2 *ctw;      // [c][L]
    float2 *out;            // T1 [b][L][L][K + 1]
    long long out_bstride;  // float2 elements
    float *box;             // non-null: spread to this fp32 box [b][L][L][L] (stride box_bstride, floats;
    long long box_bstride;  // complex: float2 cells), then a separate z transform (spread_z.cu / passes.cu)
};
bool spread_z_supported(int L, int complex_w);
bool launch_spread_z(const SpreadZArgs &a, int batch, cudaStream_t s);  // false: unsupported plan/table

// ----------------------------------------------------------------- coset-major band order
// Band |k| <= K of an axis plan (L, c, G): coset p holds q in [0, qp] (k = c q + p >= 0) and
// [qn, L) (k = c q + p - G < 0), stored negative part first (ascending k).  Every coset
// segment starts on an even position (16-byte aligned float2 rows for cp.async).
struct CmSeg {
    int off, qn, cnt;  // segment start, first negative q, entries
};
__host__ __device__ constexpr CmSeg cm_segment(int p, int L, int c, int G, int K)
{
    int off = 0;
    for (int pp = 0; pp <= p; pp++) {
        const int qp = K >= pp ? (K - pp) / c : -1;
        const int qn = (G - K - pp + c - 1) / c;
        const int cnt = (qp + 1) + (L - qn);
        if (pp == p) return CmSeg{off, qn, cnt};
        off += (cnt + 1) & ~1;
    }
    return CmSeg{0, 0, 0};
}
__host__ __device__ constexpr int cm_row_stride(int L, int c, int G, int K)
{
    const CmSeg s = cm_segment(c - 1, L, c, G, K);
    return s.off + ((s.cnt + 1) & ~1);
}
__host__ __device__ inline int cm_max_seg(int L, int c, int G, int K)
{
    int m = 0;
    for (int p = 0; p < c; p++) {
        const CmSeg s = cm_segment(p, L, c, G, K);
        m = s.cnt > m ? s.cnt : m;
    }
    return (m + 1) & ~1;
}
// position of band mode k within its row
__host__ __device__ inline int cm_of_k(int k, int L, int c, int G, int K)
{
    const int kk = k < 0 ? k + G : k;
    const int p = kk % c, q = (kk - p) / c;
    const CmSeg s = cm_segment(p, L, c, G, K);
    return s.off + (q >= s.qn ? q - s.qn : q + (L - s.qn));
}

// ----------------------------------------------------------------- axis transforms (passes.cu)
// One axis of the box DFT:  X(k) = mult(k) sum_{n<L} x_n exp(-2 pi i k n / G),  G = c L,
// through c cosets k = c q + p of an L-point FFT of x_n exp(-2 pi i p n / G);
// the inverse passes use c = 1, sign +1 and unsigned outputs q in [0, nk).
struct PassArgs {
    int L, c, G;
    int klo, nk, signed_k;
    const float2 *mult;   // nk multipliers (nullptr => 1)
    const float2 *tw;     // exp(-2 pi i m / L), m < L
    const float2 *ctw;    // coset twiddles exp(-2 pi i p n / G), [c][L]
    // contiguous: in[b][lines][L] -> out[b][lines][nk]
    long long lines;
    int in_real;
    // strided: in[b][O][L][I] -> out[b][O][nk][I] (row pitches pitch_in / pitch_out, 0 = I)
    int O, I;
    int pitch_in, pitch_out;
    long long in_bstride, out_bstride;
    const void *in;
    float2 *out;
    // contiguous rows of a box of L columns per x (row = x L + y): zskip = 1 treats the rows of
    // the 4 x 4-column tiles that spread_z left unwritten (outside B's support cylinder, the
    // spread's own test with centre (zcx, zcy) and zero_r2) as zero without reading them
    int zskip;
    float zcx, zcy, zero_r2;
    // strided forward pass over such a box's T1 (O = x planes, rows = y): ylive = 1 loads only
    // the rows within sqrt(live_r2) of the support axis (zcx, zcy) -- the rows zskip may leave
    // unwritten lie beyond it -- and writes a zero plane without transforming it
    int ylive;
    float live_r2;
};

// fused x-pass of R B + spectral product with A + fold onto Np^3 (passes.cu)
struct FoldXArgs {
    int L, c, G;
    int K, M, Kz, Np, Fz;
    int complex_w;
    const float2 *mult;   // unused (B's x multipliers are folded into Ahat)
    const float2 *tw, *ctw;
    const float2 *T2;     // [b][ix][ky][kz]
    long long t2_bstride;
    const float2 *Ahat;   // [ky][kz][x in coset-major order of B's x plan, row stride MS]: origin phase
                          // and B's x multipliers folded in
    int MS;               // row stride of Ahat (cm_row_stride)
    const int *xtab;      // [c][L] per FFT output (p, q): segment position | fold target << 16, or -1
    const int2 *segs;     // [c] (segment offset, entries) of the coset-major rows
    float2 *F;            // [b][Np][Np][Fz], or X1 [b][N][Np][Fz] when the inverse x pass is fused
    long long f_bstride;
    int N;                // output rows of the fused inverse x pass
    int fuse_inv;         // request the fused inverse x pass (taken when fold_fuses_inverse(L, Np))
    const float2 *tw_inv; // exp(-2 pi i m / Np)
    int nb;               // rotations in the launch (set by launch_fold_x)
};

// fold_fast.cu: fold_x with the inverse x pass for the plan shape L = Np = 256, c = 4,
// G = 4 (K + 1), real weights (compile-time band and fold ownership)
struct FoldFastArgs {
    const float2 *tw, *ctw;  // exp(-2 pi i m / 256); coset twiddles [4][256]
    const float2 *T2;        // [b][ix][ky][kz]
    long long t2_bstride;
    const float2 *Ahat;      // A'' rows (coset-major, stride MS)
    int MS;
    int pos_base[4];         // per coset: segment offset - first negative q
    float2 *X1;              // [b][N][Np][x1_pitch]
    long long x1_bstride;
    int x1_pitch;            // row pitch (>= Np/2 + 1; 136 keeps 64-byte row pieces sector-aligned)
    int N;
    int nb;                  // set by launch_fold_fast
};
bool fold_fast_supported(int L, int c, int G, int K, int Np, int complex_w);

// dock_fast.cu: the docking plan shape (L = 384, c = 2, G = 768, K = 191, Np = 128, complex
// weights) with compile-time constants: z and y passes of R B and the fold.  T1 / T2 rows
// hold kz at index kz + 192 (pitch dock_t_pitch() = 384).
struct DockPassArgs {
    const float2 *tw, *ctw, *mult;  // twiddles, coset twiddles [2][384], the axis multipliers [2K + 1]
    const float2 *in;               // z: planar box [b][2][L][L][L] floats (real plane, then
                                    // imaginary plane, spread_z planar); y: T1 [b][L][L][384]
    long long in_bstride;
    float2 *out;                    // z: T1; y: T2 [b][L][kz + 192][ky + 192] (384 x 384 per x)
    long long out_bstride;
    float cx, cy, live_r2, zero_r2; // B's support cylinder (spread_z's tile and row tests)
};
struct DockFoldArgs {
    const float2 *tw, *ctw;
    const float2 *T2;
    long long t2_bstride;
    const float2 *Ahat;             // A'' rows (coset-major, stride MS)
    int MS;
    int pos_base[2];
    float2 *F;                      // [b][Np][Np][Np] (k'x, k'y, k'z)
    long long f_bstride;
    float cx, live_r2;              // live x planes of T2
    int nb;                         // set by launch_fold_dk
};
bool dock_fast_supported(int L, int c, int G, int K, int Np, int complex_w);
void launch_pass_z_dk(const DockPassArgs &a, int batch, cudaStream_t s);
void launch_pass_y_dk(const DockPassArgs &a, int batch, cudaStream_t s);
bool launch_fold_dk(const DockFoldArgs &a, int batch, cudaStream_t s);
size_t dock_t_pitch();

// fold_fast.cu: forward y pass of R B for the same plan shape (live-row input skipping)
struct PassYFastArgs {
    const float2 *tw, *ctw, *mult;  // twiddles, coset twiddles [4][256], mult_y [2K + 1]
    const float2 *T1;               // [b][L][L][K + 1]
    long long t1_bstride;
    float2 *T2;                     // [b][L][2K + 1][K + 1]
    long long t2_bstride;
    float cx, cy, live_r2;          // B's support cylinder (cells)
};
bool pass_y_fast_supported(int L, int c, int G, int K, int complex_w);
void launch_pass_y_fast(const PassYFastArgs &a, int batch, cudaStream_t s);
bool launch_fold_fast(const FoldFastArgs &a, int batch, cudaStream_t s);  // false: strides not the compiled ones

// contiguous inverse z pass + epilogue
struct LastArgs {
    int Np, N, Fz;
    int pitch;           // row pitch of `in` in float2 (0 = Fz)
    int hermitian;       // 1: C2R from Fz = Np/2+1 stored modes; 0: C2C, Fz = Np
    float scale;
    const float2 *tw;    // exp(-2 pi i m / Np)
    const float2 *in;    // [b][N*N lines][Fz]
    long long in_bstride;
    int out_kind;        // BC_OUT_*
    void *out_full;      // float [b][N^3] or float2
    long long full_bstride;
    unsigned long long *keys;  // [b][2]: (min key, max key)
};

void launch_spread(const SpreadArgs &a, int batch, cudaStream_t s);
bool fft_size_supported(int L);
// kind: 0 forward contiguous (z), 1 forward strided (y), 2 forward strided -> rows (x of A),
//       3 inverse strided (x, y of the inverse transform)
void launch_pass(const PassArgs &a, int kind, int batch, cudaStream_t s);
void launch_fold_x(const FoldXArgs &a, int batch, cudaStream_t s);
bool fold_fuses_inverse(int L, int Np);
void launch_last(const LastArgs &a, int batch, cudaStream_t s);
void launch_permute_cm(const float2 *in, const float2 *mult, float2 *out, long long rows, int K, int L, int c, int G,
                       int neg, int MS, int Kz, double band_radius, const float *dec, cudaStream_t s, const float2 *mult_y = nullptr, const float2 *mult_z = nullptr);
void launch_keys_init(unsigned long long *keys, int n, cudaStream_t s);
// peers: result buffers (bc_extremum[], device pointers, possibly mapped from other GPUs) that
// receive the same records at global rotation index peer_base + r (nullptr / 0: none)
struct ResultPeers {
    void *buf[BC_MAX_PEERS];
    int n;
    long long base;
};
void launch_keys_finalize(const unsigned long long *keys, int batch, int out_kind, void *out, const ResultPeers &peers,
                          cudaStream_t s);

// collectives.cu: all-reduce of partial spectra (peer reads) fused into the A'' build
struct ReducePermuteArgs {
    const float2 *parts[BC_MAX_PEERS];  // partial band spectra [ky][kz][kx], one per rank, rank order
    int n_parts;
    float2 *Ahat;                       // reduced spectrum (this rank)
    const float2 *mult;                 // B's x multipliers
    float2 *out;                        // A'' (coset-major rows, stride MS)
    long long rows;
    int K, L, c, G, neg, MS, Kz;
    double R2;
    const float *dec;
    const float2 *mult_y, *mult_z;      // B's y / z multipliers folded in too (fast plan), or nullptr
};
void launch_reduce_permute(const ReducePermuteArgs &a, cudaStream_t s);

// ----------------------------------------------------------------- exact mode
struct ExactArgs {
    int nA, nB, N;
    double h, inv_h, t0x, t0y, t0z;
    const double4 *A;    // (x, y, z, r)
    const double4 *B;
    const double2 *wA;   // (re, im)
    const double2 *wB;
    const double *rot;   // [b][9]
    int complex_w;
    int fp64;            // evaluate V in double (1) or float (0)
    long long *iacc;     // [b][N^3] (re) followed by [b][N^3] (im) when complex: fixed point, value * qscale
    long long acc_bstride;
    double qscale;       // 2^61 / (bound on |f|)
    int i0;              // first A ball of the launch (set by launch_exact_scatter)
    int thread_per_knot; // 1: thread per knot (small footprints), 0: warp per knot
    const int *permB;    // B's balls in order of radius (thread-per-knot kernel)
    int packed;          // fp32: two 32-bit point sums per 64-bit word (exact_knot_pack_kernel)
};
void launch_exact_scatter(const ExactArgs &a, int batch, cudaStream_t s);

struct ExactOutArgs {
    int N;
    int complex_w, fp64;
    const long long *iacc;
    long long acc_bstride;
    double inv_qscale;
    int packed;          // accumulators as packed 32-bit pairs (ExactArgs::packed)
    int out_kind;
    void *out;           // full output or bc_extremum[]
    double *partials;    // scratch: [b][nblocks][2] vals
    long long *partial_idx;
};
void launch_exact_out(const ExactOutArgs &a, int batch, cudaStream_t s, int *launches);

// ----------------------------------------------------------------- single-configuration query (query.cu)
struct QueryArgs {
    int nq, nB;
    const double *R, *t;            // [nq][9], [nq][3]
    const double4 *A, *B;           // (x, y, z, r)
    const double2 *wA, *wB;         // (re, im)
    const int *start, *idx;         // A's uniform grid: CSR over cells (ball order within a cell)
    int nx, ny, nz;
    double gx0, gy0, gz0, inv_cs;
    double *partial;                // [nq][blocks][2]
    double *out;                    // [nq] (real) or [nq][2] (complex)
    int complex_w;
};
int query_blocks(int nB);
void launch_query(const QueryArgs &a, cudaStream_t s);

// ----------------------------------------------------------------- device-side validation (validate.cu)
enum : unsigned {
    BC_DEFER_NONFINITE_R = 1u,
    BC_DEFER_NOT_ORTHONORMAL = 2u,
    BC_DEFER_DET = 4u,
    BC_DEFER_NONFINITE_T = 8u,
};
struct RotPrepArgs {
    const double *R;     // [n][9] caller array (device)
    const double *t;     // [n][3] caller translations (device) or nullptr
    long long n;
    long long index_base;  // index of R[0] in the caller's array (chunked calls)
    double tol;          // max |R R^T - I| entry
    float *r32;          // [n][9] fp32 copy or nullptr
    double *r64;         // [n][9] fp64 copy or nullptr
    double *t64;         // [n][3] fp64 copy of t or nullptr
    unsigned *status;    // [2] (mapped host memory): OR of BC_DEFER_* flags, lowest bad index
};
void launch_rot_prep(const RotPrepArgs &a, cudaStream_t s);

// ----------------------------------------------------------------- spectral single-configuration query (query_spectral.cu)
struct QsArgs {
    int nq, nB, nm, nsh;
    const double *R, *t;     // [nq][9], [nq][3]
    const double4 *B;        // B's balls (x, y, z, s)
    double t0x, t0y, t0z, invP;
    const int4 *modes;       // [nm] (kx, ky, kz, shell index)
    const float2 *bv;        // [nB][nsh] v_j beta_hat(s_j, |k_shell| / P)
    const float2 *Aq;        // [nm] A'(k) of the retained modes
    const float *mult;       // [nm] 1 (k = 0, or complex weights) or 2 (a +-k pair, real weights)
    float2 *part;            // [nq][ball chunks][nm]
    double *mpart;           // [nq][mode blocks][2]
    double *out;             // [nq] or [nq][2]
    double scale;            // 1 / P^3
    int complex_w;
};
struct QsTableArgs {
    const double4 *B;
    const double2 *wB;
    int nB;
    const int *k2;           // [nsh] |k|^2 of each shell
    int nsh;
    double P;
    int complex_w;
    float2 *bv;              // [nB][nsh]
    const float2 *Ahat;      // band spectrum [ky][kz][kx]
    const int4 *modes;
    int nm, K, Kz;
    float2 *Aq;              // [nm]
};
int qs_ball_chunks(int nB);
int qs_mode_blocks(int nm);
void launch_qs_tables(const QsTableArgs &t, cudaStream_t s);
void launch_qs(const QsArgs &a, cudaStream_t s);

// ----------------------------------------------------------------- spectral fp64 parity mode (spectral64.cu)
struct Sp64SpreadArgs {
    int L;                  // box edge (cells)
    double o[3];            // box origin (cells)
    double hf, tau, cut;    // fine spacing, Gaussian sigma, footprint beyond the radius (length)
    const double4 *balls;   // (x, y, z, r)
    const double2 *w;       // weights (re, im)
    int n;
    const double *rot;      // 9 doubles (row-major R) or nullptr (identity)
    double2 *out;           // box [L][L][L]
};
struct Sp64DftArgs {
    const double2 *in;      // [O][Lin][I]
    double2 *out;           // [O][nq][I]
    int O, Lin, I, nq;
    long long qlo, nlo;     // output index q <-> qlo + q, input n <-> nlo + n
    long long G;            // period of the phase (fine grid G forward, Np inverse)
    int sign;               // -1 forward, +1 inverse
    const double2 *tw;      // e^{-2 pi i r / G}, r in [0, G)
    int mult;               // forward multipliers (below) or none
    long long off;          // box origin on this axis (cells)
    double hf, tau, P, t0;
    int origin;             // A: times the origin phase e^{2 pi i k t0 / P}
};
void launch_sp64_spread(const Sp64SpreadArgs &a, cudaStream_t s);
void launch_sp64_dft(const Sp64DftArgs &a, cudaStream_t s);
void launch_sp64_product(const double2 *A, const double2 *B, double2 *Gk, int M, cudaStream_t s);
void launch_sp64_output(const double2 *f, long long n, double scale, int complex_w, double *out, cudaStream_t s);
