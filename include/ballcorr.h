/*
 * ballcorr.h -- C ABI of the B200 ball-set correlator (libballcorr.so).
 *
 * Operation (eq_relg_0 / eq_relg):
 *
 *     f_R(t) = < f_A , f_{RB} o T^{-1} > = integral rho_A(x) rho_{RB}(x - t) dx
 *
 * for two solids given as weighted sums of ball indicators (eq_un;
 * sharp alpha -> infinity limit of eq_psi)
 *
 *     rho_A(x) = sum_i w_i 1{|x - a_i| <= r_i},   rho_B(x) = sum_j v_j 1{|x - b_j| <= s_j},
 *
 * rotated about B's frame origin (x -> R x, eq_Mink0, Appendix B)
 * and evaluated on the translation grid t_m = t0 + m h, m in [0, N)^3.  Up to
 * rounding and the band limit below, f_R(t) = sum_ij w_i v_j V(r_i, s_j,
 * |a_i - R b_j - t|) with V the two-ball lens volume (eq_ORP / eq_convgP,
 * L343-L360).
 *
 * Two modes compute it:
 *   BC_MODE_SPECTRAL  the paper's Fourier route (L398-L419 eq_ccghat,
 *                     L276-L294 eq_fballhat / eq_rhoPhat): knot spectra with
 *                     the exact ball transform, the conjugate spectral
 *                     product, one inverse FFT per rotation.  Result = the
 *                     Fourier partial sum over the band |k_i| <= K (k/P,
 *                     P = Np h) of the P-periodised f (fp32).
 *   BC_MODE_EXACT     the paper's combinatorial route (obstacle knots
 *                     a_i - R b_j with primitive kernel f_{B1} * f_{B2} = V,
 *                     L347-L360): direct pair-lens spreading (fp32 or fp64).
 *
 * Conventions
 *   * Arrays are C order.  A full output f[n_rot][N][N][N] is indexed
 *     f[r][mx][my][mz] (z fastest); the linear index reported by the
 *     reductions is (mx*N + my)*N + mz.  Ties resolve to the lowest index.
 *   * Complex weights (BC_WEIGHTS_COMPLEX) are interleaved (re, im) doubles.
 *     f is defined WITHOUT conjugating weights (reading C-3): the
 *     pair weight is w_i * v_j.
 *   * Pointers documented "host or device" are classified with
 *     cudaPointerGetAttributes; host buffers are staged by the library.
 *   * `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *
 * Ownership and threading: the caller owns every buffer it passes; the
 * library copies inputs it keeps (shapes, R) and owns all device scratch,
 * freed by bc_destroy.  A context is bound to one device and is NOT
 * thread-safe: one host thread per context.
 *
 * Errors: every call returns bc_status; bc_last_error(ctx) gives a message.
 * Asynchronous CUDA faults surface at the next synchronising call as
 * BC_ECUDA.  No call falls back to a CPU implementation.
 */
#ifndef BALLCORR_H
#define BALLCORR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BC_OK = 0,
    BC_EINVAL = 1,        /* bad argument: NULL, size <= 0, non-finite, r <= 0, R not a rotation */
    BC_ERANGE = 2,        /* support would wrap onto the grid (P too small) or exceed the plan */
    BC_ENOMEM = 3,        /* device allocation failed */
    BC_ESTATE = 4,        /* call out of order (e.g. correlate before upload / spectrum) */
    BC_EUNSUPPORTED = 5,  /* parameter combination not implemented */
    BC_ECUDA = 6          /* CUDA runtime error (message in bc_last_error) */
} bc_status;

typedef enum { BC_FP32 = 0, BC_FP64 = 1 } bc_precision;
typedef enum { BC_MODE_SPECTRAL = 0, BC_MODE_EXACT = 1 } bc_mode;
typedef enum { BC_WEIGHTS_REAL = 0, BC_WEIGHTS_COMPLEX = 1 } bc_weight_kind;

typedef enum {
    BC_OUT_F_FULL = 0,     /* f[n_rot][N][N][N]: float (FP32), double (FP64); complex: (re,im) pairs */
    BC_OUT_MIN_ARGMIN = 1, /* bc_extremum[n_rot]: min of f (real weights) */
    BC_OUT_MAX_ARGMAX = 2, /* bc_extremum[n_rot]: max of f (real weights) */
    BC_OUT_MINMAX = 3,     /* bc_extremum[n_rot][2]: {min, max} (real weights) */
    BC_OUT_MAX_REAL = 4    /* bc_extremum[n_rot]: max of Re f (any weights; docking score) */
} bc_out_kind;

/* Per-rotation extremum; idx = (mx*N + my)*N + mz. */
typedef struct {
    double val;
    int64_t idx;
} bc_extremum;

typedef struct {
    int32_t N;            /* translations per axis, >= 1 */
    double h;             /* grid spacing, > 0 */
    double t0[3];         /* grid origin */
    int32_t Np;           /* FFT period in grid cells: P = Np*h; Np >= N; factors in {2,3,5} (spectral) */
    int32_t K;            /* band half-width: modes |k_i| <= K, K < 4096 (spectral) */
    int32_t precision;    /* bc_precision; SPECTRAL with BC_FP64 is a parity mode: the same plan and
                             method with direct fp64 sums instead of the fp32 FFT kernels (K <= 64,
                             Np <= 256, box <= 160 cells, BC_OUT_F_FULL only; no tolerance probe,
                             spectral query or spectrum exchange) */
    int32_t mode;         /* bc_mode */
    int32_t weights;      /* bc_weight_kind */
    int32_t max_batch;    /* rotations processed per launch; 0 = library default */
    double spread_eps;    /* spectral: target aliasing/truncation level of the spreading (0 = 1e-7) */
    double band_radius;   /* spectral: > 0 additionally restricts the band to |k| <= band_radius */
    int32_t generic_only; /* spectral: nonzero disables the fused per-plan kernels (spread + z
                             transform, fold + inverse x) and runs the generic passes instead;
                             same result up to fp32 rounding order (a test hook) */
    int32_t concurrency;  /* spectral: rotation batches in flight on internal streams forked from
                             and joined to the caller's stream (0 or 1 = one batch at a time, on
                             the caller's stream; 2 = two) */
    double tolerance;     /* spectral: > 0 enables the band-error guard: before the first
                             correlation of a pair of uploaded shapes the library estimates the
                             relative band error max|f_spec - f| / max|f| (two probe rotations,
                             the spectral grid against the exact pair-lens f at ~3,800 sampled
                             translations) and bc_correlate_rotations returns BC_ERANGE when it
                             exceeds `tolerance` (raise K).  That first call is then synchronous.
                             0 = off.  The estimate: bc_query("band_error"). */
} bc_params;

typedef struct bc_ctx bc_ctx;

/* Create a context on `device`.  Validates params (EINVAL / EUNSUPPORTED). */
bc_status bc_create(int device, const bc_params *params, bc_ctx **out);

/* Release every device and host resource of the context (NULL is a no-op). */
bc_status bc_destroy(bc_ctx *ctx);

/*
 * Upload shape `which` (0 = A, the fixed solid; 1 = B, the moving solid).
 *   xyzr: host or device, n rows of (x, y, z, r) doubles, r > 0, all finite.
 *   w:    host or device; n doubles (REAL) or 2n interleaved doubles (COMPLEX);
 *         NULL means every weight is 1.
 * The data are copied; re-uploading A invalidates the spectrum of A.
 * Spectral mode additionally checks, once both shapes exist, that no
 * periodic image of f's support reaches the grid: with the per-axis support
 * bound S = max_i |a_i,axis| + max_j |b_j| + max r + max s it requires
 * P >= max(S - t0, t0 + (N-1) h + S) on every axis (P = Np h), else
 * BC_ERANGE.  The box of each shape must also fit its spreading plan.
 * Synchronous with respect to the host; device xyzr / w are read after a device-wide
 * synchronisation (they may come from any stream).
 */
bc_status bc_shape_upload(bc_ctx *ctx, int which, const double *xyzr, const double *w, int64_t n);

/* Compute and keep the spectrum of A on the band (PAPER.md L280-L294 eq_rhoPhat /
 * eq_fballhat: knot transform times the ball transform; spectral mode, a no-op in exact
 * mode).  Idempotent.  BC_ESTATE if A is missing.  Asynchronous on `stream`: runs in the
 * context's workspaces, allocating them only on first use (no per-call allocation or
 * synchronisation). */
bc_status bc_spectrum_A(bc_ctx *ctx, void *stream);

/*
 * Distribution of A's spectrum over GPUs (north_star: "A's spectrum broadcast"; SURVEY
 * §8(b)/(e)): rotations are sharded over ranks and every rank needs the same band spectrum
 * of A (the factor rho_A_hat of the spectral product), so one rank
 * computes it and the others receive it instead of recomputing it.
 *
 * bc_spectrum_A_buffer: the device buffer (on the context's device) that holds A's band
 * spectrum, M*M*Kz complex64 values (M = 2K+1, Kz = K+1 for real and M for complex
 * weights; layout private to the library, identical for identical bc_params).  Allocated on
 * first use and owned by the context (freed by bc_destroy; valid until then).  After
 * bc_spectrum_A it holds the spectrum.  Spectral mode only (BC_EUNSUPPORTED otherwise).
 *
 * bc_spectrum_A_import: declare the buffer's current contents to be A's spectrum, written
 * by the caller (e.g. an NCCL broadcast from a context with identical bc_params that ran
 * bc_spectrum_A on the same shape A).  The caller must have completed those writes (device
 * synchronised).  Shape A must be uploaded (its extent enters the support check); BC_ESTATE
 * otherwise.  Re-uploading A invalidates the import as it invalidates bc_spectrum_A.
 */
bc_status bc_spectrum_A_buffer(bc_ctx *ctx, void **dev_ptr, int64_t *bytes);
bc_status bc_spectrum_A_import(bc_ctx *ctx);

/*
 * Correlate A with R B for n_rot rotations (PAPER.md L316-L322 eq_relg; spectral route
 * L398-L419 eq_ccghat, one inverse transform per rotation).
 *   R:   host or device, n_rot row-major 3x3 doubles; every entry finite, |R R^T - I| <= 1e-5
 *        (BC_FP32) or 1e-12 (BC_FP64) entrywise and det R > 0 (R in SO(3), L221-L233).
 *        Host R: checked before any work, BC_EINVAL.  Device R: checked ON THE DEVICE by a
 *        kernel on `stream` (no host round trip); a violation is reported as BC_EINVAL by the
 *        next call on this context or by bc_sync (the outputs of the offending call are
 *        undefined), like an asynchronous CUDA fault.
 *   out: host or device buffer laid out per bc_out_kind, at least n_rot * (bytes per rotation)
 *        bytes (BC_OUT_F_FULL: N^3 values of the result type; reductions: sizeof(bc_extremum),
 *        twice for BC_OUT_MINMAX).  The library cannot check its size.
 * Device R and out: asynchronous on `stream` -- no host synchronisation, no host copies
 * (except the one-time band-error probe when bc_params.tolerance > 0).  Host buffers: the
 * call stages them and returns after the result has reached `out`.  Calls on one context
 * must be ordered by the caller (same stream, or synchronised): they share workspaces.
 * Spectral mode needs bc_spectrum_A first (BC_ESTATE otherwise).
 * CUDA graphs: with device R and out, a call made after a first (warm-up) call with the same
 * n_rot and out_kind (workspaces then exist) may be captured into a CUDA graph on `stream`;
 * replaying the graph recomputes from the current contents of R (and the uploaded shapes)
 * into the same out, bitwise as an eager call.  Re-uploading a shape or changing n_rot
 * invalidates the graph (workspaces may move).
 */
bc_status bc_correlate_rotations(bc_ctx *ctx, const double *R, int64_t n_rot, int out_kind,
                                 void *out, void *stream);

/*
 * Time-critical single-configuration query: f_R(t) at n
 * arbitrary configurations (R_q, t_q), off the translation grid, evaluated EXACTLY as the
 * pair-lens sum of the combinatorial route (eq_ORP / eq_convgP) over the pairs
 * that overlap (uniform grid of A's centres); fp64, any mode.  The spectral grid of
 * bc_correlate_rotations approximates the same f within its band error.
 *   R:   host or device, n row-major 3x3 doubles (validated as for bc_correlate_rotations:
 *        host arrays at once, device arrays on the device with a deferred BC_EINVAL).
 *   t:   host or device, n x 3 doubles (finite; same rule).
 *   out: host or device, n doubles (REAL weights) or 2n interleaved (COMPLEX: Re, Im).
 * Device R, t and out: asynchronous on `stream`; host out: returns after the values are
 * written.
 */
bc_status bc_evaluate_points(bc_ctx *ctx, const double *R, const double *t, int64_t n, double *out,
                             void *stream);

/*
 * The paper's time-critical single-configuration query (PAPER.md L432-L439 eq_single, "a
 * spiral traversal of the frequency grid starting from the dominant modes"; accuracy vs
 * time L539-L546): by Parseval, f_R(t) evaluated in the frequency domain over a truncated
 * set of m' modes,
 *     f_m'(t) = (1/P^3) sum_{k in S_m'} A_hat(k) B_hat_R(-k) e^{2 pi i k . t / P},
 * with A_hat the band spectrum of bc_spectrum_A and B_hat_R the direct NDFT of the rotated
 * knots times the ball transform (eq_rhoPhat / eq_fballhat).  S_m' = the first m' band modes
 * (|k_i| <= K) in radial-shell order (|k|^2, then kx, ky, kz), a mode and its mirror -k kept
 * together for real weights (so m' counts them both).  Cost linear in m' x n_B per query.
 * With m' = all modes of |k| <= rho it equals the band-limited f of the spherical band; with
 * m' = (2K + 1)^3 it equals the spectral grid of bc_correlate_rotations at grid points.
 *   R, t, out: as bc_evaluate_points (host or device; device R / t validated on the device).
 *   m_prime:   1 <= m' <= min((2K + 1)^3, 2^22), else BC_ERANGE.
 * Spectral mode only (BC_EUNSUPPORTED); needs bc_spectrum_A (BC_ESTATE).  The first call for
 * a larger m' (or after an upload / a new spectrum) builds the mode list on the host and
 * synchronises `stream` once; later calls are asynchronous for device buffers.
 */
bc_status bc_evaluate_points_spectral(bc_ctx *ctx, const double *R, const double *t, int64_t n, int64_t m_prime,
                                      double *out, void *stream);

/*
 * Fused exchanges over peer memory for rotation-sharded multi-GPU runs (one process per GPU
 * of an NVLink / NVSwitch box).  The caller moves 64-byte IPC handles
 * between its processes (e.g. torch.distributed all_gather_object) and orders the steps with
 * its own barriers; the library does the data movement inside its kernels.
 *
 * bc_ipc_handle / bc_ipc_open / bc_ipc_close: cudaIpcGetMemHandle / cudaIpcOpenMemHandle
 *   (peer access enabled lazily) / cudaIpcCloseMemHandle of a device allocation of the
 *   calling process (handle: BC_IPC_HANDLE_BYTES bytes).  dev_ptr must be the BASE of its
 *   allocation (a handle maps the whole allocation): BC_EINVAL otherwise -- pass the
 *   context's own buffers (bc_spectrum_A_partial_buffer, bc_result_buffer).
 *
 * bc_result_buffer(ctx, bytes, dev_ptr): a context-owned device buffer of at least `bytes`
 *   (zeroed when first allocated or grown), for the job-wide records of bc_set_result_peers.
 *
 * A's spectrum sharded by balls (rho_hat_A is linear in the knots):
 *   bc_spectrum_A_partial(ctx, lo, hi, stream): the band spectrum of A's balls [lo, hi) (A is
 *     uploaded whole on every rank) into the context's PARTIAL buffer
 *     (bc_spectrum_A_partial_buffer: device pointer and bytes, owned by the context).
 *     Synchronises `stream` once (the slice's candidate lists are built on the host).
 *   bc_spectrum_A_reduce(ctx, partials, n, stream): partials[0..n) are the partial buffers of
 *     all n ranks in rank order (this rank's own and peers' mapped ones, n <= BC_MAX_PEERS);
 *     one kernel reads them all over NVLink, sums them in that order (every rank gets the same
 *     bits) and writes this rank's A spectrum and the A'' layout the fold consumes -- the
 *     all-reduce fused into the A'' build.  Needs both shapes uploaded.  Asynchronous on
 *     `stream`; the caller keeps every partial intact until all ranks' reduce kernels are done.
 *
 * bc_set_result_peers(ctx, buffers, n, base): from now on the reduction outputs of
 *   bc_correlate_rotations (spectral mode) are also stored by the epilogue kernel into each of
 *   buffers[0..n) (bc_extremum arrays of the whole job's rotations, e.g. peers' mapped
 *   buffers), at global rotation index base + (index within the call) -- the all-gather of
 *   the per-rotation results fused into a7.  n = 0 turns it off.
 */
#define BC_IPC_HANDLE_BYTES 64
#define BC_MAX_PEERS 8
bc_status bc_ipc_handle(bc_ctx *ctx, const void *dev_ptr, void *handle);
bc_status bc_ipc_open(bc_ctx *ctx, const void *handle, void **dev_ptr);
bc_status bc_ipc_close(bc_ctx *ctx, void *dev_ptr);
bc_status bc_spectrum_A_partial(bc_ctx *ctx, int64_t lo, int64_t hi, void *stream);
bc_status bc_spectrum_A_partial_buffer(bc_ctx *ctx, void **dev_ptr, int64_t *bytes);
bc_status bc_spectrum_A_reduce(bc_ctx *ctx, const void *const *partials, int n, void *stream);
bc_status bc_result_buffer(bc_ctx *ctx, int64_t bytes, void **dev_ptr);
bc_status bc_set_result_peers(bc_ctx *ctx, void *const *buffers, int n, int64_t base);

/* Synchronise `stream` and report a deferred error of earlier calls on this context
 * (BC_EINVAL from device-side validation of R / t, BC_ECUDA from a CUDA fault). */
bc_status bc_sync(bc_ctx *ctx, void *stream);

/* Last error message of the context (static string if ctx == NULL). */
const char *bc_last_error(const bc_ctx *ctx);
const char *bc_status_string(int status);

/*
 * Introspection (tests / bench): named double-valued properties of the plan.
 * Keys: "P", "K", "Np", "tau_A", "tau_B", "G_A", "G_B", "L_A", "L_B", "c_A", "c_B",
 * "cut_A", "cut_B", "band_modes", "batch", "bytes_workspace", "band_error" (the band-error
 * probe's estimate, -1 before it ran; see bc_params.tolerance), "query_modes" (m' the spectral
 * query's tables serve), "blob_B" (B smoothed with the
 * KB blob window), "fused_spread_z", "fused_fold_inv", "fold_fast", "dock_fast" (which fused kernels the
 * plan takes), "spread_cells_B" (sum of B's footprint volumes in fine cells), "live_tiles_B".
 * Unknown keys: BC_EINVAL.
 */
bc_status bc_query(const bc_ctx *ctx, const char *key, double *value);

/* Number of kernels this context has launched so far. */
int64_t bc_launch_count(const bc_ctx *ctx);

/*
 * Per-stage device timing: when enabled, the library records CUDA events on
 * the launching stream around every kernel of bc_correlate_rotations and
 * accumulates their durations per stage.  bc_stage_times fills up to `cap`
 * entries of names/total_ms/launches and returns the number of stages.
 */
bc_status bc_set_profiling(bc_ctx *ctx, int enabled);
int bc_stage_times(bc_ctx *ctx, const char **names, double *total_ms, int64_t *launches, int cap);
bc_status bc_reset_stage_times(bc_ctx *ctx);

#ifdef __cplusplus
}
#endif

#endif /* BALLCORR_H */
