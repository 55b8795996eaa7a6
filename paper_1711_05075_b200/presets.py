"""Per-workload parameters of the correlator (mode, FFT period, band).

Chosen from the band-error measurements recorded in DESIGN.md §5 (spectral f at
several bands against the exact pair-lens f, which tests pin to the fp64
oracle): the smallest band whose error stays well inside the north_star
tolerance max|f_gpu - f_cpu| <= 1e-4 max|f_cpu|.

* tiny    exact mode, fp64 (the 1e-9 bar is unreachable for any band limit)
* single  exact mode, fp32 (0.01-radius balls need sigma_f ~ 8 spectrally; exact is cheaper)
* torus   spectral, Np = 144 (P = 2.25), K = 71: 2.2e-5 measured
* sweep   spectral, Np = 256 (P = 2), K = 255: 3.8e-5 measured (K = 191: 7.4e-5)
* docking spectral, Np = 128 (P = 128 A), K = 191: 5.2e-5 measured (K = 127: 1.3e-4 fails)
"""
from __future__ import annotations

PRESETS = {
    "tiny": dict(mode="exact", precision="f64", Np=0, K=0),
    "single": dict(mode="exact", precision="f32", Np=0, K=0),
    "torus": dict(mode="spectral", precision="f32", Np=144, K=71),
    "sweep": dict(mode="spectral", precision="f32", Np=256, K=255),
    "docking": dict(mode="spectral", precision="f32", Np=128, K=191),
}


def correlator_kwargs(name: str, N: int, h: float, t0, weights: str, **overrides) -> dict:
    p = dict(PRESETS[name])
    p.update(overrides)
    return dict(N=N, h=h, t0=t0, Np=p["Np"], K=p["K"], mode=p["mode"], precision=p["precision"],
                weights=weights, max_batch=p.get("max_batch", 0), spread_eps=p.get("spread_eps", 0.0),
                generic_only=p.get("generic_only", False), concurrency=p.get("concurrency", 0),
                tolerance=p.get("tolerance", 0.0))


def choose_band(name: str, N: int, h: float, t0, weights: str, A, wA, B, wB, tol: float = 5e-5,
                K_max: int = 2047, growth: float = 1.25, device: int = 0, **overrides) -> dict:
    """(Correlator kwargs, band-error estimate): a band K meeting a requested tolerance for
    THESE shapes.

    Starts at the preset's K and widens it by `growth` until the library's band-error guard
    (bc_params.tolerance: two probe rotations of the spectral grid against the exact pair-lens
    f at sampled translations) accepts it; raises BallCorrError(BC_ERANGE) past K_max.  Exact
    mode needs no band and is returned unchanged.  The default 5e-5 keeps a 2x margin under the
    north_star 1e-4 for the translations and rotations the probe did not sample."""
    from .ballcorr import Correlator, BallCorrError, BC_ERANGE
    kw = correlator_kwargs(name, N, h, t0, weights, **overrides)
    if kw["mode"] != "spectral":
        return kw, 0.0
    K = kw["K"]
    last = None
    while K <= K_max:
        kw.update(K=K, tolerance=tol)
        c = Correlator(device=device, **kw)
        try:
            c.shape_upload(0, A, wA)  # errors here (support wrap, no box) are not band errors
            c.shape_upload(1, B, wB)
            c.spectrum_A()
            try:
                c.correlate_rotations([[[1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0]]],
                                      "full" if weights == "complex" else "max_argmax")
                return kw, c.query("band_error")
            except BallCorrError as e:
                if e.status != BC_ERANGE:
                    raise
                last = e
        finally:
            c.close()
        K = int(K * growth) + 1
    raise last
