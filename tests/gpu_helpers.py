"""Shared helpers of the -m gpu parity tests (no method arithmetic here)."""
import numpy as np


def rel_max_err(got, ref):
    ref = np.asarray(ref)
    return float(np.abs(np.asarray(got) - ref).max() / max(np.abs(ref).max(), 1e-300))


def as_complex(full):
    """(…, 2) float array of interleaved (re, im) -> complex."""
    return full[..., 0] + 1j * full[..., 1]


def check_extremum(val, idx, f_ref, kind, tol_abs):
    """Reading C-10: values within tolerance of the oracle extremum, and the GPU index
    must point at a grid value (oracle) within tolerance of that extremum; index
    equality is not required."""
    flat = np.asarray(f_ref).reshape(-1)
    ext = flat.min() if kind == "min" else flat.max()
    assert abs(val - ext) <= tol_abs, (kind, val, ext)
    assert abs(flat[idx] - ext) <= 2 * tol_abs, (kind, idx, flat[idx], ext)
