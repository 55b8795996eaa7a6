"""ctypes front-end of oracle/lens_oracle.c (TEST INFRASTRUCTURE ONLY).

The C file is compiled here with the system gcc (`build_oracle`).  Nothing in
this module touches the CUDA library.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lens_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build_oracle(force: bool = False) -> str:
    """Compile lens_oracle.c -> liboracle.so (gcc, OpenMP, -O2, strict IEEE: no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c99",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_lens_volume.restype = ctypes.c_double
        lib.oracle_lens_volume.argtypes = [ctypes.c_double] * 3
        lib.oracle_num_threads.restype = ctypes.c_int
        common = [_dp, _dp, _dp, ctypes.c_int64, _dp, _dp, _dp, ctypes.c_int64,
                  _dp, ctypes.c_int64, ctypes.c_double, _dp]
        lib.oracle_correlate_grid.restype = None
        lib.oracle_correlate_grid.argtypes = common + [_i64p, _i64p, _dp, _dp]
        lib.oracle_correlate_points.restype = None
        lib.oracle_correlate_points.argtypes = common + [_i64p, ctypes.c_int64, _dp, _dp]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _split_weights(w, n):
    if w is None:
        return None, None
    w = np.asarray(w)
    if np.iscomplexobj(w):
        return (np.ascontiguousarray(w.real, dtype=np.float64),
                np.ascontiguousarray(w.imag, dtype=np.float64))
    return np.ascontiguousarray(w, dtype=np.float64), None


def oracle_threads() -> int:
    return int(_load().oracle_num_threads())


def lens_volume(r: float, s: float, d: float) -> float:
    """V(r, s, d): volume of B(0, r) intersected with B(d e, s) (closed form)."""
    return float(_load().oracle_lens_volume(float(r), float(s), float(d)))


def _prep(A, wA, B, wB, R):
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    R = np.ascontiguousarray(np.asarray(R, dtype=np.float64).reshape(9))
    war, wai = _split_weights(wA, len(A))
    wbr, wbi = _split_weights(wB, len(B))
    cplx = wai is not None or wbi is not None
    return A, war, wai, B, wbr, wbi, R, cplx


def correlate_grid(A, wA, B, wB, R, N, h, t0, lo=(0, 0, 0), hi=None):
    """f_R on the N^3 grid (or the sub-box [lo, hi)); returns float64 or complex128
    array of shape (N, N, N) (entries outside the sub-box are 0)."""
    A, war, wai, B, wbr, wbi, R, cplx = _prep(A, wA, B, wB, R)
    hi = (N, N, N) if hi is None else hi
    out_re = np.zeros(N ** 3)
    out_im = np.zeros(N ** 3) if cplx else None
    t0a = np.ascontiguousarray(t0, dtype=np.float64)
    lo_a = np.ascontiguousarray(lo, dtype=np.int64)
    hi_a = np.ascontiguousarray(hi, dtype=np.int64)
    _load().oracle_correlate_grid(
        _ptr(A), _ptr(war), _ptr(wai), len(A), _ptr(B), _ptr(wbr), _ptr(wbi), len(B),
        _ptr(R), int(N), float(h), _ptr(t0a), lo_a.ctypes.data_as(_i64p),
        hi_a.ctypes.data_as(_i64p), _ptr(out_re), _ptr(out_im))
    out = out_re if not cplx else out_re + 1j * out_im
    return out.reshape(N, N, N)


def correlate_points(A, wA, B, wB, R, N, h, t0, flat_idx):
    """f_R at flat C-order grid indices, brute force over every pair."""
    A, war, wai, B, wbr, wbi, R, cplx = _prep(A, wA, B, wB, R)
    idx = np.ascontiguousarray(flat_idx, dtype=np.int64)
    out_re = np.zeros(len(idx))
    out_im = np.zeros(len(idx)) if cplx else None
    t0a = np.ascontiguousarray(t0, dtype=np.float64)
    _load().oracle_correlate_points(
        _ptr(A), _ptr(war), _ptr(wai), len(A), _ptr(B), _ptr(wbr), _ptr(wbi), len(B),
        _ptr(R), int(N), float(h), _ptr(t0a), idx.ctypes.data_as(_i64p), len(idx),
        _ptr(out_re), _ptr(out_im))
    return out_re if not cplx else out_re + 1j * out_im
