"""Thin ctypes binding of libballcorr.so (include/ballcorr.h).

Argument marshalling only: every step of the correlation runs in the CUDA
kernels behind the C ABI.  If the shared library is missing this module
raises at import time; there is no CPU fallback.

The C entry points are re-exported under their own names (`bc_create`,
`bc_shape_upload`, `bc_spectrum_A`, `bc_correlate_rotations`, ...);
`Correlator` wraps them for numpy / torch callers.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BALLCORR_LIB: an alternative in-tree build (development A/B timing); default lib/libballcorr.so
LIB_PATH = os.environ.get("BALLCORR_LIB") or os.path.join(_HERE, "lib", "libballcorr.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libballcorr.so not found at {LIB_PATH}: build it with `make` (or __graft_entry__.build()). "
        "There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

BC_OK, BC_EINVAL, BC_ERANGE, BC_ENOMEM, BC_ESTATE, BC_EUNSUPPORTED, BC_ECUDA = range(7)
BC_FP32, BC_FP64 = 0, 1
BC_MODE_SPECTRAL, BC_MODE_EXACT = 0, 1
BC_WEIGHTS_REAL, BC_WEIGHTS_COMPLEX = 0, 1
BC_OUT_F_FULL, BC_OUT_MIN_ARGMIN, BC_OUT_MAX_ARGMAX, BC_OUT_MINMAX, BC_OUT_MAX_REAL = range(5)

OUT_KINDS = {"full": BC_OUT_F_FULL, "min_argmin": BC_OUT_MIN_ARGMIN, "max_argmax": BC_OUT_MAX_ARGMAX,
             "minmax": BC_OUT_MINMAX, "max_real": BC_OUT_MAX_REAL}


class bc_params(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("h", ctypes.c_double), ("t0", ctypes.c_double * 3),
                ("Np", ctypes.c_int32), ("K", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("weights", ctypes.c_int32), ("max_batch", ctypes.c_int32),
                ("spread_eps", ctypes.c_double), ("band_radius", ctypes.c_double),
                ("generic_only", ctypes.c_int32), ("concurrency", ctypes.c_int32),
                ("tolerance", ctypes.c_double)]


EXTREMUM_DTYPE = np.dtype([("val", np.float64), ("idx", np.int64)])

_vp = ctypes.c_void_p
_lib.bc_create.argtypes = [ctypes.c_int, ctypes.POINTER(bc_params), ctypes.POINTER(_vp)]
_lib.bc_create.restype = ctypes.c_int
_lib.bc_destroy.argtypes = [_vp]
_lib.bc_destroy.restype = ctypes.c_int
_lib.bc_shape_upload.argtypes = [_vp, ctypes.c_int, _vp, _vp, ctypes.c_int64]
_lib.bc_shape_upload.restype = ctypes.c_int
_lib.bc_spectrum_A.argtypes = [_vp, _vp]
_lib.bc_spectrum_A.restype = ctypes.c_int
_lib.bc_spectrum_A_buffer.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int64)]
_lib.bc_spectrum_A_buffer.restype = ctypes.c_int
_lib.bc_spectrum_A_import.argtypes = [_vp]
_lib.bc_spectrum_A_import.restype = ctypes.c_int
_lib.bc_correlate_rotations.argtypes = [_vp, _vp, ctypes.c_int64, ctypes.c_int, _vp, _vp]
_lib.bc_correlate_rotations.restype = ctypes.c_int
_lib.bc_evaluate_points.argtypes = [_vp, _vp, _vp, ctypes.c_int64, _vp, _vp]
_lib.bc_evaluate_points.restype = ctypes.c_int
_lib.bc_evaluate_points_spectral.argtypes = [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp]
_lib.bc_evaluate_points_spectral.restype = ctypes.c_int
_lib.bc_ipc_handle.argtypes = [_vp, _vp, _vp]
_lib.bc_ipc_handle.restype = ctypes.c_int
_lib.bc_ipc_open.argtypes = [_vp, _vp, ctypes.POINTER(_vp)]
_lib.bc_ipc_open.restype = ctypes.c_int
_lib.bc_ipc_close.argtypes = [_vp, _vp]
_lib.bc_ipc_close.restype = ctypes.c_int
_lib.bc_spectrum_A_partial.argtypes = [_vp, ctypes.c_int64, ctypes.c_int64, _vp]
_lib.bc_spectrum_A_partial.restype = ctypes.c_int
_lib.bc_spectrum_A_partial_buffer.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int64)]
_lib.bc_spectrum_A_partial_buffer.restype = ctypes.c_int
_lib.bc_spectrum_A_reduce.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.c_int, _vp]
_lib.bc_spectrum_A_reduce.restype = ctypes.c_int
_lib.bc_result_buffer.argtypes = [_vp, ctypes.c_int64, ctypes.POINTER(_vp)]
_lib.bc_result_buffer.restype = ctypes.c_int
_lib.bc_set_result_peers.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.c_int, ctypes.c_int64]
_lib.bc_set_result_peers.restype = ctypes.c_int
_lib.bc_sync.argtypes = [_vp, _vp]
_lib.bc_sync.restype = ctypes.c_int
_lib.bc_last_error.argtypes = [_vp]
_lib.bc_last_error.restype = ctypes.c_char_p
_lib.bc_status_string.argtypes = [ctypes.c_int]
_lib.bc_status_string.restype = ctypes.c_char_p
_lib.bc_query.argtypes = [_vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double)]
_lib.bc_query.restype = ctypes.c_int
_lib.bc_launch_count.argtypes = [_vp]
_lib.bc_launch_count.restype = ctypes.c_int64
_lib.bc_set_profiling.argtypes = [_vp, ctypes.c_int]
_lib.bc_set_profiling.restype = ctypes.c_int
_lib.bc_stage_times.argtypes = [_vp, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
_lib.bc_stage_times.restype = ctypes.c_int
_lib.bc_reset_stage_times.argtypes = [_vp]
_lib.bc_reset_stage_times.restype = ctypes.c_int

# the C names, re-exported
bc_create = _lib.bc_create
bc_destroy = _lib.bc_destroy
bc_shape_upload = _lib.bc_shape_upload
bc_spectrum_A = _lib.bc_spectrum_A
bc_spectrum_A_buffer = _lib.bc_spectrum_A_buffer
bc_spectrum_A_import = _lib.bc_spectrum_A_import
bc_correlate_rotations = _lib.bc_correlate_rotations
bc_evaluate_points_spectral = _lib.bc_evaluate_points_spectral
bc_sync = _lib.bc_sync
bc_ipc_handle = _lib.bc_ipc_handle
bc_ipc_open = _lib.bc_ipc_open
bc_ipc_close = _lib.bc_ipc_close
bc_spectrum_A_partial = _lib.bc_spectrum_A_partial
bc_spectrum_A_partial_buffer = _lib.bc_spectrum_A_partial_buffer
bc_spectrum_A_reduce = _lib.bc_spectrum_A_reduce
bc_set_result_peers = _lib.bc_set_result_peers
bc_result_buffer = _lib.bc_result_buffer
IPC_HANDLE_BYTES = 64
MAX_PEERS = 8
bc_last_error = _lib.bc_last_error
bc_status_string = _lib.bc_status_string
bc_query = _lib.bc_query
bc_launch_count = _lib.bc_launch_count
bc_set_profiling = _lib.bc_set_profiling
bc_stage_times = _lib.bc_stage_times
bc_reset_stage_times = _lib.bc_reset_stage_times


class BallCorrError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"{_lib.bc_status_string(status).decode()}: {msg}")


def _ptr(a):
    """(address, keepalive) of a numpy array or torch tensor (host or device)."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr"):  # torch tensor
        if not a.is_contiguous():
            a = a.contiguous()
        return a.data_ptr(), a
    a = np.ascontiguousarray(a)
    return a.ctypes.data, a


def _out_ptr(out, nbytes, dtype, what="out"):
    """Address of a caller-provided output buffer after checking it can hold `nbytes`: a
    C-contiguous numpy array or torch tensor (host or cuda) of the result dtype (`dtype`) or
    of raw bytes (uint8).  Never copies: the library writes into `out` itself."""
    if hasattr(out, "data_ptr"):  # torch tensor
        import torch
        if not out.is_contiguous():
            raise ValueError(f"{what} must be contiguous")
        size = out.numel() * out.element_size()
        ok_dt = out.dtype == torch.uint8 or (out.element_size() == np.dtype(dtype).itemsize and
                                              out.dtype.is_floating_point == (np.dtype(dtype).kind == "f"))
        ptr = out.data_ptr()
    else:
        if not isinstance(out, np.ndarray):
            raise ValueError(f"{what} must be a numpy array or a torch tensor")
        if not out.flags.c_contiguous or not out.flags.writeable:
            raise ValueError(f"{what} must be C-contiguous and writeable")
        size = out.nbytes
        ok_dt = out.dtype == np.uint8 or out.dtype == np.dtype(dtype)
        ptr = out.ctypes.data
    if not ok_dt:
        raise ValueError(f"{what} has dtype {out.dtype}; expected {np.dtype(dtype)} or uint8 bytes")
    if size < nbytes:
        raise ValueError(f"{what} holds {size} bytes; the call writes {nbytes}")
    return ptr


def _as_f64(a, cols=None):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        import torch
        return a.to(torch.float64).contiguous()
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _weights_f64(w, complex_w):
    if w is None:
        return None
    if hasattr(w, "data_ptr"):
        import torch
        if complex_w:
            return torch.view_as_real(w.to(torch.complex128).contiguous()).contiguous()
        return w.to(torch.float64).contiguous()
    w = np.asarray(w)
    if complex_w:
        w = np.ascontiguousarray(w, dtype=np.complex128).view(np.float64)
    else:
        w = np.ascontiguousarray(w, dtype=np.float64)
    return w


def _stream_handle(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


class Correlator:
    """One libballcorr context on one device."""

    def __init__(self, N, h, t0, Np=0, K=0, mode="spectral", precision="f32", weights="real",
                 max_batch=0, spread_eps=0.0, band_radius=0.0, generic_only=False, concurrency=0, tolerance=0.0,
                 device=0):
        p = bc_params()
        p.N = int(N)
        p.h = float(h)
        for i in range(3):
            p.t0[i] = float(t0[i])
        p.Np = int(Np)
        p.K = int(K)
        p.precision = BC_FP64 if precision in ("f64", "fp64", BC_FP64) else BC_FP32
        p.mode = BC_MODE_EXACT if mode in ("exact", BC_MODE_EXACT) else BC_MODE_SPECTRAL
        p.weights = BC_WEIGHTS_COMPLEX if weights in ("complex", BC_WEIGHTS_COMPLEX) else BC_WEIGHTS_REAL
        p.max_batch = int(max_batch)
        p.spread_eps = float(spread_eps)
        p.band_radius = float(band_radius)
        p.generic_only = int(bool(generic_only))
        p.concurrency = int(concurrency)
        p.tolerance = float(tolerance)
        self.params = p
        self.device = int(device)
        self.N = p.N
        self.complex = p.weights == BC_WEIGHTS_COMPLEX
        self.f64 = p.precision == BC_FP64
        self._ctx = _vp()
        st = _lib.bc_create(int(device), ctypes.byref(p), ctypes.byref(self._ctx))
        if st != BC_OK:
            raise BallCorrError(st, "bc_create failed")

    # -- error helper
    def _check(self, st):
        if st != BC_OK:
            raise BallCorrError(st, _lib.bc_last_error(self._ctx).decode())

    def close(self):
        if self._ctx:
            _lib.bc_destroy(self._ctx)
            self._ctx = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the three calls of the path
    def shape_upload(self, which, xyzr, w=None):
        x = _as_f64(xyzr)
        n = int(x.shape[0]) if x is not None else 0
        wv = _weights_f64(w, self.complex)
        px, kx = _ptr(x)
        pw, kw = _ptr(wv)
        self._check(_lib.bc_shape_upload(self._ctx, int(which), px, pw, n))

    def spectrum_A(self, stream=None):
        self._check(_lib.bc_spectrum_A(self._ctx, _stream_handle(stream)))

    def spectrum_A_buffer(self):
        """(device pointer, bytes) of the buffer holding A's band spectrum (owned by the context)."""
        ptr, nbytes = _vp(), ctypes.c_int64()
        self._check(_lib.bc_spectrum_A_buffer(self._ctx, ctypes.byref(ptr), ctypes.byref(nbytes)))
        return int(ptr.value), int(nbytes.value)

    def spectrum_A_tensor(self):
        """The same buffer as a float32 torch tensor on the context's device (zero copy, via the
        CUDA array interface) -- for a torch.distributed broadcast of A's spectrum."""
        import torch
        ptr, nbytes = self.spectrum_A_buffer()

        class _Iface:
            __cuda_array_interface__ = {"shape": (nbytes // 4,), "typestr": "<f4", "data": (ptr, False),
                                        "version": 3, "strides": None}
        return torch.as_tensor(_Iface(), device=torch.device("cuda", self.device))

    def spectrum_A_import(self):
        """Declare the buffer's contents (written by the caller) to be A's spectrum."""
        self._check(_lib.bc_spectrum_A_import(self._ctx))

    # -- fused exchanges over peer memory (include/ballcorr.h; sharding.py drives them)
    def ipc_handle(self, dev_ptr):
        """64-byte cudaIpc handle (bytes) of a device allocation of this process."""
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        self._check(_lib.bc_ipc_handle(self._ctx, dev_ptr, buf))
        return buf.raw

    def ipc_open(self, handle):
        """Map a peer's allocation; returns its device pointer in this process."""
        ptr = _vp()
        buf = ctypes.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES)
        self._check(_lib.bc_ipc_open(self._ctx, buf, ctypes.byref(ptr)))
        return int(ptr.value)

    def ipc_close(self, dev_ptr):
        self._check(_lib.bc_ipc_close(self._ctx, dev_ptr))

    def spectrum_A_partial(self, lo, hi, stream=None):
        """Band spectrum of A's balls [lo, hi) into the context's partial buffer."""
        self._check(_lib.bc_spectrum_A_partial(self._ctx, int(lo), int(hi), _stream_handle(stream)))

    def spectrum_A_partial_buffer(self):
        ptr, nbytes = _vp(), ctypes.c_int64()
        self._check(_lib.bc_spectrum_A_partial_buffer(self._ctx, ctypes.byref(ptr), ctypes.byref(nbytes)))
        return int(ptr.value), int(nbytes.value)

    def spectrum_A_reduce(self, partial_ptrs, stream=None):
        """A's spectrum = the sum of the ranks' partial spectra (device pointers, rank order),
        read over peer memory by one kernel fused with the A'' build."""
        arr = (_vp * len(partial_ptrs))(*[int(p) for p in partial_ptrs])
        self._check(_lib.bc_spectrum_A_reduce(self._ctx, arr, len(partial_ptrs), _stream_handle(stream)))

    def result_buffer(self, nbytes):
        """(device pointer, torch uint8 tensor view) of the context-owned job-wide record buffer
        (an allocation base, so it can be exported with ipc_handle)."""
        import torch
        ptr = _vp()
        self._check(_lib.bc_result_buffer(self._ctx, int(nbytes), ctypes.byref(ptr)))

        class _Iface:
            __cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr.value), False),
                                        "version": 3, "strides": None}
        return int(ptr.value), torch.as_tensor(_Iface(), device=torch.device("cuda", self.device))

    def set_result_peers(self, buffers, base=0):
        """Reduction records of later correlate calls also go to these device buffers at global
        rotation index base + i (the fused result exchange); [] turns it off."""
        arr = (_vp * max(len(buffers), 1))(*[int(p) for p in buffers])
        self._check(_lib.bc_set_result_peers(self._ctx, arr, len(buffers), int(base)))

    def out_shape(self, n_rot, out_kind):
        kind = OUT_KINDS.get(out_kind, out_kind)
        if kind == BC_OUT_F_FULL:
            shp = (n_rot, self.N, self.N, self.N) + ((2,) if self.complex else ())
            return kind, shp, (np.float64 if self.f64 else np.float32)
        return kind, (n_rot, 2) if kind == BC_OUT_MINMAX else (n_rot,), EXTREMUM_DTYPE

    def correlate_rotations(self, R, out_kind="full", out=None, stream=None):
        """R: (n_rot, 3, 3) host numpy / torch (host or cuda).  `out`: optional preallocated
        numpy array or torch tensor (host or cuda) of the right byte size.  Returns `out`
        (numpy structured array for reductions when allocated here)."""
        Rv = _as_f64(R)
        if tuple(Rv.shape[1:]) != (3, 3) and not (Rv.ndim == 2 and Rv.shape[1] == 9):
            raise ValueError("R must have shape (n_rot, 3, 3)")
        n_rot = int(Rv.shape[0])
        kind, shp, dt = self.out_shape(n_rot, out_kind)
        if out is None:
            out = np.empty(shp, dtype=dt)
        po = _out_ptr(out, int(np.prod(shp)) * np.dtype(dt).itemsize, dt)
        pr, kr = _ptr(Rv)
        self._check(_lib.bc_correlate_rotations(self._ctx, pr, n_rot, kind, po, _stream_handle(stream)))
        return out

    def evaluate_points(self, R, t, out=None, stream=None):
        """f_R(t) at n arbitrary configurations (exact pair-lens sum, fp64): R (n, 3, 3) and
        t (n, 3), host numpy / torch (host or cuda).  Returns float64 (n,) or complex128 (n,)
        when allocated here; `out` may be a preallocated float64 buffer (n or (n, 2))."""
        Rv = _as_f64(R)
        tv = _as_f64(t)
        n = int(Rv.shape[0])
        if tuple(tv.shape) != (n, 3):
            raise ValueError("t must have shape (n, 3)")
        ret_complex = out is None and self.complex
        if out is None:
            out = np.empty((n, 2) if self.complex else (n,), dtype=np.float64)
        po = _out_ptr(out, n * (2 if self.complex else 1) * 8, np.float64)
        pr, kr = _ptr(Rv)
        pt, kt = _ptr(tv)
        self._check(_lib.bc_evaluate_points(self._ctx, pr, pt, n, po, _stream_handle(stream)))
        return out[:, 0] + 1j * out[:, 1] if ret_complex else out

    def evaluate_points_spectral(self, R, t, m_prime, out=None, stream=None):
        """The paper's truncated-Parseval query: f_R(t) over the first
        m_prime band modes in radial-shell order.  Same arguments and results as
        evaluate_points."""
        Rv = _as_f64(R)
        tv = _as_f64(t)
        n = int(Rv.shape[0])
        if tuple(tv.shape) != (n, 3):
            raise ValueError("t must have shape (n, 3)")
        ret_complex = out is None and self.complex
        if out is None:
            out = np.empty((n, 2) if self.complex else (n,), dtype=np.float64)
        po = _out_ptr(out, n * (2 if self.complex else 1) * 8, np.float64)
        pr, kr = _ptr(Rv)
        pt, kt = _ptr(tv)
        self._check(_lib.bc_evaluate_points_spectral(self._ctx, pr, pt, n, int(m_prime), po, _stream_handle(stream)))
        return out[:, 0] + 1j * out[:, 1] if ret_complex else out

    # -- introspection / profiling
    def query(self, key):
        v = ctypes.c_double()
        self._check(_lib.bc_query(self._ctx, key.encode(), ctypes.byref(v)))
        return v.value

    def sync(self, stream=None):
        """bc_sync: wait for `stream` and raise a deferred error of earlier calls (BC_EINVAL from
        on-device validation of device-resident R / t)."""
        self._check(_lib.bc_sync(self._ctx, _stream_handle(stream)))

    def launch_count(self):
        return int(_lib.bc_launch_count(self._ctx))

    def set_profiling(self, on=True):
        self._check(_lib.bc_set_profiling(self._ctx, 1 if on else 0))

    def reset_stage_times(self):
        self._check(_lib.bc_reset_stage_times(self._ctx))

    def stage_times(self):
        cap = 64
        names = (ctypes.c_char_p * cap)()
        ms = (ctypes.c_double * cap)()
        cnt = (ctypes.c_int64 * cap)()
        n = _lib.bc_stage_times(self._ctx, names, ms, cnt, cap)
        return {names[i].decode(): (ms[i], int(cnt[i])) for i in range(min(n, cap))}


def extremum_to_numpy(buf):
    """View a torch uint8/float buffer holding bc_extremum records as a numpy structured array."""
    return np.frombuffer(bytes(buf), dtype=EXTREMUM_DTYPE)
