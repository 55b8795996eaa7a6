"""CPU checks of the C ABI: the library loads, exports every symbol the header
declares, and validates parameters before touching a device (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ballcorr.h")


@pytest.fixture(scope="module")
def bc():
    lib = os.path.join(ROOT, "paper_1711_05075_b200", "lib", "libballcorr.so")
    if not os.path.exists(lib):
        import subprocess
        subprocess.check_call(["make", "-C", ROOT, "-j4"], stdout=subprocess.DEVNULL)
    from paper_1711_05075_b200 import ballcorr
    return ballcorr


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bc_[a-z_A-Z]+)\s*\(", text)))


def test_header_declares_the_path(bc):
    names = declared_functions()
    for required in ("bc_create", "bc_destroy", "bc_shape_upload", "bc_spectrum_A", "bc_correlate_rotations",
                     "bc_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(bc):
    lib = ctypes.CDLL(bc.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_status_strings(bc):
    assert bc.bc_status_string(0) == b"BC_OK"
    assert bc.bc_status_string(2) == b"BC_ERANGE"
    assert bc.bc_status_string(99) == b"BC_UNKNOWN"


def test_params_struct_layout(bc, tmp_path):
    """ctypes' bc_params agrees with the C compiler's layout of include/ballcorr.h."""
    P = bc.bc_params
    names = [f[0] for f in P._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "ballcorr.h"\nint main(void){\n' +
                   "".join(f'printf("%zu\\n", offsetof(bc_params, {n}));\n' for n in names) +
                   'printf("%zu\\n", sizeof(bc_params));return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()]
    assert got[:-1] == [getattr(P, n).offset for n in names]
    assert got[-1] == ctypes.sizeof(P)


@pytest.mark.parametrize("kw", [
    dict(N=0, h=0.1, t0=(0, 0, 0)),
    dict(N=8, h=-1.0, t0=(0, 0, 0)),
    dict(N=8, h=0.1, t0=(0, 0, 0), Np=7, K=4),          # Np odd
    dict(N=8, h=0.1, t0=(0, 0, 0), Np=14, K=4),         # 7 is not a {2,3,5} factor
    dict(N=8, h=0.1, t0=(0, 0, 0), Np=6, K=4),          # Np < N
    dict(N=8, h=0.1, t0=(0, 0, 0), Np=8, K=0),          # empty band
])
def test_create_rejects_bad_params_without_gpu(bc, kw):
    with pytest.raises(bc.BallCorrError) as e:
        bc.Correlator(**kw)
    assert e.value.status == bc.BC_EINVAL


def test_spectral_fp64_limits(bc):
    """Spectral fp64 is a small-problem parity mode (include/ballcorr.h): a band beyond K = 64,
    or the fp32-only band-error probe, is refused before any device work."""
    for kw in (dict(K=65), dict(K=4, tolerance=1e-4)):
        with pytest.raises(bc.BallCorrError) as e:
            bc.Correlator(N=8, h=0.1, t0=(0, 0, 0), Np=8, precision="f64", **kw)
        assert e.value.status == bc.BC_EUNSUPPORTED


def test_null_context_is_safe(bc):
    assert bc.bc_destroy(None) == 0
    assert bc.bc_last_error(None) == b"no context"
    assert bc.bc_launch_count(None) == 0


def test_out_buffers_are_checked_not_copied(bc):
    """ballcorr._out_ptr: a caller's `out` must hold the bytes the call writes, be
    C-contiguous, and have the result dtype or raw bytes; it is never silently replaced by a
    contiguous copy (the library would write into a temporary)."""
    import numpy as np
    import torch
    f32 = np.float32
    assert bc._out_ptr(np.empty((2, 4, 4, 4), f32), 2 * 64 * 4, f32) > 0
    assert bc._out_ptr(np.empty(512, np.uint8), 512, f32) > 0
    assert bc._out_ptr(torch.empty(512, dtype=torch.uint8), 512, f32) > 0
    assert bc._out_ptr(torch.empty((2, 64), dtype=torch.float32), 512, f32) > 0
    bad = [
        (np.empty((2, 4, 4, 3), f32), 2 * 64 * 4, f32),            # too small
        (np.empty((4, 4, 8), f32)[:, :, ::2], 64 * 4, f32),        # not contiguous
        (np.empty(128, np.float64), 512, f32),                      # wrong dtype
        (torch.empty((8, 16), dtype=torch.float32).t(), 512, f32),  # non-contiguous tensor
        (torch.empty(100, dtype=torch.uint8), 512, f32),           # too small tensor
        ([0.0] * 128, 512, f32),                                    # not an array
    ]
    for out, nbytes, dt in bad:
        with pytest.raises(ValueError):
            bc._out_ptr(out, nbytes, dt)
    ext = np.empty(3, bc.EXTREMUM_DTYPE)
    assert bc._out_ptr(ext, 3 * 16, bc.EXTREMUM_DTYPE) > 0
    with pytest.raises(ValueError):
        bc._out_ptr(np.empty(2, bc.EXTREMUM_DTYPE), 3 * 16, bc.EXTREMUM_DTYPE)
