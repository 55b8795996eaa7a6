"""Exact (pair-lens) mode on the GPU vs the fp64 lens oracle.

Tolerances (north_star): max|f_gpu - f_cpu| <= 1e-9 max|f_cpu| in fp64 mode and
1e-4 max|f_cpu| in fp32 mode (fp32 lens evaluation, fp64 accumulation: ~1e-6).
"""
import numpy as np
import pytest

from synth import make_config, random_small_case, random_rotations
from gpu_helpers import rel_max_err, as_complex, check_extremum

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bc():
    import torch
    assert torch.cuda.is_available()
    from paper_1711_05075_b200 import ballcorr
    return ballcorr


def make_exact(bc, w, precision=None):
    c = bc.Correlator(N=w.N, h=w.h, t0=w.t0, mode="exact", precision=precision or w.precision,
                      weights=w.weights)
    c.shape_upload(0, w.A_xyzr, w.A_w)
    c.shape_upload(1, w.B_xyzr, w.B_w)
    c.spectrum_A()
    return c


def test_tiny_fp64_full_grid(bc, oracle_mod):
    w = make_config("tiny")
    c = make_exact(bc, w)
    f = c.correlate_rotations(w.R, "full")
    ref = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], w.N, w.h, w.t0)
    assert f.dtype == np.float64
    assert rel_max_err(f[0], ref) <= 1e-9
    assert c.launch_count() >= 2


def test_tiny_fp64_rotated_and_reductions(bc, oracle_mod):
    w = make_config("tiny")
    R = random_rotations(np.random.default_rng(3), 3)
    c = make_exact(bc, w)
    f = c.correlate_rotations(R, "full")
    mm = c.correlate_rotations(R, "minmax")
    for r in range(3):
        ref = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, R[r], w.N, w.h, w.t0)
        assert rel_max_err(f[r], ref) <= 1e-9
        tol = 1e-9 * np.abs(ref).max()
        check_extremum(mm[r, 0]["val"], mm[r, 0]["idx"], ref, "min", tol)
        check_extremum(mm[r, 1]["val"], mm[r, 1]["idx"], ref, "max", tol)
        # exact ties at the minimum (f == 0 far from the obstacle): lowest index
        flat = ref.reshape(-1)
        if np.count_nonzero(flat == flat.min()) > 1:
            assert mm[r, 0]["idx"] == int(np.flatnonzero(f[r].reshape(-1) == f[r].min())[0])


def test_single_fp32_full_grid(bc, oracle_mod):
    w = make_config("single")
    c = make_exact(bc, w)
    f = c.correlate_rotations(w.R, "full")
    ref = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], w.N, w.h, w.t0)
    assert f.dtype == np.float32
    assert rel_max_err(f[0], ref) <= 1e-4


@pytest.mark.parametrize("seed", [21, 22])
def test_small_complex_exact(bc, oracle_mod, seed):
    w = random_small_case(seed, n_a=9, n_b=7, n_rot=3, N=14, complex_weights=True)
    c = make_exact(bc, w, precision="f64")
    f = as_complex(c.correlate_rotations(w.R, "full"))
    mr = c.correlate_rotations(w.R, "max_real")
    for r in range(w.n_rot):
        ref = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[r], w.N, w.h, w.t0)
        assert rel_max_err(f[r], ref) <= 1e-9
        check_extremum(mr[r]["val"], mr[r]["idx"], ref.real, "max", 1e-9 * np.abs(ref).max())


def test_empty_shape_gives_zero(bc):
    w = random_small_case(30, N=10)
    c = bc.Correlator(N=w.N, h=w.h, t0=w.t0, mode="exact", precision="f64")
    c.shape_upload(0, w.A_xyzr, w.A_w)
    c.shape_upload(1, np.zeros((0, 4)))
    c.spectrum_A()
    f = c.correlate_rotations(w.R, "full")
    assert np.all(f == 0)


def test_invalid_rotation_and_radius(bc):
    w = random_small_case(31, N=10)
    c = make_exact(bc, w, precision="f64")
    bad = w.R.copy()
    bad[0, 0, 0] *= 1.01
    with pytest.raises(bc.BallCorrError) as e:
        c.correlate_rotations(bad, "full")
    assert e.value.status == bc.BC_EINVAL
    refl = np.diag([1.0, 1.0, -1.0])[None]
    with pytest.raises(bc.BallCorrError):
        c.correlate_rotations(refl, "full")
    bad_b = w.B_xyzr.copy()
    bad_b[0, 3] = 0.0
    with pytest.raises(bc.BallCorrError) as e:
        c.shape_upload(1, bad_b)
    assert e.value.status == bc.BC_EINVAL


def test_exact_is_deterministic_across_batchings(bc):
    """Output tiles owned by blocks, fixed-point integer sums (exact.cu): the bits of every
    value are independent of launch order, list splits and batching -- repeated calls and
    batch sizes 1 / 3 / 8 agree bitwise (fp64, complex weights, rotated)."""
    w = random_small_case(71, n_a=40, n_b=30, n_rot=7, N=24, complex_weights=True)
    outs = []
    for nb in (1, 3, 8):
        c = bc.Correlator(N=w.N, h=w.h, t0=w.t0, mode="exact", precision="f64", weights="complex", max_batch=nb)
        c.shape_upload(0, w.A_xyzr, w.A_w)
        c.shape_upload(1, w.B_xyzr, w.B_w)
        outs.append(c.correlate_rotations(w.R, "full"))
        outs.append(c.correlate_rotations(w.R, "full"))
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    # the thread-per-knot kernel (>= 2^18 small knots: the Single workload, 3 rotations)
    ws = make_config("single")
    R3 = random_rotations(np.random.default_rng(3), 3)
    fs = []
    for nb in (1, 3):
        c = bc.Correlator(N=ws.N, h=ws.h, t0=ws.t0, mode="exact", precision="f32", max_batch=nb)
        c.shape_upload(0, ws.A_xyzr, ws.A_w)
        c.shape_upload(1, ws.B_xyzr, ws.B_w)
        fs.append(c.correlate_rotations(R3, "full"))
        fs.append(c.correlate_rotations(R3, "full"))
    for o in fs[1:]:
        assert np.array_equal(o, fs[0])


def test_single_exact_reductions_and_large_knots(bc, oracle_mod):
    """Single-rotation workload (fp32): min/max against the oracle's full grid; and knots
    much larger than a tile (radii 0.3-0.45 on h = 1/16: footprints of ~15 points per axis
    span several 8^3 output tiles) in fp64 against the oracle."""
    w = make_config("single")
    c = make_exact(bc, w)
    mm = c.correlate_rotations(w.R, "minmax")
    ref = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], w.N, w.h, w.t0)
    tol = 1e-4 * np.abs(ref).max()
    check_extremum(mm[0, 0]["val"], mm[0, 0]["idx"], ref, "min", tol)
    check_extremum(mm[0, 1]["val"], mm[0, 1]["idx"], ref, "max", tol)
    big = random_small_case(72, n_a=6, n_b=5, n_rot=2, N=32, r_lo=0.3, r_hi=0.45)
    cb = make_exact(bc, big, precision="f64")
    f = cb.correlate_rotations(big.R, "full")
    for r in range(2):
        rb = oracle_mod.correlate_grid(big.A_xyzr, big.A_w, big.B_xyzr, big.B_w, big.R[r], big.N, big.h, big.t0)
        assert rel_max_err(f[r], rb) <= 1e-9


def test_packed_pairs_signed_complex_weights(bc, oracle_mod):
    """fp32 thread-per-knot path with packed 32-bit pair accumulators (exact_knot_pack_kernel):
    the Single shapes with complex weights of both signs (negative terms exercise the signed
    low/high-half decoding) on the full grid against the oracle; and odd N (no packing) agrees."""
    ws = make_config("single")
    rng = np.random.default_rng(5)
    wa = rng.uniform(-1, 1, ws.A_xyzr.shape[0]) + 1j * rng.uniform(-1, 1, ws.A_xyzr.shape[0])
    wb = rng.uniform(-1, 1, ws.B_xyzr.shape[0]) + 1j * rng.uniform(-1, 1, ws.B_xyzr.shape[0])
    c = bc.Correlator(N=ws.N, h=ws.h, t0=ws.t0, mode="exact", precision="f32", weights="complex")
    c.shape_upload(0, ws.A_xyzr, wa)
    c.shape_upload(1, ws.B_xyzr, wb)
    f = as_complex(c.correlate_rotations(ws.R, "full"))[0]
    ref = oracle_mod.correlate_grid(ws.A_xyzr, wa, ws.B_xyzr, wb, ws.R[0], ws.N, ws.h, ws.t0)
    assert rel_max_err(f, ref) <= 1e-4
    best = c.correlate_rotations(ws.R, "max_real")
    check_extremum(best[0]["val"], best[0]["idx"], ref.real, "max", 1e-4 * np.abs(ref).max())
    # odd N (63): the unpacked 64-bit kernel, same grid points as the first 63^3 of N = 64
    co = bc.Correlator(N=ws.N - 1, h=ws.h, t0=ws.t0, mode="exact", precision="f32", weights="complex")
    co.shape_upload(0, ws.A_xyzr, wa)
    co.shape_upload(1, ws.B_xyzr, wb)
    fo = as_complex(co.correlate_rotations(ws.R, "full"))[0]
    assert rel_max_err(fo, ref[:-1, :-1, :-1]) <= 1e-4
