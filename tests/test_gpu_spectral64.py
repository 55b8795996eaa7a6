"""Spectral mode in fp64 (spectral64.cu) against the band-limited reference at 1e-9 --
SURVEY.md §8(c) reading C-1 (iii).

The fp64 mode runs the spectral METHOD with the library's own host plan (the spreading box
and its origin, the Gaussian window width, the per-axis multipliers: fine spacing, box shift,
deconvolution, A's origin phase; the band and the fold onto the output period by the inverse
DFT) in direct fp64 sums; oracle.bandlimited_correlation is the method's definition (direct
NDFT x ball transform, product, inverse DFT).  Agreement at 1e-9 of max|f| pins the plan's
phases, signs and normalisations far below where the fp32 kernels' own 1e-5 pins could hide
an error."""
import numpy as np
import pytest

from synth import random_small_case
from gpu_helpers import rel_max_err, as_complex

pytestmark = pytest.mark.gpu

TOL64 = 1e-9


@pytest.fixture(scope="module")
def bc():
    import torch
    assert torch.cuda.is_available()
    from paper_1711_05075_b200 import ballcorr
    return ballcorr


@pytest.mark.parametrize("seed,N,Np,K,cplx", [(91, 12, 16, 10, False), (92, 16, 20, 19, False),
                                              (93, 12, 24, 14, True), (94, 10, 12, 17, False)])
def test_fp64_spectral_vs_bandlimited(bc, oracle_mod, seed, N, Np, K, cplx):
    w = random_small_case(seed, n_a=7, n_b=5, n_rot=2, N=N, complex_weights=cplx)
    c = bc.Correlator(N=w.N, h=w.h, t0=w.t0, Np=Np, K=K, precision="f64", weights=w.weights)
    c.shape_upload(0, w.A_xyzr, w.A_w)
    c.shape_upload(1, w.B_xyzr, w.B_w)
    c.spectrum_A()
    f = c.correlate_rotations(w.R, "full")
    assert f.dtype == np.float64
    if cplx:
        f = as_complex(f)
    for r in range(w.n_rot):
        ref = oracle_mod.bandlimited_correlation(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[r], w.N, w.h, w.t0,
                                                 Np * w.h, K)
        assert rel_max_err(f[r], ref) <= TOL64, (r, rel_max_err(f[r], ref))


def test_fp64_and_fp32_spectral_agree(bc):
    """The fp32 kernels and the fp64 parity mode compute the same band-limited f."""
    w = random_small_case(95, n_a=9, n_b=7, n_rot=2, N=16)
    out = []
    for prec in ("f32", "f64"):
        c = bc.Correlator(N=w.N, h=w.h, t0=w.t0, Np=20, K=19, precision=prec)
        c.shape_upload(0, w.A_xyzr, w.A_w)
        c.shape_upload(1, w.B_xyzr, w.B_w)
        c.spectrum_A()
        out.append(c.correlate_rotations(w.R, "full"))
    assert rel_max_err(out[0], out[1]) <= 1e-5


def test_fp64_spectral_limits(bc):
    w = random_small_case(96, N=8)
    c = bc.Correlator(N=w.N, h=w.h, t0=w.t0, Np=16, K=7, precision="f64")
    c.shape_upload(0, w.A_xyzr)
    c.shape_upload(1, w.B_xyzr)
    c.spectrum_A()
    with pytest.raises(bc.BallCorrError) as e:
        c.correlate_rotations(w.R, "minmax")
    assert e.value.status == bc.BC_EUNSUPPORTED
    with pytest.raises(bc.BallCorrError) as e:
        c.evaluate_points_spectral(w.R, np.zeros((w.n_rot, 3)), 10)
    assert e.value.status == bc.BC_EUNSUPPORTED
