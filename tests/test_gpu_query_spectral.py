"""The paper's time-critical query (bc_evaluate_points_spectral; PAPER.md L432-L439 eq_single,
L539-L546): f_R(t) by Parseval over the first m' band modes in radial-shell order.

Pins:
* m' = every mode of |k| <= rho (complete shells) is the band-limited f of the SPHERICAL band
  |k_i| <= K, |k| <= rho -- oracle.bandlimited_correlation(K_sphere=rho), whose sphere mask is
  pinned in tests/test_oracle.py (cube cover, 7-mode closed form, Parseval) -- at grid and
  off-grid translations, real and complex weights;
* m' = the whole cube band equals the spectral grid of bc_correlate_rotations;
* the error against the exact pair-lens f shrinks as m' grows (the accuracy / time trade-off).
"""
import numpy as np
import pytest

from synth import random_small_case, random_rotations
from gpu_helpers import rel_max_err

pytestmark = pytest.mark.gpu

TOL = 2e-5  # A's spectrum from the spreading path (~1e-6) and fp32 phases / sums


@pytest.fixture(scope="module")
def bc():
    import torch
    assert torch.cuda.is_available()
    from paper_1711_05075_b200 import ballcorr
    return ballcorr


def n_modes(K, rho):
    """Band modes with |k| <= rho, counted one by one (brute force over the cube)."""
    k = np.arange(-K, K + 1)
    kk = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
    return int((kk <= rho * rho).sum())


def spectral(bc, w, Np, K):
    c = bc.Correlator(N=w.N, h=w.h, t0=w.t0, Np=Np, K=K, weights=w.weights)
    c.shape_upload(0, w.A_xyzr, w.A_w)
    c.shape_upload(1, w.B_xyzr, w.B_w)
    c.spectrum_A()
    return c


@pytest.mark.parametrize("cplx", [False, True])
def test_complete_shells_equal_the_spherical_band(bc, oracle_mod, cplx):
    w = random_small_case(81 + cplx, n_a=9, n_b=7, n_rot=2, N=12, complex_weights=cplx)
    Np, K = 24, 12
    P = Np * w.h
    c = spectral(bc, w, Np, K)
    rng = np.random.default_rng(3)
    for rho in (3.5, 7.2):
        m = n_modes(K, rho)
        for r in range(w.n_rot):
            ref = oracle_mod.bandlimited_correlation(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[r], w.N, w.h, w.t0, P, K,
                                                     K_sphere=rho)
            scale = np.abs(ref).max()
            idx = rng.choice(w.N ** 3, 12, replace=False)
            mm = np.stack(np.unravel_index(idx, (w.N,) * 3), axis=1)
            t = np.asarray(w.t0) + w.h * mm
            got = c.evaluate_points_spectral(np.repeat(w.R[r:r + 1], len(t), axis=0), t, m)
            assert np.abs(got - ref.reshape(-1)[idx]).max() <= TOL * scale, (rho, r)
            # off the grid: a 1-point grid at t
            toff = rng.uniform(-0.4, 0.4, size=3)
            ref1 = oracle_mod.bandlimited_correlation(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[r], 1, w.h, tuple(toff),
                                                      P, K, K_sphere=rho).reshape(-1)[0]
            got1 = c.evaluate_points_spectral(w.R[r:r + 1], toff[None, :], m)[0]
            assert abs(got1 - ref1) <= TOL * scale


def test_full_band_equals_the_spectral_grid(bc, oracle_mod):
    """m' = (2K + 1)^3: the cube band's f -- against the band-limited oracle (1e-5 of max|f|,
    the query's own error) and the spectral grid of bc_correlate_rotations (each within
    1e-5 of the oracle, so 2e-5 between them)."""
    w = random_small_case(83, n_a=10, n_b=8, n_rot=2, N=16)
    Np, K = 20, 19
    c = spectral(bc, w, Np, K)
    f = c.correlate_rotations(w.R, "full")
    assert c.query("query_modes") == 0
    rng = np.random.default_rng(4)
    for r in range(2):
        ref = oracle_mod.bandlimited_correlation(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[r], w.N, w.h, w.t0, Np * w.h, K)
        idx = np.concatenate([rng.choice(w.N ** 3, 20, replace=False), [int(np.argmax(f[r]))]])
        mm = np.stack(np.unravel_index(idx, (w.N,) * 3), axis=1)
        t = np.asarray(w.t0) + w.h * mm
        got = c.evaluate_points_spectral(np.repeat(w.R[r:r + 1], len(t), axis=0), t, (2 * K + 1) ** 3)
        scale = np.abs(ref).max()
        assert np.abs(got - ref.reshape(-1)[idx]).max() <= 1e-5 * scale
        assert np.abs(got - f[r].reshape(-1)[idx]).max() <= 2e-5 * scale
    assert c.query("query_modes") == (2 * K + 1) ** 3
    # a smaller m' reuses the tables (a prefix of the list)
    c.evaluate_points_spectral(w.R[:1], np.zeros((1, 3)), 4096)
    assert c.query("query_modes") == (2 * K + 1) ** 3


def test_error_shrinks_with_m_prime(bc):
    """Accuracy-for-time (L539-L546): the truncated sum approaches the exact f as m' grows."""
    w = random_small_case(84, n_a=12, n_b=10, n_rot=1, N=16, r_lo=0.15, r_hi=0.3)
    c = spectral(bc, w, 32, 47)
    rng = np.random.default_rng(5)
    R = random_rotations(rng, 6)
    t = rng.uniform(-0.3, 0.3, size=(6, 3))
    exact = c.evaluate_points(R, t)
    errs = []
    for m in (33, 257, 2109, 17077, 95 ** 3):
        errs.append(np.abs(c.evaluate_points_spectral(R, t, m) - exact).max() / np.abs(exact).max())
    assert errs[0] > errs[2] > errs[-1]
    assert errs[-1] < 1e-3


def test_spectral_query_errors(bc):
    w = random_small_case(85, N=8)
    c = spectral(bc, w, 16, 7)
    with pytest.raises(bc.BallCorrError) as e:
        c.evaluate_points_spectral(w.R, np.zeros((w.n_rot, 3)), 0)
    assert e.value.status == bc.BC_ERANGE
    with pytest.raises(bc.BallCorrError) as e:
        c.evaluate_points_spectral(w.R, np.zeros((w.n_rot, 3)), 15 ** 3 + 1)
    assert e.value.status == bc.BC_ERANGE
    x = bc.Correlator(N=w.N, h=w.h, t0=w.t0, mode="exact")
    x.shape_upload(0, w.A_xyzr)
    x.shape_upload(1, w.B_xyzr)
    with pytest.raises(bc.BallCorrError) as e:
        x.evaluate_points_spectral(w.R, np.zeros((w.n_rot, 3)), 10)
    assert e.value.status == bc.BC_EUNSUPPORTED
