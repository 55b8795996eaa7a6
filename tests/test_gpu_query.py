"""Single-configuration query (PAPER.md L432-L439 / L539-L546):
bc_evaluate_points gives f_R(t) at arbitrary (R, t), off the grid, exactly (pair-lens sum).

Checked against the fp64 lens oracle evaluated at the same configurations (a one-point grid
with t0 = t), on the tiny, sweep and docking workloads; against the spectral grid of the
same context at grid translations (within the band tolerance); and for its error paths.
"""
import numpy as np
import pytest

from synth import make_config, random_rotations

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bc():
    import torch
    assert torch.cuda.is_available()
    from paper_1711_05075_b200 import ballcorr
    return ballcorr


def correlator(bc, w):
    from paper_1711_05075_b200.presets import correlator_kwargs
    c = bc.Correlator(**correlator_kwargs(w.name, w.N, w.h, w.t0, w.weights))
    c.shape_upload(0, w.A_xyzr, w.A_w)
    c.shape_upload(1, w.B_xyzr, w.B_w)
    return c


def oracle_at(oracle_mod, w, R, t):
    return np.array([oracle_mod.correlate_points(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, R[q], 1, 1.0, t[q], [0])[0]
                     for q in range(len(t))])


def test_tiny_offgrid(bc, oracle_mod):
    w = make_config("tiny")
    c = correlator(bc, w)
    rng = np.random.default_rng(5)
    R = random_rotations(rng, 12)
    t = rng.uniform(-0.6, 0.6, size=(12, 3))
    got = c.evaluate_points(R, t)
    ref = oracle_at(oracle_mod, w, R, t)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.array_equal(got, c.evaluate_points(R, t))  # deterministic


def test_sweep_offgrid_and_grid(bc, oracle_mod):
    w = make_config("sweep", n_rot=4)
    c = correlator(bc, w)
    c.spectrum_A()
    rng = np.random.default_rng(6)
    r = 1
    f = c.correlate_rotations(w.R[r:r + 1], "full")[0]
    m = np.array(np.unravel_index(int(np.argmax(f)), f.shape))
    t_grid = w.t0 + w.h * m
    # around the overlap peak, off the grid, plus the grid point itself
    t = np.vstack([t_grid + rng.uniform(-2 * w.h, 2 * w.h, size=(5, 3)), t_grid[None, :]])
    R = np.repeat(w.R[r:r + 1], len(t), axis=0)
    got = c.evaluate_points(R, t)
    ref = oracle_at(oracle_mod, w, R, t)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    # the spectral grid approximates the same exact value within the north_star tolerance
    assert abs(got[-1] - f.max()) <= 1e-4 * abs(got[-1])


def test_docking_complex(bc, oracle_mod):
    w = make_config("docking", n_rot=3)
    c = correlator(bc, w)
    rng = np.random.default_rng(7)
    t = rng.uniform(-20, 20, size=(3, 3))
    got = c.evaluate_points(w.R, t)
    ref = oracle_at(oracle_mod, w, w.R, t)
    assert np.iscomplexobj(got)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_errors(bc):
    w = make_config("tiny")
    c = correlator(bc, w)
    R = np.eye(3)[None] * np.array([1.0, 1.0, -1.0])[None, :, None]   # det = -1
    with pytest.raises(bc.BallCorrError):
        c.evaluate_points(R, np.zeros((1, 3)))
    with pytest.raises(bc.BallCorrError):
        c.evaluate_points(np.eye(3)[None], np.array([[0.0, np.nan, 0.0]]))
    e = bc.Correlator(N=w.N, h=w.h, t0=w.t0, mode="exact", precision="f64")
    e.shape_upload(0, w.A_xyzr[:0], None)
    e.shape_upload(1, w.B_xyzr, w.B_w)
    assert np.all(e.evaluate_points(np.eye(3)[None], np.zeros((1, 3))) == 0.0)
