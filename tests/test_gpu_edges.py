"""Edge cases of the spectral path on the sweep plan (the launch configuration bench.py
times): empty shapes, ties in the reduction, a B whose balls sit on the edge of its
rotation-invariant support, and the n_rot < 1 error.  Oracle: the fp64 pair-lens sum."""
import numpy as np
import pytest

from synth import make_config

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-4


@pytest.fixture(scope="module")
def bc():
    import torch
    assert torch.cuda.is_available()
    from paper_1711_05075_b200 import ballcorr
    return ballcorr


@pytest.fixture(scope="module")
def sweep():
    return make_config("sweep", n_rot=3)


def correlator(bc, w, A, wA, B, wB):
    from paper_1711_05075_b200.presets import correlator_kwargs
    c = bc.Correlator(**correlator_kwargs("sweep", w.N, w.h, w.t0, "real"))
    c.shape_upload(0, A, wA)
    c.shape_upload(1, B, wB)
    c.spectrum_A()
    return c


@pytest.mark.parametrize("empty", ["A", "B"])
def test_empty_shape_is_zero_and_ties_pick_lowest_index(bc, sweep, empty):
    w = sweep
    A, wA = (w.A_xyzr[:0], None) if empty == "A" else (w.A_xyzr, w.A_w)
    B, wB = (w.B_xyzr[:0], None) if empty == "B" else (w.B_xyzr, w.B_w)
    c = correlator(bc, w, A, wA, B, wB)
    f = c.correlate_rotations(w.R[:1], "full")
    assert np.all(f == 0)
    for kind in ("min_argmin", "max_argmax"):
        r = c.correlate_rotations(w.R, kind)
        assert np.all(r["val"] == 0) and np.all(r["idx"] == 0)  # every value ties: lowest index


def test_balls_on_the_support_edge(bc, oracle_mod, sweep):
    """Balls on the edge of B's extent (centres at 0.2, radius 0.02: the sweep recipe's
    bound) and at the rotation centre.  (a) Alone: the fast plan (blob box spread) against the
    generic plan (Gaussian spread, no box), same band, so the difference isolates the
    spreading up to the two windows' alias levels (6e-6 + 1.4e-5, R-1): <= 5e-5.
    A five-ball B is outside the regime the K = 255 band was chosen for (its band-truncation
    error relative to max|f| is ~2.5e-4: few balls add no coherent peak), so (b) the oracle
    parity at the north_star 1e-4 is taken with the edge balls added to the workload's B."""
    from gpu_helpers import rel_max_err
    from paper_1711_05075_b200.presets import correlator_kwargs
    w = sweep
    E = np.array([[0.0, 0.0, 0.0, 0.02], [0.2, 0.0, 0.0, 0.02], [0.0, -0.2, 0.0, 0.005],
                  [0.0, 0.0, 0.2, 0.01], [-0.1155, 0.1155, -0.1155, 0.02]])
    fast = correlator(bc, w, w.A_xyzr, w.A_w, E, np.ones(len(E)))
    assert fast.query("fold_fast") == 1 and fast.query("L_B") == 256
    gen = bc.Correlator(**correlator_kwargs("sweep", w.N, w.h, w.t0, "real", generic_only=True))
    gen.shape_upload(0, w.A_xyzr, w.A_w)
    gen.shape_upload(1, E, np.ones(len(E)))
    gen.spectrum_A()
    a = fast.correlate_rotations(w.R[:2], "full")
    b = gen.correlate_rotations(w.R[:2], "full")
    for r in range(2):
        assert rel_max_err(a[r], b[r]) <= 5e-5, rel_max_err(a[r], b[r])

    B = np.concatenate([w.B_xyzr, E])
    c = correlator(bc, w, w.A_xyzr, w.A_w, B, np.ones(len(B)))
    f = c.correlate_rotations(w.R[:2], "full")
    red = c.correlate_rotations(w.R[:2], "max_argmax")
    for r in range(2):
        rng = np.random.default_rng(40 + r)
        flat = f[r].reshape(-1)
        idx = np.unique(np.concatenate([rng.choice(flat.size, 100, replace=False),
                                        np.argpartition(np.abs(flat), -40)[-40:], [int(red[r]["idx"])]]))
        ref = oracle_mod.correlate_points(w.A_xyzr, w.A_w, B, np.ones(len(B)), w.R[r], w.N, w.h, w.t0, idx)
        scale = np.abs(ref).max()
        assert np.abs(flat[idx] - ref).max() <= TOL_F32 * scale
        assert red[r]["val"] == pytest.approx(float(flat.max()), abs=1e-12 * scale)


def test_zero_rotations_is_einval(bc, sweep):
    w = sweep
    c = correlator(bc, w, w.A_xyzr, w.A_w, w.B_xyzr, w.B_w)
    with pytest.raises(bc.BallCorrError) as e:
        c.correlate_rotations(w.R[:0], "min_argmin")
    assert e.value.status == bc.BC_EINVAL
