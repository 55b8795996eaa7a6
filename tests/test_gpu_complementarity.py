"""Shape complementarity on the GPU.

The score G of eq_score is ONE complex correlation of the two affinity ball sets
(complementarity.py) on the docking plan (N_p = 128, K = 191, the preset bench and the
docking parity test use), compared with the oracle's four real correlations at sampled
grid points, the GPU's best-score index and off-grid configurations (exact query).
Recipe: the docking molecules' atoms (synth C-9), r0 = 1.4 A (the water-molecule offset
the paper names, L451), lambda = 3.
"""
import numpy as np
import pytest

from synth import make_config

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-4
R0, LAM = 1.4, 3.0


@pytest.fixture(scope="module")
def sc():
    import torch
    assert torch.cuda.is_available()
    from paper_1711_05075_b200.complementarity import Complementarity
    from paper_1711_05075_b200.presets import correlator_kwargs
    w = make_config("docking", n_rot=8)
    atoms1 = w.A_xyzr[: len(w.A_xyzr) // 2]  # core balls = the atoms (synth C-4 layout)
    atoms2 = w.B_xyzr[: len(w.B_xyzr) // 2]
    c = Complementarity(R0, LAM, **correlator_kwargs("docking", w.N, w.h, w.t0, "complex"))
    c.upload(atoms1, atoms2)
    return c, w, atoms1, atoms2


def test_scores_sampled(sc, oracle_mod):
    c, w, S1, S2 = sc
    r = 3
    G = c.scores(w.R[r:r + 1])[0]
    best = c.best(w.R[:4])
    rng = np.random.default_rng(11)
    flat = np.abs(G).reshape(-1)
    idx = np.unique(np.concatenate([rng.choice(flat.size, 100, replace=False),
                                    np.argpartition(flat, -40)[-40:], [int(best[r]["idx"])]]))
    ref = oracle_mod.sc_score_points(S1, S2, R0, LAM, w.R[r], w.N, w.h, w.t0, idx)
    scale = np.abs(ref).max()
    assert np.abs(G.reshape(-1)[idx] - ref).max() <= TOL_F32 * scale
    # the imaginary plane is zero up to the band error (all weight products are real)
    f = c.corr.correlate_rotations(w.R[r:r + 1], "full")[0]
    assert np.abs(f[..., 1]).max() <= TOL_F32 * scale
    # best score: value equals the full output's max, and the oracle agrees at its index
    assert best[r]["val"] == pytest.approx(float(G.max()), abs=1e-12 * scale)
    k = int(np.searchsorted(idx, int(best[r]["idx"])))
    assert abs(ref[k] - best[r]["val"]) <= TOL_F32 * scale


def test_offgrid_exact(sc, oracle_mod):
    c, w, S1, S2 = sc
    rng = np.random.default_rng(12)
    t = rng.uniform(-15, 15, size=(3, 3))
    got = c.evaluate_points(w.R[:3], t)
    ref = np.array([oracle_mod.sc_score_points(S1, S2, R0, LAM, w.R[q], 1, 1.0, t[q], [0])[0]
                    for q in range(3)])
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
