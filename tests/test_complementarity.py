"""Shape complementarity, CPU side.

* The oracle's score (four real correlations, oracle/complementarity.py) against the
  definition itself: F_S = i (f_{S (+) B0} - lambda f_S) sampled on a fine voxel lattice
  and G(t) = sum_x F_{S1}(x) F_{RS2}(x - t) dx integrated by brute force (midpoint rule).
* The special case r0 = 0, where F_S = i (1 - lambda) f_S and G = -(1 - lambda)^2 g.
* The product's host logic (affinity ball sets of complementarity.py) run through the
  oracle's complex pair sum equals the oracle's four-term score (no CUDA call).
"""
import numpy as np
import pytest

from synth import random_rotations


def _shapes(seed):
    rng = np.random.default_rng(seed)
    S1 = np.column_stack([rng.uniform(-0.15, 0.15, size=(3, 3)), rng.uniform(0.12, 0.2, size=3)])
    S2 = np.column_stack([rng.uniform(-0.12, 0.12, size=(2, 3)), rng.uniform(0.1, 0.18, size=2)])
    return S1, S2, random_rotations(rng, 1)[0]


def _affinity_on_lattice(balls, centres, r0, lam, pts):
    """F_S at lattice points: i (sum_j 1[|x - c_j| < r_j + r0] - lambda sum_j 1[|x - c_j| < r_j])."""
    off = np.zeros(len(pts))
    core = np.zeros(len(pts))
    for c, r in zip(centres, balls[:, 3]):
        d2 = ((pts - c) ** 2).sum(axis=1)
        off += d2 < (r + r0) ** 2
        core += d2 < r * r
    return 1j * (off - lam * core)


def test_oracle_score_matches_voxel_definition(oracle_mod):
    S1, S2, R = _shapes(3)
    r0, lam = 0.06, 2.5
    hv = 0.006
    ax = (np.arange(-0.5, 0.5, hv) + hv / 2)
    pts = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), axis=-1).reshape(-1, 3)
    F1 = _affinity_on_lattice(S1, S1[:, :3], r0, lam, pts)
    RB = S2[:, :3] @ R.T
    # translations on a coarse grid t0 + m h with overlaps of every kind
    N, h, t0 = 5, 0.1, (-0.2, -0.2, -0.2)
    idx = np.array([0, 31, 62, 93, 124, 7, 112, 55])
    m = np.stack(np.unravel_index(idx, (N, N, N)), axis=1)
    ref = oracle_mod.sc_score_points(S1, S2, r0, lam, R, N, h, t0, idx)
    for k, mm in enumerate(m):
        t = np.asarray(t0) + h * mm
        F2 = _affinity_on_lattice(S2, RB + t, r0, lam, pts)  # F_{(R,t)S2}(x) = F_{RS2}(x - t)
        G = (F1 * F2).sum() * hv ** 3  # no conjugation (reading C-3)
        assert abs(G.imag) < 1e-12
        assert G.real == pytest.approx(ref[k], abs=1e-2 * np.abs(ref).max()), (k, G, ref[k])
    # the terms do not nearly cancel: a dropped cross term would move G by more than the bar
    g_cross = oracle_mod.correlate_points(S1, None, np.column_stack([S2[:, :3], S2[:, 3] + r0]), None,
                                          R, N, h, t0, idx)
    assert (lam * np.abs(g_cross)).max() > 0.2 * np.abs(ref).max()


def test_eq_score_verbatim_matches_conjugated_voxel_integral(oracle_mod):
    """eq_score read literally: G_eq(t) = (F_{RS2} star F_{S1})(t) with star as defined at
    PAPER.md L791, (f1 star f2)(t) = int conj(f1(x)) f2(x + t) dx.  Substituting y = x + t,
    G_eq = int conj(F_{RS2}(y - t)) F_{S1}(y) dy: the brute-force voxel integral with the
    moving shape's affinity CONJUGATED pins oracle.eq_score_points, and the score the
    package maximises (sc_score_points, reading R-5) is exactly its negative."""
    S1, S2, R = _shapes(6)
    r0, lam = 0.05, 3.0
    hv = 0.006
    ax = (np.arange(-0.5, 0.5, hv) + hv / 2)
    pts = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), axis=-1).reshape(-1, 3)
    F1 = _affinity_on_lattice(S1, S1[:, :3], r0, lam, pts)
    RB = S2[:, :3] @ R.T
    N, h, t0 = 5, 0.1, (-0.2, -0.2, -0.2)
    idx = np.array([0, 31, 62, 93, 124, 7, 112, 55, 68])
    m = np.stack(np.unravel_index(idx, (N, N, N)), axis=1)
    G_eq = oracle_mod.eq_score_points(S1, S2, r0, lam, R, N, h, t0, idx)
    assert np.abs(G_eq.imag).max() <= 1e-13 * np.abs(G_eq).max()
    G_eq = G_eq.real
    for k, mm in enumerate(m):
        t = np.asarray(t0) + h * mm
        F2 = _affinity_on_lattice(S2, RB + t, r0, lam, pts)      # F_{RS2}(y - t)
        G = (np.conj(F2) * F1).sum() * hv ** 3                    # L791: first argument conjugated
        assert abs(G.imag) < 1e-12
        assert G.real == pytest.approx(G_eq[k], abs=1e-2 * np.abs(G_eq).max()), (k, G, G_eq[k])
    # the package's score is -G_eq (R-5: the L458 narrative, not eq_score's algebra)
    sc = oracle_mod.sc_score_points(S1, S2, r0, lam, R, N, h, t0, idx)
    assert np.abs(sc + G_eq).max() <= 1e-13 * np.abs(G_eq).max()
    # interior-interior collision dominates at lambda = 3: literal G_eq > 0 there (a PENALTY
    # only under the sign flip of R-5)
    deep = oracle_mod.eq_score_points(S1, S2, r0, lam, np.eye(3), 1, 1.0, (0.0, 0.0, 0.0), [0])
    assert deep.real[0] > 0


def test_zero_offset_reduces_to_scaled_correlation(oracle_mod):
    S1, S2, R = _shapes(4)
    lam = 3.0
    idx = np.arange(0, 125, 3)
    G = oracle_mod.sc_score_points(S1, S2, 0.0, lam, R, 5, 0.1, (-0.2, -0.2, -0.2), idx)
    g = oracle_mod.correlate_points(S1, None, S2, None, R, 5, 0.1, (-0.2, -0.2, -0.2), idx)
    assert np.abs(G + (1 - lam) ** 2 * g).max() <= 1e-13 * np.abs(g).max()


def test_affinity_ball_sets_give_the_oracle_score(oracle_mod):
    from paper_1711_05075_b200.complementarity import affinity_balls
    S1, S2, R = _shapes(5)
    r0, lam = 0.05, 4.0
    A, wA = affinity_balls(S1, r0, lam)
    B, wB = affinity_balls(S2, r0, lam)
    assert A.shape == (6, 4) and np.iscomplexobj(wA)
    N, h, t0 = 6, 0.08, (-0.2, -0.2, -0.2)
    idx = np.arange(N ** 3)
    f = oracle_mod.correlate_points(A, wA, B, wB, R, N, h, t0, idx)
    G = oracle_mod.sc_score_points(S1, S2, r0, lam, R, N, h, t0, idx)
    assert np.abs(f.imag).max() <= 1e-13 * np.abs(G).max()
    assert np.abs(f.real - G).max() <= 1e-12 * np.abs(G).max()


def test_affinity_balls_rejects_bad_parameters():
    from paper_1711_05075_b200.complementarity import affinity_balls
    S = np.zeros((2, 4))
    with pytest.raises(ValueError):
        affinity_balls(S, -0.1, 1.0)
    with pytest.raises(ValueError):
        affinity_balls(S, 0.1, 0.0)
    with pytest.raises(ValueError):
        affinity_balls(S[:, :3], 0.1, 1.0)
