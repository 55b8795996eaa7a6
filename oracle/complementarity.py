"""Shape-complementarity score, fp64 (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md L447-L461 (Section "Shape Complementarity"): F_S = i (f_{S (+) B0} - lambda f_S)
(L449-L451) and G_{S1,S2}(R, t) = (F_{RS2} * F_{S1})(t) (eq_score).
Substituting F and expanding the product under the integral (weights multiplied without
conjugation, reading C-3: i * i = -1) gives, term by term as eq_score lists them,

    G = -[ lambda^2 g(S1, S2) - lambda g(S1 (+) B0, S2) - lambda g(S1, S2 (+) B0)
           + g(S1 (+) B0, S2 (+) B0) ]

where g is the plain ball-set correlation (lens.correlate_points) and S (+) B0 raises
every primitive radius by r0 (L459: "the offsets correspond to an increase of radii in
the primitive balls").  The paper writes the two cross terms as one, -2 lambda g * f_B0,
which holds in its bump-function algebra; for ball sets they are two correlations
(reading R-5).  Four real correlations, summed in the order above.

`eq_score_points` evaluates eq_score VERBATIM instead: G_eq = (F_{RS2} star F_{S1})(t) with
the cross-correlation of PAPER.md L791, (f1 star f2)(t) = int conj(f1(x)) f2(x + t) dx,
which conjugates the first argument (the moving shape's affinity).  With i * conj(i) = +1
its expansion is the paper's own algebra (L455-L457),

    G_eq = lambda^2 g(S1, S2) - lambda g(S1 (+) B0, S2) - lambda g(S1, S2 (+) B0)
           + g(S1 (+) B0, S2 (+) B0),

so sc_score_points = -G_eq exactly: the score this package (and the library's
max_real reduction of the complementarity product) maximises is -G_eq, i.e. the
library's best configuration is the one MINIMISING the paper's literal G_eq.  Which sign
the paper intends is contradictory in the text (L458's penalty/reward narrative vs the
algebra of eq_score); reading R-5 takes the narrative.  Both are pinned to
brute-force voxel integrals of their definitions in tests/test_complementarity.py.
"""
from __future__ import annotations

import numpy as np

from . import lens


def _offset(xyzr, r0):
    x = np.array(xyzr, dtype=np.float64)
    x[:, 3] += r0
    return x


def _affinity(xyzr, r0, lam, conj):
    """F_S = i (f_{S (+) B0} - lambda f_S) (L449-L451) as a weighted ball set: every ball
    B(c, r) of S gives B(c, r + r0) with weight i and B(c, r) with weight -i lambda
    (conjugated weights when conj)."""
    x = np.asarray(xyzr, dtype=np.float64)
    balls = np.concatenate([_offset(x, r0), x], axis=0)
    w = np.concatenate([np.full(len(x), 1j), np.full(len(x), -1j * lam)])
    return balls, (np.conj(w) if conj else w)


def eq_score_points(S1, S2, r0, lam, R, N, h, t0, flat_idx):
    """G_eq(R, t_m) = (F_{RS2} star F_{S1})(t_m) of eq_score (L453-L454) with star as at
    L791 (first argument conjugated): sum over affinity ball pairs of
    alpha_a conj(beta_b) V(r_a, s_b, |a - R b - t|).  Real for these weights; returned as
    float64 (the imaginary part is checked to vanish by the tests)."""
    A, wa = _affinity(S1, r0, lam, conj=False)
    B, wb = _affinity(S2, r0, lam, conj=True)
    return lens.correlate_points(A, wa, B, wb, R, N, h, t0, flat_idx)


def sc_score_points(S1, S2, r0, lam, R, N, h, t0, flat_idx):
    """G(R, t_m) at flat C-order grid indices m of t_m = t0 + m h (unit weights per ball)."""
    S1o, S2o = _offset(S1, r0), _offset(S2, r0)
    g = lambda a, b: lens.correlate_points(a, None, b, None, R, N, h, t0, flat_idx)
    return -(lam * lam * g(S1, S2) - lam * g(S1o, S2) - lam * g(S1, S2o) + g(S1o, S2o))
