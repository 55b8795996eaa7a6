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
"""
from __future__ import annotations

import numpy as np

from . import lens


def _offset(xyzr, r0):
    x = np.array(xyzr, dtype=np.float64)
    x[:, 3] += r0
    return x


def sc_score_points(S1, S2, r0, lam, R, N, h, t0, flat_idx):
    """G(R, t_m) at flat C-order grid indices m of t_m = t0 + m h (unit weights per ball)."""
    S1o, S2o = _offset(S1, r0), _offset(S2, r0)
    g = lambda a, b: lens.correlate_points(a, None, b, None, R, N, h, t0, flat_idx)
    return -(lam * lam * g(S1, S2) - lam * g(S1o, S2) - lam * g(S1, S2o) + g(S1o, S2o))
