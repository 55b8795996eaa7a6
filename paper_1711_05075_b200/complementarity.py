"""Shape complementarity score (Section "Shape
Complementarity").

The paper's complex affinity function of a shape S with offset ball B0 = B(0, r0) and
penalty factor lambda,

    F_S(x) = i (f_{S (+) B0}(x) - lambda f_S(x))

and the score G(R, t) = (F_{RS2} * F_{S1})(t) (eq_score).  For a spherically
sampled shape the offset S (+) B0 raises every primitive radius by r0 (L459), so F_S is
itself a weighted ball set: every ball B(c, r) of S contributes B(c, r + r0) with weight i
and B(c, r) with weight -i lambda.  The score is then ONE complex correlation of the two
affinity ball sets on the same spectral/exact path as any other weighted ball set -- the
paper's "cumulatively obtained from a single 4D NDFT" (L459-L460) -- and, with products
of weights taken without conjugation (reading C-3),

    G = -lambda^2 g(S1, S2) + lambda g(S1 (+) B0, S2) + lambda g(S1, S2 (+) B0)
        - g(S1 (+) B0, S2 (+) B0),

real: interior-interior overlaps penalised by lambda^2, offset-interior overlaps
rewarded, offset-offset overlaps penalised by 1, which is the sign pattern L458 states
(reading R-5).  This module only builds the ball sets and reads the real part;
all arithmetic runs in libballcorr's kernels.

Sign, stated explicitly: eq_score read literally, with the cross-correlation of L791
conjugating its first argument (F_{RS2}), is G_eq = lambda^2 g - lambda g(S1 (+) B0, S2)
- lambda g(S1, S2 (+) B0) + g(S1 (+) B0, S2 (+) B0) (the paper's algebra).
The score returned here is G = -G_eq, so `best` returns max(-G_eq) = -min G_eq and its
index is the argmin of the literal G_eq (pinned: oracle.eq_score_points against a
conjugated voxel integral, tests/test_complementarity.py).
"""
from __future__ import annotations

import numpy as np

from .ballcorr import BC_MODE_SPECTRAL, Correlator, BallCorrError


def affinity_balls(xyzr, r0: float, lam: float):
    """(n, 4) balls (x, y, z, r) of S -> (2n, 4) balls and complex weights of F_S:
    rows [0, n) the offset balls (r + r0, weight i), rows [n, 2n) the balls of S
    (weight -i lambda)."""
    x = np.asarray(xyzr, dtype=np.float64)
    if x.ndim != 2 or x.shape[1] != 4:
        raise ValueError("xyzr must have shape (n, 4)")
    if not (np.isfinite(r0) and r0 >= 0.0 and np.isfinite(lam) and lam > 0.0):
        raise ValueError("need r0 >= 0 and lambda > 0")
    off = x.copy()
    off[:, 3] += r0
    w = np.concatenate([np.full(len(x), 1j), np.full(len(x), -1j * lam)])
    return np.concatenate([off, x], axis=0), w


class Complementarity:
    """Shape-complementarity scores G(R, t) of S1 (fixed, "A") and rotated S2 ("B") on the
    translation grid t_m = t0 + m h; the correlator runs with complex weights."""

    def __init__(self, r0: float, lam: float, **correlator_kwargs):
        correlator_kwargs = dict(correlator_kwargs)
        correlator_kwargs["weights"] = "complex"
        self.r0, self.lam = float(r0), float(lam)
        self.corr = Correlator(**correlator_kwargs)

    def upload(self, S1_xyzr, S2_xyzr):
        for which, s in ((0, S1_xyzr), (1, S2_xyzr)):
            xyzr, w = affinity_balls(s, self.r0, self.lam)
            self.corr.shape_upload(which, xyzr, w)
        if self.corr.params.mode == BC_MODE_SPECTRAL:  # A's band spectrum, once
            self.corr.spectrum_A()

    def scores(self, R, out=None, stream=None):
        """Full G for each rotation: (n_rot, N, N, N) real (a view of the complex output's
        real plane when `out` is None)."""
        f = self.corr.correlate_rotations(R, "full", out=out, stream=stream)
        return f[..., 0] if out is None else f

    def best(self, R, out=None, stream=None):
        """Per rotation, the largest score G = -G_eq and its flat grid index (lowest on ties):
        val = max_t(-G_eq) = -min_t G_eq of the literal eq_score (see the module docstring)."""
        return self.corr.correlate_rotations(R, "max_real", out=out, stream=stream)

    def evaluate_points(self, R, t):
        """G at arbitrary configurations (exact pair-lens sum, fp64)."""
        return self.corr.evaluate_points(R, t).real


__all__ = ["affinity_balls", "Complementarity", "BallCorrError"]
