"""oracle/ -- TEST INFRASTRUCTURE ONLY (never on the product path).

Plain fp64 CPU implementations of what the CUDA path computes, written from
PAPER.md.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import this package.  It shares
no code with `paper_1711_05075_b200/`; the two meet only through the seeded
arrays of `synth/`.

* `lens.py`         -- ctypes front-end of `lens_oracle.c`: the direct pair sum
                       f_R(t) = sum_ij w_i v_j V(r_i, s_j, |a_i - R b_j - t|)
                       (PAPER.md L316-L322 eq_relg_0, L343-L360 eq_ORP/eq_convgP).
* `bandlimited.py`  -- the spectral method step by step in numpy: NDFT of the
                       knots times the ball transform (L276-L294 eq_fballhat,
                       eq_rhoPhat), the Fourier correlation (L398-L404 eq_ccghat)
                       and a direct inverse DFT onto the translation grid.
* `complementarity.py` -- the shape-complementarity score G of eq_score (L447-L461)
                       as the four real correlations of its expansion.
"""
from .lens import (  # noqa: F401
    build_oracle,
    lens_volume,
    correlate_grid,
    correlate_points,
    oracle_threads,
)
from .bandlimited import (  # noqa: F401
    ball_transform,
    ndft_density,
    bandlimited_correlation,
    band_modes,
)
from .complementarity import sc_score_points, eq_score_points  # noqa: F401
