"""Full-grid parity of the three spectral workloads against the fp64 lens oracle, on the
rotation the GPU scores best, in bench.py's launch configuration (presets.py).

north_star: max|f_gpu - f_cpu| <= 1e-4 max|f_cpu| over EVERY translation of the grid.
The rotation is chosen by the GPU's own per-rotation reduction over the config's rotation
set (SURVEY.md §8(d) "each sample always includes the rotation holding the GPU's best
score"); the oracle (oracle/lens_oracle.c, OpenMP over x-slabs) then evaluates all N^3
translations of it.  The extrema are checked by reading C-10 against the oracle's FULL
grid (check_extremum): the value within tolerance of the oracle's extremum, and the
oracle's value at the GPU's index within tolerance of it too -- a wrong-but-self-consistent
index fails.  Oracle cost on the 16-thread GPU host: torus ~1 min, sweep ~2 min, docking
~15 s.
"""
import numpy as np
import pytest

from synth import make_config
from gpu_helpers import rel_max_err, as_complex, check_extremum

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-4


@pytest.fixture(scope="module")
def bc():
    import torch
    assert torch.cuda.is_available()
    from paper_1711_05075_b200 import ballcorr
    return ballcorr


def correlator(bc, w, **over):
    from paper_1711_05075_b200.presets import correlator_kwargs
    c = bc.Correlator(**correlator_kwargs(w.name, w.N, w.h, w.t0, w.weights, **over))
    c.shape_upload(0, w.A_xyzr, w.A_w)
    c.shape_upload(1, w.B_xyzr, w.B_w)
    c.spectrum_A()
    return c


def test_torus_full_grid_best_rotation(bc, oracle_mod):
    w = make_config("torus")                       # 64 rotations
    c = correlator(bc, w)
    mm = c.correlate_rotations(w.R, "minmax")
    r = int(np.argmax(mm[:, 1]["val"]))            # the rotation with the largest overlap
    f = c.correlate_rotations(w.R[r:r + 1], "full")[0]
    ref = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[r], w.N, w.h, w.t0)
    tol = TOL_F32 * np.abs(ref).max()
    assert rel_max_err(f, ref) <= TOL_F32, (r, rel_max_err(f, ref))
    check_extremum(mm[r, 1]["val"], mm[r, 1]["idx"], ref, "max", tol)
    check_extremum(mm[r, 0]["val"], mm[r, 0]["idx"], ref, "min", tol)


def test_sweep_full_grid_best_rotation(bc, oracle_mod):
    w = make_config("sweep")                       # 512 rotations, the bench's call
    c = correlator(bc, w)
    red = c.correlate_rotations(w.R, "min_argmin")
    r = int(np.argmin(red["val"]))                 # the best-scoring rotation of the output
    mm = c.correlate_rotations(w.R[r:r + 1], "minmax")[0]
    assert mm[0]["val"] == red[r]["val"] and mm[0]["idx"] == red[r]["idx"]
    f = c.correlate_rotations(w.R[r:r + 1], "full")[0]
    ref = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[r], w.N, w.h, w.t0)
    tol = TOL_F32 * np.abs(ref).max()
    assert rel_max_err(f, ref) <= TOL_F32, (r, rel_max_err(f, ref))
    check_extremum(red[r]["val"], red[r]["idx"], ref, "min", tol)
    check_extremum(mm[1]["val"], mm[1]["idx"], ref, "max", tol)


def test_docking_full_grid_best_rotation(bc, oracle_mod):
    w = make_config("docking", n_rot=360)          # a tenth of the config's 3,600
    c = correlator(bc, w)
    best = c.correlate_rotations(w.R, "max_real")
    r = int(np.argmax(best["val"]))                # the best docking score over the rotations
    f = as_complex(c.correlate_rotations(w.R[r:r + 1], "full"))[0]
    ref = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[r], w.N, w.h, w.t0)
    tol = TOL_F32 * np.abs(ref).max()
    assert rel_max_err(f, ref) <= TOL_F32, (r, rel_max_err(f, ref))
    check_extremum(best[r]["val"], best[r]["idx"], ref.real, "max", tol)
