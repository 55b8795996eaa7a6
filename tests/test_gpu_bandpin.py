"""The sweep plan's specialised kernels pinned to the band-limited reference.

bench.py's headline runs the kernels the plan shape L = Np = 256, c = 4, K = 255 selects:
spread_z_kernel<256, BOX> + pass_z_fast_kernel (spread and z transform of R B),
pass_y_fast_kernel, fold_fast_kernel (x transform, spectral product with A, fold, inverse
x), the inverse y pass and last_tma_kernel<256> (inverse z + reduction).  Their sum is the
Fourier partial sum over the cube band |k_i| <= 255 of the P-periodised f (P = 2), which
oracle.bandlimited_correlation computes by direct fp64 sums (NDFT x ball transform,
product, inverse DFT).  Against it the only differences are
the spreading windows' alias levels (blob <= 6e-6, Gaussian 1e-7 of the band, DESIGN.md
R-1) and fp32 rounding, so the pin is tight: 1e-5 of max|f| (SURVEY.md §8(c) fp32 bar).

Inputs: three balls of the sweep's A and, as B, five balls on the edge of the sweep B's
support (the rotation centre and |b| = 0.2 with the recipe's largest radius) -- the case
whose BAND error against the lens oracle is ~2.5e-4 (tests/test_gpu_edges.py), so the pin
separates implementation error (here) from band error (there).  Oracle ~2 min.
"""
import numpy as np
import pytest

from synth import make_config
from gpu_helpers import rel_max_err, check_extremum

pytestmark = pytest.mark.gpu

IMPL_TOL = 1e-5

EDGE_B = np.array([[0.0, 0.0, 0.0, 0.02], [0.2, 0.0, 0.0, 0.02], [0.0, -0.2, 0.0, 0.005],
                   [0.0, 0.0, 0.2, 0.01], [-0.1155, 0.1155, -0.1155, 0.02]])


@pytest.fixture(scope="module")
def bc():
    import torch
    assert torch.cuda.is_available()
    from paper_1711_05075_b200 import ballcorr
    return ballcorr


def test_sweep_plan_kernels_vs_bandlimited(bc, oracle_mod):
    from paper_1711_05075_b200.presets import correlator_kwargs
    w = make_config("sweep", n_rot=2)
    A = w.A_xyzr[:3]
    r = 1
    P, K = 256 * w.h, 255
    ref = oracle_mod.bandlimited_correlation(A, None, EDGE_B, None, w.R[r], w.N, w.h, w.t0, P, K)
    tol = IMPL_TOL * np.abs(ref).max()
    for generic in (False, True):
        c = bc.Correlator(**correlator_kwargs("sweep", w.N, w.h, w.t0, "real", generic_only=generic))
        c.shape_upload(0, A)
        c.shape_upload(1, EDGE_B)
        c.spectrum_A()
        if not generic:
            assert c.query("fold_fast") == 1 and c.query("fused_spread_z") == 1 and c.query("L_B") == 256
        f = c.correlate_rotations(w.R[r:r + 1], "full")[0]
        err = rel_max_err(f, ref)
        assert err <= IMPL_TOL, (generic, err)
        mm = c.correlate_rotations(w.R[r:r + 1], "minmax")[0]
        check_extremum(mm[1]["val"], mm[1]["idx"], ref, "max", tol)
        check_extremum(mm[0]["val"], mm[0]["idx"], ref, "min", tol)
        c.close()


# Docking plan (L = 384, c = 2, K = 191, Np = 128, complex weights): spread_z_kernel<384, BOX,
# CPLX> + pass_z_dk / pass_y_dk / fold_dk (dock_fast.cu), then the generic inverse passes.  B:
# the docking B's support edge (|b| = 26.6 A, the recipe's largest skin radius 3.2 A, weight 1)
# around a core ball at the rotation centre (weight -15i); A: two core and two skin atoms of the
# docking A.  Oracle ~1 min.
EDGE_B_DK = np.array([[0.0, 0.0, 0.0, 1.7], [26.6, 0.0, 0.0, 3.2], [0.0, -26.6, 0.0, 2.6],
                      [0.0, 0.0, 26.6, 1.2], [-15.3, 15.3, -15.3, 3.2]])
EDGE_WB_DK = np.array([-15j, 1.0, 1.0, -15j, 1.0])


def test_docking_plan_kernels_vs_bandlimited(bc, oracle_mod):
    from paper_1711_05075_b200.presets import correlator_kwargs
    from gpu_helpers import as_complex
    w = make_config("docking", n_rot=2)
    skin = np.flatnonzero(w.A_w == 1.0)[:2]
    core = np.flatnonzero(w.A_w != 1.0)[:2]
    sel = np.concatenate([core, skin])
    A, wA = w.A_xyzr[sel], w.A_w[sel]
    r = 1
    P, K = 128 * w.h, 191
    ref = oracle_mod.bandlimited_correlation(A, wA, EDGE_B_DK, EDGE_WB_DK, w.R[r], w.N, w.h, w.t0, P, K)
    for generic in (False, True):
        c = bc.Correlator(**correlator_kwargs("docking", w.N, w.h, w.t0, "complex", generic_only=generic))
        c.shape_upload(0, A, wA)
        c.shape_upload(1, EDGE_B_DK, EDGE_WB_DK)
        c.spectrum_A()
        if not generic:
            assert c.query("dock_fast") == 1 and c.query("blob_B") == 1 and c.query("L_B") == 384
        f = as_complex(c.correlate_rotations(w.R[r:r + 1], "full"))[0]
        err = np.abs(f - ref).max() / np.abs(ref).max()
        assert err <= IMPL_TOL, (generic, err)
        best = c.correlate_rotations(w.R[r:r + 1], "max_real")[0]
        check_extremum(best["val"], best["idx"], ref.real, "max", IMPL_TOL * np.abs(ref).max())
        c.close()
