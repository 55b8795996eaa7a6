"""A's spectrum moved between contexts (the multi-GPU broadcast of north_star, here between
two contexts on one GPU): a context that imports the bytes another context computed gives
bitwise the same correlation; the state rules of include/ballcorr.h hold."""
import numpy as np
import pytest

from synth import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bc():
    import torch
    assert torch.cuda.is_available()
    from paper_1711_05075_b200 import ballcorr
    return ballcorr


def make(bc, w, **over):
    from paper_1711_05075_b200.presets import correlator_kwargs
    c = bc.Correlator(**correlator_kwargs(w.name, w.N, w.h, w.t0, w.weights, **over))
    c.shape_upload(0, w.A_xyzr, w.A_w)
    c.shape_upload(1, w.B_xyzr, w.B_w)
    return c


@pytest.mark.parametrize("name", ["sweep", "docking"])
def test_imported_spectrum_gives_identical_results(bc, name):
    import torch
    w = make_config(name, n_rot=3)
    src = make(bc, w)
    src.spectrum_A()
    dst = make(bc, w)
    with pytest.raises(bc.BallCorrError) as e:  # nothing imported yet
        dst.correlate_rotations(w.R[:1], "max_real")
    assert e.value.status == bc.BC_ESTATE
    a, b = src.spectrum_A_tensor(), dst.spectrum_A_tensor()
    assert a.numel() == b.numel() and a.data_ptr() != b.data_ptr()
    b.copy_(a)
    torch.cuda.synchronize()
    dst.spectrum_A_import()
    kind = "max_real" if w.weights == "complex" else "minmax"
    assert np.array_equal(src.correlate_rotations(w.R, kind), dst.correlate_rotations(w.R, kind))
    # the buffer pointer is stable, and re-uploading A invalidates the import
    assert dst.spectrum_A_buffer()[0] == b.data_ptr()
    dst.shape_upload(0, w.A_xyzr, w.A_w)
    with pytest.raises(bc.BallCorrError) as e:
        dst.correlate_rotations(w.R[:1], kind)
    assert e.value.status == bc.BC_ESTATE


def test_exact_mode_has_no_spectrum_buffer(bc):
    w = make_config("tiny")
    c = make(bc, w)
    with pytest.raises(bc.BallCorrError) as e:
        c.spectrum_A_buffer()
    assert e.value.status == bc.BC_EUNSUPPORTED
