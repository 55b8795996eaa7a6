"""The fused exchanges (collectives.cu), data path on one GPU: two
contexts stand in for two ranks and hand each other plain device pointers where the
multi-process run maps peers' allocations through cudaIpc (the protocol itself runs on
gloo in tests/test_sharding.py).

* A's spectrum sharded by balls: each "rank" computes the partial spectrum of half of A's
  balls; bc_spectrum_A_reduce (peer reads fused with the A'' build) gives both the same bits,
  within fp32 rounding of the one-rank spectrum, and the lens oracle agrees at 1e-4.
* Result exchange fused into the reduction epilogue: each "rank" correlates its rotation
  block and its epilogue stores the records straight into the job-wide buffer at their
  global indices -- bitwise the one-rank records, with no gather.
"""
import numpy as np
import pytest

from synth import make_config
from gpu_helpers import rel_max_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bc():
    import torch
    assert torch.cuda.is_available()
    from paper_1711_05075_b200 import ballcorr
    return ballcorr


@pytest.fixture(scope="module")
def sweep():
    return make_config("sweep", n_rot=12)


def ctx_for(bc, w):
    from paper_1711_05075_b200.presets import correlator_kwargs
    c = bc.Correlator(**correlator_kwargs("sweep", w.N, w.h, w.t0, w.weights))
    c.shape_upload(0, w.A_xyzr, w.A_w)
    c.shape_upload(1, w.B_xyzr, w.B_w)
    return c


def test_sharded_spectrum_reduced_over_peers(bc, oracle_mod, sweep):
    import torch
    w = sweep
    nA = len(w.A_xyzr)
    ranks = [ctx_for(bc, w) for _ in range(2)]
    blocks = [(0, nA // 2), (nA // 2, nA)]
    for c, (lo, hi) in zip(ranks, blocks):
        c.spectrum_A_partial(lo, hi)
    parts = [c.spectrum_A_partial_buffer()[0] for c in ranks]
    torch.cuda.synchronize()
    for c in ranks:
        c.spectrum_A_reduce(parts)          # the fused all-reduce + A'' build
    torch.cuda.synchronize()
    full = ctx_for(bc, w)
    full.spectrum_A()
    # the reduced spectra are bitwise equal on every rank and match the one-rank spectrum
    s0 = ranks[0].spectrum_A_tensor().clone()
    s1 = ranks[1].spectrum_A_tensor().clone()
    assert torch.equal(s0, s1)
    sf = full.spectrum_A_tensor()
    assert (s0 - sf).abs().max().item() <= 1e-5 * sf.abs().max().item()
    R = w.R[:3]
    f0 = ranks[0].correlate_rotations(R, "full")
    f1 = ranks[1].correlate_rotations(R, "full")
    ff = full.correlate_rotations(R, "full")
    assert np.array_equal(f0, f1)
    for r in range(3):
        assert rel_max_err(f0[r], ff[r]) <= 1e-5
    rng = np.random.default_rng(2)
    flat = f0[1].reshape(-1)
    idx = np.unique(np.concatenate([rng.choice(flat.size, 60, replace=False), np.argpartition(flat, -30)[-30:]]))
    ref = oracle_mod.correlate_points(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, R[1], w.N, w.h, w.t0, idx)
    assert np.abs(flat[idx] - ref).max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("kind", ["min_argmin", "minmax"])
def test_results_stored_into_peers_by_the_epilogue(bc, sweep, kind):
    import torch
    w = sweep
    per = 2 if kind == "minmax" else 1
    n = w.n_rot
    ranks = [ctx_for(bc, w) for _ in range(2)]
    for c in ranks:
        c.spectrum_A()
    glob = [torch.zeros(n * per * 16, dtype=torch.uint8, device="cuda") for _ in range(2)]
    from paper_1711_05075_b200.sharding import rotation_block
    for g, c in enumerate(ranks):
        s, e = rotation_block(n, g, 2)
        c.set_result_peers([b.data_ptr() for b in glob], base=s)
        local = torch.empty((e - s) * per * 16, dtype=torch.uint8, device="cuda")
        c.correlate_rotations(torch.tensor(w.R[s:e], device="cuda"), kind, out=local)
    torch.cuda.synchronize()
    one = ctx_for(bc, w)
    one.spectrum_A()
    ref = one.correlate_rotations(w.R, kind)
    for b in glob:
        got = bc.extremum_to_numpy(b.cpu().numpy()).reshape(ref.shape)
        assert np.array_equal(got, ref)
    # off again: later calls leave the peers untouched
    ranks[0].set_result_peers([])
    before = glob[0].clone()
    ranks[0].correlate_rotations(w.R[:2], kind)
    torch.cuda.synchronize()
    assert torch.equal(glob[0], before)


def test_ipc_handle_of_a_device_buffer(bc, sweep):
    import torch
    c = ctx_for(bc, sweep)
    ptr, view = c.result_buffer(1 << 20)
    assert view.numel() == 1 << 20 and int(view.sum().item()) == 0
    h = c.ipc_handle(ptr)
    assert isinstance(h, bytes) and len(h) == bc.IPC_HANDLE_BYTES
    # a pointer inside an allocation would map the allocation's base on the peer: refused
    with pytest.raises(bc.BallCorrError) as e:
        c.ipc_handle(ptr + 256)
    assert e.value.status == bc.BC_EINVAL
    with pytest.raises(bc.BallCorrError):
        c.set_result_peers([0])
    with pytest.raises(bc.BallCorrError):
        c.spectrum_A_reduce([])
