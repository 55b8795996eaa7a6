"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): rotation blocks and the
all-gather of per-rotation results reproduce the single-rank global order exactly; the
broadcast of A's spectrum has one rank compute it and every other rank import the same bytes."""
import os
import socket

import numpy as np
import pytest

from paper_1711_05075_b200.sharding import rotation_block, gather_extrema, global_best, broadcast_spectrum_A


def test_rotation_blocks_cover_exactly():
    for n in (1, 7, 64, 512, 3600):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s, e = rotation_block(n, r, world)
                assert 0 <= s <= e <= n
                seen.extend(range(s, e))
            assert seen == list(range(n))
            sizes = [rotation_block(n, r, world)[1] - rotation_block(n, r, world)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_global_best_tie_break():
    v = np.array([3.0, 1.0, 1.0, 2.0])
    i = np.array([5, 9, 2, 0])
    assert global_best(v, i, "min") == (1, 1.0, 9)
    assert global_best(v, i, "max") == (0, 3.0, 5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_rot, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(123)
    all_val = rng.normal(size=n_rot)
    all_idx = rng.integers(0, 2 ** 31, size=n_rot)
    s, e = rotation_block(n_rot, rank, world)
    vals, idxs = gather_extrema(all_val[s:e], all_idx[s:e], n_rot)
    ok = bool(np.array_equal(vals, all_val) and np.array_equal(idxs, all_idx))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_rot", [(2, 512), (3, 64), (2, 7)])
def test_gather_extrema_gloo(world, n_rot):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_rot, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=10) for _ in range(world))
    assert all(res[r] for r in range(world)), res
    assert all(p.exitcode == 0 for p in procs)


class _FakeCorrelator:
    """Stands in for ballcorr.Correlator on CPU: a host tensor as the spectrum buffer."""

    def __init__(self, rank):
        import torch
        self.buf = torch.full((1000,), float(-1 - rank))  # garbage that differs per rank
        self.computed = self.imported = 0

    def spectrum_A(self):
        import torch
        self.buf.copy_(torch.arange(1000, dtype=torch.float32) * 0.5)
        self.computed += 1

    def spectrum_A_tensor(self):
        return self.buf

    def spectrum_A_import(self):
        self.imported += 1


def _bcast_worker(rank, world, port, src, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = _FakeCorrelator(rank)
    nbytes = broadcast_spectrum_A(c, src=src)
    ok = bool(torch.equal(c.buf, torch.arange(1000, dtype=torch.float32) * 0.5)) and nbytes == 4000
    ok = ok and (c.computed, c.imported) == ((1, 0) if rank == src else (0, 1))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,src", [(2, 0), (3, 2)])
def test_broadcast_spectrum_gloo(world, src):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bcast_worker, args=(r, world, port, src, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=10) for _ in range(world))
    assert all(res[r] for r in range(world)), res
    assert all(p.exitcode == 0 for p in procs)


class _FakePeerCorrelator:
    """CPU stand-in for the fused-exchange API: 'device pointers' are (rank, name) tokens and
    IPC handles encode them, so the protocol's pointer lists can be checked across ranks."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []
        self.opened, self.closed = [], []

    def spectrum_A_partial(self, lo, hi):
        self.calls.append(("partial", lo, hi))

    def spectrum_A_partial_buffer(self):
        return ("part", self.rank), 0

    def ipc_handle(self, ptr):
        return repr(ptr).encode()

    def ipc_open(self, handle):
        p = ("mapped",) + eval(handle.decode())
        self.opened.append(p)
        return p

    def ipc_close(self, p):
        self.closed.append(p)

    def spectrum_A_reduce(self, ptrs):
        self.calls.append(("reduce", list(ptrs)))

    def set_result_peers(self, ptrs, base=0):
        self.calls.append(("peers", list(ptrs), base))


def _p2p_worker(rank, world, port, n_A, n_rot, q):
    import torch.distributed as dist
    from paper_1711_05075_b200.sharding import allreduce_spectrum_A_p2p, result_peers_p2p
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = _FakePeerCorrelator(rank)
    lo, hi = allreduce_spectrum_A_p2p(c, n_A, sync=lambda: None)
    (s, e), to_close = result_peers_p2p(c, ("glob", rank), n_rot)
    q.put((rank, lo, hi, s, e, c.calls, c.opened, c.closed, to_close))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_protocol_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n_A, n_rot = 50000, 512
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, n_A, n_rot, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = {r[0]: r for r in (q.get(timeout=10) for _ in range(world))}
    assert all(p.exitcode == 0 for p in procs)
    # A's balls and the rotations are covered by contiguous blocks in rank order
    assert [res[r][1] for r in range(world)][0] == 0 and res[world - 1][2] == n_A
    assert all(res[r][2] == res[r + 1][1] for r in range(world - 1))
    assert all(res[r][4] == res[r + 1][3] for r in range(world - 1)) and res[world - 1][4] == n_rot
    for r in range(world):
        calls = res[r][5]
        assert calls[0] == ("partial", res[r][1], res[r][2])
        # the reduce reads every rank's partial in rank order: own pointer, peers mapped
        expect = [("part", g) if g == r else ("mapped", "part", g) for g in range(world)]
        assert calls[1] == ("reduce", expect)
        # mapped partials are closed after the reduce; the result buffers stay mapped
        assert sorted(res[r][7]) == sorted(p for p in expect if p[0] == "mapped")
        expect_glob = [("glob", g) if g == r else ("mapped", "glob", g) for g in range(world)]
        assert calls[2] == ("peers", expect_glob, res[r][3])
        assert sorted(res[r][8]) == sorted(p for p in expect_glob if p[0] == "mapped")
