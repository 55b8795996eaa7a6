"""Rotation sharding across ranks (one process per GPU, torch.distributed).

Rotations are independent units: a rank correlates its own block of
rotations with no data-path collective.  Two exchanges sit outside the per-rotation path:
A's band spectrum, computed once by one rank and broadcast to the others (north_star "A's
spectrum broadcast"), and the gather of the tiny per-rotation results (NCCL over NVLink on
the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def rotation_block(n_rot: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [start, stop) of rank `rank`; blocks differ in size by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    base, extra = divmod(n_rot, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def broadcast_spectrum_A(corr, src: int = 0, group=None):
    """Rank `src` computes A's band spectrum (bc_spectrum_A); every rank receives it into its
    context's spectrum buffer (in place, zero copy) and the others import it.  All ranks must
    have uploaded the same shapes with identical parameters.  Collective over `group`."""
    import torch
    import torch.distributed as dist

    if dist.get_rank(group) == src:
        corr.spectrum_A()
    buf = corr.spectrum_A_tensor()
    dist.broadcast(buf, src=src, group=group)
    if buf.is_cuda:
        torch.cuda.synchronize(buf.device)
    if dist.get_rank(group) != src:
        corr.spectrum_A_import()
    return buf.numel() * buf.element_size()


def gather_extrema(local_val: np.ndarray, local_idx: np.ndarray, n_rot: int, group=None, device="cpu"):
    """All-gather per-rotation (val, idx) blocks into global rotation order on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    start, stop = rotation_block(n_rot, rank, world)
    assert len(local_val) == stop - start
    cap = -(-n_rot // world)
    buf = torch.zeros((cap, 2), dtype=torch.float64, device=device)
    buf[: stop - start, 0] = torch.as_tensor(np.asarray(local_val, dtype=np.float64), device=device)
    buf[: stop - start, 1] = torch.as_tensor(np.asarray(local_idx, dtype=np.float64), device=device)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    vals = np.empty(n_rot)
    idxs = np.empty(n_rot, dtype=np.int64)
    for r in range(world):
        s, e = rotation_block(n_rot, r, world)
        blk = out[r].cpu().numpy()
        vals[s:e] = blk[: e - s, 0]
        idxs[s:e] = blk[: e - s, 1].astype(np.int64)
    return vals, idxs


def global_best(vals: np.ndarray, idxs: np.ndarray, kind: str = "min"):
    """(rotation, value, translation index) of the best rotation; ties -> lowest rotation."""
    r = int(np.argmin(vals)) if kind == "min" else int(np.argmax(vals))
    return r, float(vals[r]), int(idxs[r])


# ----------------------------------------------------------------------------- fused exchanges
# (include/ballcorr.h "Fused exchanges over peer memory").  The library does
# the data movement inside its kernels over NVLink; these helpers only move the 64-byte IPC
# handles between the processes and order the steps with barriers.

def _world(group=None):
    """(world size, rank); a process without a process group is a world of one."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def _barrier(group=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier(group=group)


def _exchange_handles(corr, ptr, group=None):
    """Every rank's device pointer for `ptr`'s peer allocation, in rank order (own pointer as
    is, the others mapped through cudaIpc)."""
    import torch.distributed as dist
    world, rank = _world(group)
    if world == 1:
        return [ptr]
    handles = [None] * world
    dist.all_gather_object(handles, corr.ipc_handle(ptr), group=group)
    return [ptr if r == rank else corr.ipc_open(handles[r]) for r in range(world)]


def allreduce_spectrum_A_p2p(corr, n_A: int, group=None, sync=None):
    """A's spectrum sharded by balls: rank g computes the partial spectrum of its contiguous
    block of A's balls, then one kernel per rank reads every rank's partial over peer memory,
    sums them in rank order and builds A'' (bc_spectrum_A_reduce).  Every rank ends with the
    same spectrum bits.  `sync()` waits for the device (torch.cuda.synchronize by default)."""
    if sync is None:
        import torch
        sync = torch.cuda.synchronize
    world, rank = _world(group)
    lo, hi = rotation_block(n_A, rank, world)
    corr.spectrum_A_partial(lo, hi)
    own, _ = corr.spectrum_A_partial_buffer()
    ptrs = _exchange_handles(corr, own, group)
    sync()
    _barrier(group)                    # every partial is complete
    corr.spectrum_A_reduce(ptrs)
    sync()
    _barrier(group)                    # every rank has read every partial
    for r, p in enumerate(ptrs):
        if r != rank:
            corr.ipc_close(p)
    return lo, hi


def result_peers_p2p(corr, global_buf_ptr, n_rot: int, group=None):
    """Fused result exchange: every rank allocates the WHOLE job's record buffer
    (`global_buf_ptr`, n_rot bc_extremum records); the reduction epilogue of each rank then
    stores its rotations' records into every rank's buffer at their global indices
    (bc_set_result_peers), so no all-gather follows the step -- a barrier after the step is
    all the caller needs before reading.  Returns (this rank's rotation block, mapped pointers
    to close at the end)."""
    world, rank = _world(group)
    start, stop = rotation_block(n_rot, rank, world)
    ptrs = _exchange_handles(corr, global_buf_ptr, group)
    corr.set_result_peers(ptrs, base=start)
    return (start, stop), [p for r, p in enumerate(ptrs) if r != rank]
