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
