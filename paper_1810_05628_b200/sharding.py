"""Scan-position sharding across GPUs (one process per GPU).

The objective is a sum over scan positions (objectives.cpp:59-72), so the
path shards by positions with the object replicated: rank r evaluates the
patterns of a contiguous block of scan ROWS (its gradient support is a
horizontal band of the object), then the partial gradients and misfits are
summed with one allreduce — the path's only exchange step.
"""
from __future__ import annotations

import numpy as np


def row_block(rows: int, world: int, rank: int):
    """Contiguous scan rows [lo, hi) owned by `rank` (ceil-balanced)."""
    per = -(-rows // world)
    lo = min(rank * per, rows)
    hi = min((rank + 1) * per, rows)
    return lo, hi


def shard_positions(pos: np.ndarray, row_len: int, world: int, rank: int):
    """Positions (scan order) of `rank`'s row block and their global index range."""
    pos = np.asarray(pos).reshape(-1, 2)
    rows = -(-pos.shape[0] // row_len)
    lo, hi = row_block(rows, world, rank)
    a, b = lo * row_len, min(hi * row_len, pos.shape[0])
    return pos[a:b], (a, b)


def allreduce_eval(value: float, grad, group=None):
    """Sum a shard's (value, gradient) over ranks (torch.distributed; NCCL on GPU,
    gloo on CPU).  grad: torch tensor (complex or real view), reduced in place."""
    import torch
    import torch.distributed as dist
    g = torch.view_as_real(grad) if grad.is_complex() else grad
    dist.all_reduce(g, group=group)
    v = torch.tensor([value], dtype=torch.float64, device=g.device)
    dist.all_reduce(v, group=group)
    return float(v.item()), grad


# ----------------------------------------------------------------- bands
# Band decomposition: rank r owns an n x n square band of a
# tall object whose rows start at r * (n - overlap); consecutive bands share
# `overlap` rows.  Each rank evaluates its own positions on its band (a full
# single-GPU plan), then the gradient rows two bands share are summed with
# their neighbour's (point-to-point, only the halo crosses the interconnect)
# and the misfit with one scalar allreduce.  Per-GPU work is fixed as ranks
# are added (weak scaling of one scanned object).

def band_offset(rank: int, n: int, overlap: int) -> int:
    """Global row of band `rank`'s first row."""
    return rank * (n - overlap)


def halo_exchange(grad, overlap: int, group=None):
    """Sum the `overlap` rows a band shares with each neighbour (in place).

    grad: (n, n) torch tensor (complex or real) of this rank's band.  Both
    neighbours form own + received with IEEE-commutative addition, so the two
    copies of a shared row are bitwise identical."""
    import torch
    import torch.distributed as dist
    if overlap <= 0:
        return grad
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    g = torch.view_as_real(grad) if grad.is_complex() else grad
    n = g.shape[0]
    ops, recv = [], {}
    if rank + 1 < world:   # bottom rows <-> next band's top rows
        send_b = g[n - overlap:].contiguous()
        recv["b"] = torch.empty_like(send_b)
        ops += [dist.P2POp(dist.isend, send_b, rank + 1, group), dist.P2POp(dist.irecv, recv["b"], rank + 1, group)]
    if rank > 0:           # top rows <-> previous band's bottom rows
        send_t = g[:overlap].contiguous()
        recv["t"] = torch.empty_like(send_t)
        ops += [dist.P2POp(dist.isend, send_t, rank - 1, group), dist.P2POp(dist.irecv, recv["t"], rank - 1, group)]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if "b" in recv:
        g[n - overlap:] += recv["b"]
    if "t" in recv:
        g[:overlap] += recv["t"]
    return grad


def allreduce_value(value, group=None):
    """Sum a scalar misfit over ranks; `value` may be a float or a device tensor (in place)."""
    import torch
    import torch.distributed as dist
    if isinstance(value, torch.Tensor):
        dist.all_reduce(value, group=group)
        return value
    v = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(v, group=group)
    return float(v.item())
