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
