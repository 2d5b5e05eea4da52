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


# ------------------------------------------------- fused band exchange
def halo_bytes(n: int, overlap: int, complex_bytes: int) -> int:
    """Bytes of one rank's exchange buffer (csrc/halo.cu layout)."""
    b = 2 * overlap * n * complex_bytes + 8
    return (b + 15) // 16 * 16


class HaloExchange:
    """The band decomposition's one exchange per evaluation as ONE all-gather.

    Every rank packs [top `overlap` rows][bottom `overlap` rows][misfit f64]
    of its band into a small buffer (csrc/halo.cu on the GPU), all buffers are
    all-gathered (NCCL over NVLink; gloo on CPU), and every rank adds its
    neighbours' rows to its own (own + received: the two copies of a shared
    row stay bitwise equal) and sums the misfits in rank order.  On the GPU
    this is two kernel launches and one collective per evaluation instead of
    two point-to-point calls, two adds and a scalar allreduce.
    `val` is a float64 tensor whose element 0 holds this rank's misfit (device
    tensor on GPU); it receives the global misfit.
    """

    def __init__(self, n: int, overlap: int, dtype, device, group=None):
        import torch
        import torch.distributed as dist
        if overlap < 0 or 2 * overlap > n:   # top and bottom halo rows would overlap
            raise ValueError(f"halo: need 0 <= 2 * overlap <= n (overlap {overlap}, n {n})")
        self.n, self.ov, self.group = n, overlap, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.dtype = dtype
        self.cb = torch.empty((), dtype=dtype).element_size()
        self.nbytes = halo_bytes(n, overlap, self.cb)
        self.device = torch.device(device)
        self.cuda = self.device.type == "cuda"
        if self.cuda:
            from paper_1810_05628_b200 import _lib
            self.lib = _lib.lib()
            self.prec = 0 if dtype == torch.complex64 else 1
            assert int(self.lib.ptg_halo_bytes(self.prec, n, overlap)) == self.nbytes
        self.buf = torch.zeros(self.nbytes, dtype=torch.uint8, device=self.device)
        self.all = torch.zeros(self.world * self.nbytes, dtype=torch.uint8, device=self.device)

    # reference restatement of csrc/halo.cu on torch tensors (CPU / tests)
    def pack_torch(self, grad, val):
        import torch
        n, ov, m = self.n, self.ov, self.ov * self.n * self.cb
        b = self.buf
        b[:m] = grad[:ov].contiguous().view(torch.uint8).reshape(-1)
        b[m:2 * m] = grad[n - ov:].contiguous().view(torch.uint8).reshape(-1)
        b[2 * m:2 * m + 8] = val[:1].to(torch.float64).contiguous().view(torch.uint8)

    def unpack_torch(self, grad, val):
        import torch
        n, ov, m = self.n, self.ov, self.ov * self.n * self.cb
        rows = self.all.view(self.world, self.nbytes)
        if self.rank > 0:
            grad[:ov] += rows[self.rank - 1, m:2 * m].clone().view(self.dtype).reshape(ov, n)
        if self.rank + 1 < self.world:
            grad[n - ov:] += rows[self.rank + 1, :m].clone().view(self.dtype).reshape(ov, n)
        s = 0.0
        for r in range(self.world):
            s += float(rows[r, 2 * m:2 * m + 8].clone().view(torch.float64)[0])
        val[0] = s

    def __call__(self, grad, val):
        import torch
        import torch.distributed as dist
        if self.cuda:
            st = torch.cuda.current_stream(self.device).cuda_stream
            rc = self.lib.ptg_halo_pack(self.prec, grad.data_ptr(), self.n, self.ov, val.data_ptr(),
                                        self.buf.data_ptr(), st)
            assert rc == 0, self.lib.ptg_last_error()
            dist.all_gather_into_tensor(self.all, self.buf, group=self.group)
            rc = self.lib.ptg_halo_unpack(self.prec, grad.data_ptr(), self.n, self.ov, self.all.data_ptr(),
                                          self.rank, self.world, val.data_ptr(), st)
            assert rc == 0, self.lib.ptg_last_error()
        else:
            self.pack_torch(grad, val)
            dist.all_gather(list(self.all.view(self.world, self.nbytes).unbind(0)), self.buf, group=self.group)
            self.unpack_torch(grad, val)
        return grad, val
