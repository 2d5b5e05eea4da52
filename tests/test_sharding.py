"""Multi-rank host logic on CPU (gloo, world size 2): position sharding + the
gradient/misfit allreduce reproduce the single-process objective.  The
per-shard evaluator here is the CPU oracle (test infrastructure); on the GPU
box the same code path runs libptg + NCCL (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ptgo
        from paper_1810_05628_b200 import sharding, synth
        cfg = synth.small_config(n=64, M=16, steps=7, step=8)
        obj, probe, pos = synth.make_inputs(cfg)
        data = ptgo.simulate(cfg.n, cfg.M, cfg.w, pos, obj, probe)
        z = np.ones((cfg.n, cfg.n), np.complex128)
        sp, (a, b) = sharding.shard_positions(pos, cfg.steps, world, rank)
        val, g = ptgo.evaluate(ptgo.Problem(cfg.n, cfg.M, cfg.w, sp, data[a:b], probe), z)
        gt = torch.from_numpy(g.copy())
        val, gt = sharding.allreduce_eval(val, gt)
        if rank == 0:
            full = ptgo.evaluate(ptgo.Problem(cfg.n, cfg.M, cfg.w, pos, data, probe), z)
            q.put((val, full[0], float(np.linalg.norm(gt.numpy() - full[1]) / np.linalg.norm(full[1])),
                   (a, b)))
    finally:
        dist.destroy_process_group()


def test_row_blocks_cover_scan():
    from paper_1810_05628_b200 import sharding
    for rows in (1, 7, 29, 166):
        for world in (1, 2, 4, 8):
            spans = [sharding.row_block(rows, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == rows
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


@pytest.mark.timeout(120)
def test_two_rank_allreduce_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(90)
    assert all(p.exitcode == 0 for p in ps)
    val, full_val, grad_rel, span = q.get(timeout=5)
    assert abs(val - full_val) <= 1e-12 * abs(full_val)
    assert grad_rel <= 1e-12


def _band_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ptgo
        from paper_1810_05628_b200 import sharding, synth
        nb, M, s = 40, 16, 8                 # band side, frame, stride
        ov = M - s                           # rows shared by consecutive bands' scans
        H = world * (nb - ov) + ov           # global rows; the scan uses columns [0, nb)
        obj = synth.make_object(H, 2.0)
        probe = synth.make_probe(M, 4.0, 0.01)
        loc = np.array([[r, c] for r in range(0, nb - M + 1, s) for c in range(0, nb - M + 1, s)], np.int32)
        glob = np.concatenate([loc + [sharding.band_offset(b, nb, ov), 0] for b in range(world)])
        data = ptgo.simulate(H, M, M, glob, obj, probe)
        z = obj * 0.9 + 0.05
        off = sharding.band_offset(rank, nb, ov)
        k = loc.shape[0]
        band = np.ascontiguousarray(z[off:off + nb, :nb])
        val, g = ptgo.evaluate(ptgo.Problem(nb, M, M, loc, data[rank * k:(rank + 1) * k], probe), band)
        gt = torch.from_numpy(g.copy())
        sharding.halo_exchange(gt, ov)
        val = sharding.allreduce_value(val)
        full_val, full_g = ptgo.evaluate(ptgo.Problem(H, M, M, glob, data, probe), z)
        want = full_g[off:off + nb, :nb]
        q.put((rank, val, full_val, float(np.linalg.norm(gt.numpy() - want) / np.linalg.norm(want))))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("world", [2, 3])
def test_band_decomposition_matches_global_object(world):
    """Weak-scaling layout: each rank evaluates its own band; halo rows summed
    point-to-point with the neighbours reproduce the global gradient."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_band_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(150)
    assert all(p.exitcode == 0 for p in ps)
    for _ in range(world):
        rank, val, full_val, grad_rel = q.get(timeout=5)
        assert abs(val - full_val) <= 1e-12 * abs(full_val)
        assert grad_rel <= 1e-12


def _fused_band_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ptgo
        from paper_1810_05628_b200 import sharding, synth
        nb, M, s = 40, 16, 8
        ov = M - s
        H = world * (nb - ov) + ov
        obj = synth.make_object(H, 2.0)
        probe = synth.make_probe(M, 4.0, 0.01)
        loc = np.array([[r, c] for r in range(0, nb - M + 1, s) for c in range(0, nb - M + 1, s)], np.int32)
        glob = np.concatenate([loc + [sharding.band_offset(b, nb, ov), 0] for b in range(world)])
        data = ptgo.simulate(H, M, M, glob, obj, probe)
        z = obj * 0.9 + 0.05
        off = sharding.band_offset(rank, nb, ov)
        k = loc.shape[0]
        band = np.ascontiguousarray(z[off:off + nb, :nb])
        val, g = ptgo.evaluate(ptgo.Problem(nb, M, M, loc, data[rank * k:(rank + 1) * k], probe), band)
        gt = torch.from_numpy(g.copy())
        vt = torch.tensor([val, 0.0], dtype=torch.float64)
        ex = sharding.HaloExchange(nb, ov, gt.dtype, "cpu")
        ex(gt, vt)
        full_val, full_g = ptgo.evaluate(ptgo.Problem(H, M, M, glob, data, probe), z)
        want = full_g[off:off + nb, :nb]
        # the rows shared with a neighbour must be bitwise equal on both ranks
        shared = [gt[:ov].numpy().copy(), gt[nb - ov:].numpy().copy()]
        q.put((rank, float(vt[0]), full_val, float(np.linalg.norm(gt.numpy() - want) / np.linalg.norm(want)),
               shared))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("world", [2, 3])
def test_fused_halo_exchange_matches_global_object(world):
    """The band exchange as one all-gather (sharding.HaloExchange, the layout of
    csrc/halo.cu): the exchanged gradients equal the global gradient's rows, the
    misfit is the global misfit, and shared rows are bitwise equal on both sides."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_fused_band_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(150)
    assert all(p.exitcode == 0 for p in ps)
    got = {}
    for _ in range(world):
        rank, val, full_val, grad_rel, shared = q.get(timeout=5)
        assert abs(val - full_val) <= 1e-12 * abs(full_val)
        assert grad_rel <= 1e-12
        got[rank] = shared
    for r in range(world - 1):
        assert np.array_equal(got[r][1], got[r + 1][0])


# --------------------------------------------- libptg's band partition (CPU)
def _shard_band_worker(rank, world, port, q):
    """Rank r: the library's partition (ptg_shard_layout) of the global scan;
    its positions evaluated (CPU oracle) on the whole object; its band rows
    [row0, row0 + rows) kept; halo rows sent to rank r + 1 (gloo) and added
    there -- the exchange libptg's BANDS layout performs with NCCL.  The own
    rows must equal the global gradient's rows; the misfits sum to the value."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ptgo
        from paper_1810_05628_b200 import shard_layout, synth
        cfg = synth.small_config(n=96, M=16, steps=11, step=8, jitter=1)
        obj, probe, pos = synth.make_inputs(cfg)
        data = ptgo.simulate(cfg.n, cfg.M, cfg.w, pos, obj, probe)
        z = obj * 0.9 + 0.01
        L = shard_layout(cfg.n, cfg.w, pos, world, rank, "bands")
        a, b, r0, rows, own, hprev = (L[k] for k in ("pos_begin", "pos_end", "row0", "rows", "own_rows", "halo_prev"))
        val, g = ptgo.evaluate(ptgo.Problem(cfg.n, cfg.M, cfg.w, pos[a:b], data[a:b], probe), z)
        band = torch.from_numpy(g[r0:r0 + rows].copy())
        # nothing outside the band (the layout's promise)
        assert np.abs(np.delete(g, np.s_[r0:r0 + rows], axis=0)).max(initial=0.0) == 0.0
        if rank + 1 < world:
            dist.send(band[own:].contiguous(), rank + 1)
        if rank > 0 and hprev:
            buf = torch.empty((hprev, cfg.n), dtype=band.dtype)
            dist.recv(buf, rank - 1)
            band[:hprev] += buf
        v = torch.tensor([val], dtype=torch.float64)
        dist.all_reduce(v)
        full_v, full_g = ptgo.evaluate(ptgo.Problem(cfg.n, cfg.M, cfg.w, pos, data, probe), z)
        err = float(np.linalg.norm(band[:own].numpy() - full_g[r0:r0 + own]) / max(np.linalg.norm(full_g[r0:r0 + own]), 1e-300))
        q.put((rank, float(v.item()), full_v, err, (a, b, r0, rows, own)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("world", [2, 3])
def test_band_layout_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_shard_band_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=150) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    spans = [r[4] for r in res]
    assert spans[0][0] == 0 and spans[-1][1] == 121                       # every position once
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    assert spans[0][2] == 0 and sum(s[4] for s in spans) == 96              # own rows tile the object
    for _, v, fv, err, _ in res:
        assert abs(v - fv) <= 1e-12 * abs(fv)
        assert err <= 1e-12


def test_shard_layout_rejects_bad_partitions():
    from paper_1810_05628_b200 import ConfigError, shard_layout, synth
    pos = synth.raster(64, 16, 7, 8)
    with pytest.raises(ConfigError):
        shard_layout(64, 16, pos, 8, 0, "bands")      # 7 scan rows for 8 ranks
    dense = synth.raster(64, 16, 13, 4)               # step 4: halo 12 rows
    with pytest.raises(ConfigError):
        shard_layout(64, 16, dense, 13, 0, "bands")   # one 4-row scan row per rank < the 12-row halo
    ok = shard_layout(64, 16, dense, 3, 1, "bands")
    assert ok["halo_prev"] == 12 and ok["own_rows"] >= 12
    rep = shard_layout(64, 16, pos, 2, 1, "replicated")
    assert rep["row0"] == 0 and rep["rows"] == 64 and rep["pos_begin"] > 0
