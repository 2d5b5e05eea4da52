"""Sharded plans on the GPU (libptg's BANDS / REPLICATED layouts).

Multi-GPU boxes are not available to the test tier, so the ranks of a world
are simulated on one GPU WITHOUT a communicator (each rank's band evaluated
by the real device kernels, the halo exchange restated with torch) -- and the
NCCL path itself runs with a world of one rank (ncclCommInitRank, the
grouped send/recv/allreduce calls of comm.cu)."""
import numpy as np
import pytest

from conftest import rand_field, rel, rel_l2

pytestmark = pytest.mark.gpu


def _r64(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def _problem(oracle, steps=9, step=48, M=256, jitter=0):
    from paper_1810_05628_b200 import synth
    n = (steps - 1) * step + M + 2 * jitter + 8
    cfg = synth.Config(0, n, M, steps, step, 6.0, M / 4, 0.001, "c64", jitter=jitter)
    obj, probe, pos = synth.make_inputs(cfg)
    probe, obj = _r64(probe), _r64(obj)
    data = oracle.simulate(n, M, M, pos, obj, probe).astype(np.float32)
    z = _r64(obj * 0.9 + 0.05 * rand_field(n, 7))
    v = _r64(0.01 * rand_field(n, 8))
    return n, M, pos, probe, data, z, v


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("shift", [False, True])
def test_band_shards_simulated_ranks(oracle, monkeypatch, world, shift):
    import torch

    from paper_1810_05628_b200 import Plan
    # >= 5 scan rows (240 object rows) per rank: a 256-row window's halo must fit
    n, M, pos, probe, data, z, v = _problem(oracle, steps=5 * world + 1, jitter=2 if world == 3 else 0)
    monkeypatch.setenv("PTG_NO_PLANES", "1")
    monkeypatch.setenv("PTG_RMW", "1")
    full = Plan(n, M, M, pos, data, probe, precision="c64")
    zt = torch.from_numpy(z.astype(np.complex64)).cuda()
    vt = torch.from_numpy(v.astype(np.complex64)).cuda() if shift else None
    g_full = torch.empty_like(zt)
    torch.cuda.synchronize()
    val_full = full.evaluate_device(zt, g_full, v=vt)
    bands, total = [], 0.0
    for r in range(world):
        p = Plan.sharded(n, M, M, pos, world, r, "bands", probe=probe, precision="c64")
        info = p.shard
        p.set_data(data[info["pos_begin"]:info["pos_end"]])
        r0, rows = info["row0"], info["rows"]
        zb = zt[r0:r0 + rows].contiguous()
        vb = vt[r0:r0 + rows].contiguous() if shift else None
        gb = torch.empty_like(zb)
        torch.cuda.synchronize()
        total += p.evaluate_device(zb, gb, v=vb)
        bands.append((info, gb))
        p.close()
    for r in range(1, world):   # the exchange: rank r-1's halo rows added to rank r's first rows
        prev, gprev = bands[r - 1]
        info, g = bands[r]
        g[:info["halo_prev"]] += gprev[prev["own_rows"]:]
    for info, g in bands:
        r0, own = info["row0"], info["own_rows"]
        assert float(torch.linalg.vector_norm(g[:own] - g_full[r0:r0 + own]) /
                     torch.linalg.vector_norm(g_full[r0:r0 + own])) <= 1e-5
    assert rel(total, val_full) <= 1e-6
    assert sum(i["own_rows"] for i, _ in bands) == n
    full.close()


def _bcast_identity(x):
    return x


@pytest.mark.parametrize("layout", ["bands", "replicated"])
def test_nccl_one_rank_equals_plain_plan(oracle, monkeypatch, layout):
    """The communicator-bound evaluation with a world of one rank runs the
    NCCL calls (grouped allreduce / send-recv) and returns the plain plan's
    value and gradient bitwise."""
    import torch

    from paper_1810_05628_b200 import Comm, Plan
    n, M, pos, probe, data, z, v = _problem(oracle, steps=6)
    monkeypatch.setenv("PTG_NO_PLANES", "1")
    monkeypatch.setenv("PTG_RMW", "1")
    plain = Plan(n, M, M, pos, data, probe, precision="c64")
    comm = Comm(1, 0, 0, _bcast_identity)
    sh = Plan.sharded(n, M, M, pos, 1, 0, layout, data=data, probe=probe, precision="c64")
    sh.bind_comm(comm)
    for vv in (None, v):
        want_v, want_g = plain.evaluate(z, vv)
        got_v, got_g = sh.evaluate(z, vv)
        if vv is None or layout == "bands":
            assert got_v == want_v and np.array_equal(got_g, want_g)
        else:   # REPLICATED applies the shift after the sum over ranks: (sum - v) vs (-v + sum)
            assert rel(got_v, want_v) <= 1e-12 and rel_l2(got_g, want_g) <= 1e-6
    zt = torch.from_numpy(z.astype(np.complex64)).cuda()
    gt = torch.empty_like(zt)
    torch.cuda.synchronize()
    if layout == "bands":
        sh.sync_halo(zt)   # no neighbours: a no-op
    assert sh.evaluate_device(zt, gt) == plain.evaluate(z)[0]
    sh.close()
    plain.close()
    comm.close()


def test_band_shard_rejects_solvers(oracle):
    from paper_1810_05628_b200 import ConfigError, Plan
    n, M, pos, probe, data, z, v = _problem(oracle, steps=6)
    sh = Plan.sharded(n, M, M, pos, 2, 0, "bands", probe=probe, precision="c64")
    with pytest.raises(ConfigError):
        sh.lbfgs(np.ones((sh.rows, n)), max_iters=1)
    sh.close()
