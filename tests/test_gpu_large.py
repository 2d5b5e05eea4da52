"""GPU parity at BASELINE's real sizes (configs 3-5) and on the multi-chunk
overlap-add path, against the CPU oracle (objectives.cpp:52-118 restated).

Config 3 (n=1024, M=128, jittered) and config 4 (n=4096, M=256, Poisson) run
in full; config 5 (n=8192, 27,556 patterns) is checked on a sub-problem of
its geometry against the oracle and in full through size-independent
properties (additivity over position subsets, determinism, the shift
identity).  Tolerances: complex64 objective 1e-5 relative, gradient 1e-4
relative L2 (BASELINE.json north_star).
"""
import os

import numpy as np
import pytest

from conftest import rand_field, rel, rel_l2

pytestmark = pytest.mark.gpu

C64_VAL, C64_GRAD = 1e-5, 1e-4


def _r64(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def _case(oracle, cfg, pos=None, n=None, obj=None, seed=5, photons=None):
    """(oracle problem, z, v, float32 data, probe, pos, n) for cfg's geometry."""
    from paper_1810_05628_b200 import synth
    o, probe, p = synth.make_inputs(cfg) if obj is None else (obj, synth.make_probe(cfg.M, cfg.sigma_probe, cfg.a), pos)
    n = cfg.n if n is None else n
    pos = p if pos is None else pos
    probe = _r64(probe)
    o = _r64(o[:n, :n])
    oracle.set_threads(os.cpu_count() or 1)
    data = oracle.simulate(n, cfg.M, cfg.w, pos, o, probe)
    photons = cfg.photons if photons is None else photons
    if photons:
        data = oracle.add_poisson(data, photons, seed=4)
    data = data.astype(np.float32)
    z = _r64(o * 0.9 + 0.05 * rand_field(n, seed))
    v = _r64(0.01 * rand_field(n, seed + 1))
    prob = oracle.Problem(n, cfg.M, cfg.w, pos, data.astype(np.float64), probe)
    return prob, z, v, data, probe, pos, n


def _check(plan, prob, oracle, z, v):
    gv, gg = plan.evaluate(z, v)
    wv, wg = oracle.evaluate(prob, z, v)
    assert rel(gv, wv) <= C64_VAL, (gv, wv)
    assert rel_l2(gg, wg) <= C64_GRAD, rel_l2(gg, wg)
    return gv, gg


def test_config3_full(oracle):
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.CONFIGS[3]
    prob, z, v, data, probe, pos, n = _case(oracle, cfg)
    plan = Plan(n, cfg.M, cfg.w, pos, data, probe, precision="c64")
    _check(plan, prob, oracle, z, v)
    _check(plan, prob, oracle, z, None)
    plan.close()


def test_config4_full(oracle):
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.CONFIGS[4]
    prob, z, v, data, probe, pos, n = _case(oracle, cfg)
    plan = Plan(n, cfg.M, cfg.w, pos, data, probe, precision="c64")
    _check(plan, prob, oracle, z, v)
    plan.close()


def test_config4_device_poisson_matches_oracle_sampler(oracle):
    """The bench's data path (GPU forward operator + GPU Poisson) = the oracle's."""
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.CONFIGS[4]
    obj, probe, pos = synth.make_inputs(cfg)
    sub = pos[:61 * 3]                     # three scan rows
    probe, obj = _r64(probe), _r64(obj)
    plan = Plan(cfg.n, cfg.M, cfg.w, sub, None, probe, precision="c128")
    plan.simulate(obj, copy_out=False)
    plan.add_poisson(cfg.photons, seed=4)
    got = plan.data_host()
    want = oracle.add_poisson(oracle.simulate(cfg.n, cfg.M, cfg.w, sub, obj, probe), cfg.photons, seed=4)
    assert np.isclose(got, want, rtol=1e-9, atol=0).mean() > 0.9999
    plan.close()


@pytest.mark.parametrize("budget_mb", [48, 200])
def test_multichunk_stash_matches_single(oracle, monkeypatch, budget_mb):
    """Stash budget lowered so the overlap-add runs in >= 3 chunks
    (accumulating gathers + separate shift / finalize kernels)."""
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.CONFIGS[3]
    prob, z, v, data, probe, pos, n = _case(oracle, cfg)
    monkeypatch.setenv("PTG_NO_PLANES", "1")
    monkeypatch.setenv("PTG_NO_RMW", "1")
    monkeypatch.setenv("PTG_STASH_BUDGET_MB", str(budget_mb))
    plan = Plan(n, cfg.M, cfg.w, pos, data, probe, precision="c64")
    _check(plan, prob, oracle, z, v)
    _check(plan, prob, oracle, z, None)
    plan.close()


def test_config5_subproblem(oracle):
    """Config 5's probe / step / noise on the top-left 2048^2 window (38 x 38 positions)."""
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.CONFIGS[5]
    S = 2048
    steps = (S - cfg.w) // cfg.step + 1
    obj = synth.make_object(S, cfg.sigma_obj)
    pos = synth.raster(S, cfg.w, steps, cfg.step)
    prob, z, v, data, probe, pos, n = _case(oracle, cfg, pos=pos, n=S, obj=obj)
    plan = Plan(n, cfg.M, cfg.w, pos, data, probe, precision="c64")
    _check(plan, prob, oracle, z, v)
    plan.close()


def test_config5_full_properties():
    """Full config 5 on the GPU: (1) bitwise determinism, (2) additivity: the
    evaluation over all 27,556 positions equals the sum of the evaluations
    over the even and odd scan rows, (3) the MG/OPT shift identity
    value(v) = value(0) - <v,z>, grad(v) = grad(0) - v."""
    import torch

    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.CONFIGS[5]
    obj, probe, pos = synth.make_inputs(cfg)
    rows = pos.reshape(cfg.steps, cfg.steps, 2)
    plans = []
    for sel in (pos, rows[0::2].reshape(-1, 2), rows[1::2].reshape(-1, 2)):
        p = Plan(cfg.n, cfg.M, cfg.w, sel, None, probe, precision="c64")
        p.simulate(obj, copy_out=False)
        plans.append(p)
    g = torch.Generator(device="cpu").manual_seed(3)
    z = (torch.from_numpy(obj).to(torch.complex64) * 0.9).cuda()
    z += 0.05 * torch.complex(torch.rand(cfg.n, cfg.n, generator=g) - 0.5,
                              torch.rand(cfg.n, cfg.n, generator=g) - 0.5).cuda()
    grads = [torch.empty_like(z) for _ in plans]
    torch.cuda.synchronize()   # the plans run on their own streams: z / v must be written first
    vals = [p.evaluate_device(z, gr) for p, gr in zip(plans, grads)]
    # (1) determinism
    g2 = torch.empty_like(z)
    assert plans[0].evaluate_device(z, g2) == vals[0]
    assert torch.equal(g2, grads[0])
    # (2) additivity
    assert rel(vals[0], vals[1] + vals[2]) <= 1e-6
    gsum = grads[1] + grads[2]
    assert float(torch.linalg.vector_norm(grads[0] - gsum) / torch.linalg.vector_norm(grads[0])) <= 1e-5
    # (3) shift
    v = 0.01 * torch.complex(torch.rand(cfg.n, cfg.n, generator=g), torch.rand(cfg.n, cfg.n, generator=g)).cuda()
    gv = torch.empty_like(z)
    torch.cuda.synchronize()
    val_v = plans[0].evaluate_device(z, gv, v=v)
    dot = float(torch.sum(v.real.double() * z.real.double() + v.imag.double() * z.imag.double()))
    assert rel(val_v, vals[0] - dot) <= 1e-9
    assert float(torch.linalg.vector_norm(gv - (grads[0] - v)) / torch.linalg.vector_norm(gv)) <= 1e-6
    for p in plans:
        p.close()


# ------------------------------------------------ RMW overlap-add (frame_rmw.cuh)
@pytest.mark.parametrize("M,steps,step,jitter,metric,rmw2", [(128, 6, 40, 0, 0, 0), (128, 7, 24, 2, 0, 0),
                                                             (256, 4, 48, 0, 0, 0), (256, 5, 64, 3, 0, 0),
                                                             (256, 4, 48, 0, 1, 0), (256, 5, 48, 3, 0, 1),
                                                             (256, 4, 48, 0, 1, 1)])
def test_rmw_matches_oracle(oracle, monkeypatch, M, steps, step, jitter, metric, rmw2):
    """The persistent dependency-ordered RMW path (forced for small problems
    with PTG_NO_PLANES=1): odd window columns (jitter), both metrics, shift."""
    from paper_1810_05628_b200 import Plan, synth
    n = (steps - 1) * step + M + 2 * jitter + 6
    cfg = synth.Config(0, n, M, steps, step, 6.0, M / 4, 0.001, "c64", jitter=jitter)
    obj, probe, pos = synth.make_inputs(cfg)
    probe, obj = _r64(probe), _r64(obj)
    data = oracle.simulate(n, M, M, pos, obj, probe).astype(np.float32)
    z = _r64(obj * 0.9 + 0.05 * rand_field(n, 7))
    v = _r64(0.01 * rand_field(n, 8))
    prob = oracle.Problem(n, M, M, pos, data.astype(np.float64), probe, metric)
    monkeypatch.setenv("PTG_NO_PLANES", "1")
    monkeypatch.setenv("PTG_RMW", "1")
    monkeypatch.setenv("PTG_RMW2", str(rmw2))   # frame_rmw2_kernel (two threads per line)
    plan = Plan(n, M, M, pos, data, probe, precision="c64")
    for vv in (v, None):
        gv, gg = plan.evaluate(z, vv, metric=metric)
        wv, wg = oracle.evaluate(prob, z, vv)
        assert rel(gv, wv) <= C64_VAL, (gv, wv)
        assert rel_l2(gg, wg) <= C64_GRAD, rel_l2(gg, wg)
    # bitwise reproducible run to run (fixed dependency-ordered summation)
    g1 = plan.evaluate(z, v, metric=metric)
    g2 = plan.evaluate(z, v, metric=metric)
    assert g1[0] == g2[0] and np.array_equal(g1[1], g2[1])
    plan.close()


@pytest.mark.parametrize("jitter,metric", [(0, 0), (3, 0), (0, 1)])
def test_rmw_tensor_memory_cache_bitwise(oracle, monkeypatch, jitter, metric):
    """M = 256 RMW frames keep the probe rows and the next object window in
    tensor memory (tcgen05.st / tcgen05.ld as thread-private storage).  With
    PTG_RMW_TMEM=0 the same kernel reads them from L2 instead: identical
    arithmetic, so value and gradient must agree bit for bit (odd window
    columns through jitter, both metrics, a shift)."""
    from paper_1810_05628_b200 import Plan, synth
    M, steps, step = 256, 5, 48
    n = (steps - 1) * step + M + 2 * jitter + 6
    cfg = synth.Config(0, n, M, steps, step, 6.0, M / 4, 0.001, "c64", jitter=jitter)
    obj, probe, pos = synth.make_inputs(cfg)
    probe, obj = _r64(probe), _r64(obj)
    data = oracle.simulate(n, M, M, pos, obj, probe).astype(np.float32)
    z = _r64(obj * 0.9 + 0.05 * rand_field(n, 7))
    v = _r64(0.01 * rand_field(n, 8))
    monkeypatch.setenv("PTG_NO_PLANES", "1")
    monkeypatch.setenv("PTG_RMW", "1")
    import torch
    plan = Plan(n, M, M, pos, data, probe, precision="c64")
    zt = torch.from_numpy(z.astype(np.complex64)).cuda()
    vt = torch.from_numpy(v.astype(np.complex64)).cuda()

    def run():   # device buffers: plain launches (no replayed host-evaluation graph)
        gt = torch.empty_like(zt)
        val = plan.evaluate_device(zt, gt, vt, metric=metric)
        return val, gt.cpu().numpy().astype(np.complex128)

    on = run()
    monkeypatch.setenv("PTG_RMW_TMEM", "0")
    off = run()
    monkeypatch.delenv("PTG_RMW_TMEM")
    again = run()
    assert on[0] == off[0] == again[0]
    assert np.array_equal(on[1], off[1]) and np.array_equal(on[1], again[1])
    prob = oracle.Problem(n, M, M, pos, data.astype(np.float64), probe, metric)
    wv, wg = oracle.evaluate(prob, z, v)
    assert rel(on[0], wv) <= C64_VAL and rel_l2(on[1], wg) <= C64_GRAD
    plan.close()


@pytest.mark.parametrize("steps,step,jitter,metric,tmem", [(6, 40, 0, 0, "1"), (7, 24, 2, 0, "1"), (6, 40, 0, 1, "1"),
                                                            (7, 24, 2, 0, "0")])
def test_fused_cta_m128_bitwise_vs_cluster(oracle, monkeypatch, steps, step, jitter, metric, tmem):
    """M = 128 RMW frames as ONE persistent 512-thread CTA per SM (PTG_SC=1,
    frame_sc.cuh: the four-CTA cluster fused, tensor-memory probe / window
    cache; an A/B variant, measured slower).  Same work split and arithmetic
    as frame_rmw_kernel<4, 32>, so value and gradient agree bit for bit; both
    match the oracle."""
    import torch

    from paper_1810_05628_b200 import Plan, synth
    M = 128
    n = (steps - 1) * step + M + 2 * jitter + 6
    cfg = synth.Config(0, n, M, steps, step, 6.0, M / 4, 0.001, "c64", jitter=jitter)
    obj, probe, pos = synth.make_inputs(cfg)
    probe, obj = _r64(probe), _r64(obj)
    data = oracle.simulate(n, M, M, pos, obj, probe).astype(np.float32)
    z = _r64(obj * 0.9 + 0.05 * rand_field(n, 7))
    v = _r64(0.01 * rand_field(n, 8))
    monkeypatch.setenv("PTG_NO_PLANES", "1")
    monkeypatch.setenv("PTG_RMW", "1")
    monkeypatch.setenv("PTG_RMW_TMEM", tmem)
    plan = Plan(n, M, M, pos, data, probe, precision="c64")
    zt = torch.from_numpy(z.astype(np.complex64)).cuda()
    vt = torch.from_numpy(v.astype(np.complex64)).cuda()

    def run():
        gt = torch.empty_like(zt)
        val = plan.evaluate_device(zt, gt, vt, metric=metric)
        return val, gt.cpu().numpy().astype(np.complex128)

    monkeypatch.setenv("PTG_SC", "1")
    fused = run()
    monkeypatch.setenv("PTG_SC", "0")
    cluster = run()
    monkeypatch.setenv("PTG_SC", "1")
    again = run()
    assert fused[0] == cluster[0] == again[0]
    assert np.array_equal(fused[1], cluster[1]) and np.array_equal(fused[1], again[1])
    prob = oracle.Problem(n, M, M, pos, data.astype(np.float64), probe, metric)
    wv, wg = oracle.evaluate(prob, z, v)
    assert rel(fused[0], wv) <= C64_VAL and rel_l2(fused[1], wg) <= C64_GRAD
    plan.close()


def test_rmw_two_plans_concurrent_streams(oracle, monkeypatch):
    """Two M = 256 RMW plans evaluated at the same time on two streams: both
    persistent kernels want every SM's shared memory and tensor-memory columns,
    so their clusters share the machine in whatever mix the scheduler finds.
    The dispatch protocol (a frame is claimed only by a running cluster) and
    the TMEM allocation must neither deadlock nor change a bit of the result."""
    import torch

    from paper_1810_05628_b200 import Plan, synth
    M, steps, step = 256, 6, 48
    n = (steps - 1) * step + M + 12
    monkeypatch.setenv("PTG_NO_PLANES", "1")
    monkeypatch.setenv("PTG_RMW", "1")
    plans, zs, streams, want = [], [], [], []
    for seed in (7, 9):
        cfg = synth.Config(0, n, M, steps, step, 6.0, M / 4, 0.001, "c64", jitter=3 if seed == 9 else 0)
        obj, probe, pos = synth.make_inputs(cfg)
        probe, obj = _r64(probe), _r64(obj)
        data = oracle.simulate(n, M, M, pos, obj, probe).astype(np.float32)
        z = _r64(obj * 0.9 + 0.05 * rand_field(n, seed))
        plan = Plan(n, M, M, pos, data, probe, precision="c64")
        st = torch.cuda.Stream()
        plan.set_stream(st.cuda_stream)
        zt = torch.from_numpy(z.astype(np.complex64)).cuda()
        gt = torch.empty_like(zt)
        torch.cuda.synchronize()
        val = plan.evaluate_device(zt, gt)          # alone
        want.append((val, gt.cpu().numpy().copy()))
        plans.append(plan)
        zs.append(zt)
        streams.append(st)
    for _ in range(3):
        outs = [torch.empty_like(zs[0]), torch.empty_like(zs[1])]
        vals = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
        torch.cuda.synchronize()
        for i in (0, 1):                            # both enqueued before either finishes
            for _ in range(4):
                plans[i].evaluate_device(zs[i], outs[i], value_dev=vals[i], sync_value=False)
        torch.cuda.synchronize()
        for i in (0, 1):
            assert float(vals[i].cpu()[0]) == want[i][0]
            assert np.array_equal(outs[i].cpu().numpy(), want[i][1])
    for p in plans:
        p.close()


def test_rmw_matches_stash_path(oracle, monkeypatch):
    """Config-3 geometry: RMW and stash + gather agree (different summation
    orders of the same contributions)."""
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.CONFIGS[3]
    prob, z, v, data, probe, pos, n = _case(oracle, cfg)
    monkeypatch.setenv("PTG_NO_PLANES", "1")
    monkeypatch.setenv("PTG_RMW", "1")
    a = Plan(n, cfg.M, cfg.w, pos, data, probe, precision="c64")
    monkeypatch.delenv("PTG_RMW")
    monkeypatch.setenv("PTG_NO_RMW", "1")
    b = Plan(n, cfg.M, cfg.w, pos, data, probe, precision="c64")
    va, ga = a.evaluate(z, v)
    vb, gb = b.evaluate(z, v)
    assert rel(va, vb) <= 1e-6 and rel_l2(ga, gb) <= 1e-5
    a.close()
    b.close()


@pytest.mark.parametrize("bands", ["1", "3", "8"])
def test_rmw_banded_host_eval_bitwise(oracle, monkeypatch, bands):
    """ptg_eval with host buffers on an RMW plan (banded upload / per-band
    launches / early download) = the device evaluation, bitwise."""
    import torch

    from paper_1810_05628_b200 import Plan, synth
    M, steps, step = 256, 5, 48
    n = (steps - 1) * step + M + 40
    cfg = synth.Config(0, n, M, steps, step, 6.0, M / 4, 0.001, "c64", jitter=3)
    obj, probe, pos = synth.make_inputs(cfg)
    probe, obj = _r64(probe), _r64(obj)
    data = oracle.simulate(n, M, M, pos, obj, probe).astype(np.float32)
    z = _r64(obj * 0.9 + 0.05 * rand_field(n, 7))
    monkeypatch.setenv("PTG_NO_PLANES", "1")
    monkeypatch.setenv("PTG_RMW", "1")
    monkeypatch.setenv("PTG_RMW_BANDS", bands)
    plan = Plan(n, M, M, pos, data, probe, precision="c64")
    hv, hg = plan.evaluate(z)
    zt = torch.from_numpy(z.astype(np.complex64)).cuda()
    gt = torch.empty_like(zt)
    torch.cuda.synchronize()
    dv = plan.evaluate_device(zt, gt)
    assert hv == dv
    assert np.array_equal(hg, gt.cpu().numpy().astype(np.complex128))
    prob = oracle.Problem(n, M, M, pos, data.astype(np.float64), probe)
    wv, wg = oracle.evaluate(prob, z)
    assert rel(hv, wv) <= C64_VAL and rel_l2(hg, wg) <= C64_GRAD
    plan.close()
