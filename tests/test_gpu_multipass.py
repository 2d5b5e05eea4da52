"""Frames larger than one CTA (complex64 M = 256 for BASELINE configs 4-5;
complex128 M >= 128, e.g. ref mode at n = 128 / 256) run the three-pass path
(csrc/frame_multipass.cuh).  Parity vs the oracle at the same bars."""
import numpy as np
import pytest

from conftest import rand_field, rel, rel_l2

pytestmark = pytest.mark.gpu


def _case(oracle, precision, n, M, steps, step, jitter=0, metric=0):
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.Config(0, n, M, steps, step, 8.0, M / 4, 0.0006, precision, jitter=jitter)
    obj, probe, pos = synth.make_inputs(cfg)
    z = obj * 0.9 + 0.05 * rand_field(n, 4)
    v = 0.01 * rand_field(n, 5)
    if precision == "c64":
        obj, probe, z, v = (a.astype(np.complex64).astype(np.complex128) for a in (obj, probe, z, v))
    data = oracle.simulate(n, M, M, pos, obj, probe)
    if precision == "c64":
        data = data.astype(np.float32)
    p = oracle.Problem(n, M, M, pos, data.astype(np.float64), probe, metric)
    plan = Plan(n, M, M, pos, data, probe, precision=precision)
    return p, plan, z, v, obj


@pytest.mark.parametrize("metric", [0, 1])
def test_m256_c64_eval(oracle, metric):
    p, plan, z, v, _ = _case(oracle, "c64", 512, 256, 3, 120, jitter=2, metric=metric)
    wv, wg = oracle.evaluate(p, z, v)
    gv, gg = plan.evaluate(z, v, metric=metric)
    assert rel(gv, wv) <= 1e-5
    assert rel_l2(gg, wg) <= 1e-4


@pytest.mark.parametrize("M", [128, 256])
def test_c128_large_frames(oracle, M):
    p, plan, z, v, _ = _case(oracle, "c128", 2 * M, M, 3, M // 2)
    wv, wg = oracle.evaluate(p, z, v)
    gv, gg = plan.evaluate(z, v)
    assert rel(gv, wv) <= 1e-10
    assert rel_l2(gg, wg) <= 1e-10
    assert rel_l2(plan.project_modulus(z, 1), oracle.project_modulus(p, z, 1)) <= 1e-10


def test_ref_mode_n128_vs_oracle(oracle):
    """Config-1 geometry in the reference's full-field model (M = n = 128)."""
    from paper_1810_05628_b200 import Plan, synth
    n, w, s = 128, 32, 8
    pos = synth.raster(n, w, 13, s)
    data = oracle.simulate(n, n, w, pos, rand_field(n, 1))
    z, v = rand_field(n, 2), rand_field(n, 3, 0.1)
    p = oracle.Problem(n, n, w, pos, data)
    plan = Plan(n, n, w, pos, data, None, precision="c128")
    wv, wg = oracle.evaluate(p, z, v)
    gv, gg = plan.evaluate(z, v)
    assert rel(gv, wv) <= 1e-10 and rel_l2(gg, wg) <= 1e-10
    assert rel_l2(plan.project_modulus(z, 7), oracle.project_modulus(p, z, 7)) <= 1e-10
    want = oracle.pie(p, z, 0.2, 1)
    got = plan.pie(z, gamma=0.2, sweeps=1)
    assert rel_l2(got.final_iterate, want.z) <= 1e-10


def test_m256_simulate_and_pie(oracle):
    p, plan, z, v, obj = _case(oracle, "c64", 512, 256, 2, 200)
    got = plan.simulate(obj)
    want = oracle.simulate(p.n, p.M, p.w, p.pos, obj, p.probe)
    assert rel_l2(got, want) <= 2e-6
    z0 = np.ones_like(z)
    w = oracle.pie(oracle.Problem(p.n, p.M, p.w, p.pos, got, p.probe), z0, 0.0, 1)
    g = plan.pie(z0, sweeps=1)
    assert rel_l2(g.final_iterate, w.z) <= 3e-4


def test_m256_mgopt_values(oracle):
    from paper_1810_05628_b200 import Hierarchy
    p, plan, z, v, _ = _case(oracle, "c64", 512, 256, 3, 128)
    z0 = np.ones_like(z)
    want = oracle.Hierarchy(p, 2).driver(z0, budget=1e9, max_cycles=1)
    got = Hierarchy(plan, 2).driver(z0, budget=1e9, max_cycles=1)
    assert got.history.shape == want.history.shape
    np.testing.assert_allclose(got.history[:, 1], want.history[:, 1], rtol=1e-4)


@pytest.mark.parametrize("M", [128, 256])
@pytest.mark.parametrize("with_probe", [True, False])
@pytest.mark.parametrize("metric", [0, 1])
def test_cluster_kernel_c64(oracle, M, with_probe, metric):
    """complex64 M = 128 / 256 run the cluster-split kernel (csrc/frame_cl.cuh):
    complex probe or binary window, both metrics, jittered (odd) positions."""
    from paper_1810_05628_b200 import Plan, synth
    n = 2 * M + 8
    cfg = synth.Config(0, n, M, 3, M // 2 + 3, 8.0, M / 4, 0.0006, "c64", jitter=2)
    obj, probe, pos = synth.make_inputs(cfg)
    probe = probe if with_probe else None
    z = obj * 0.9 + 0.05 * rand_field(n, 6)
    obj, z = obj.astype(np.complex64).astype(np.complex128), z.astype(np.complex64).astype(np.complex128)
    if probe is not None:
        probe = probe.astype(np.complex64).astype(np.complex128)
    data = oracle.simulate(n, M, M, pos, obj, probe).astype(np.float32)
    p = oracle.Problem(n, M, M, pos, data.astype(np.float64), probe, metric)
    plan = Plan(n, M, M, pos, data, probe, precision="c64")
    wv, wg = oracle.evaluate(p, z)
    gv, gg = plan.evaluate(z, metric=metric)
    assert rel(gv, wv) <= 1e-5
    assert rel_l2(gg, wg) <= 1e-4
