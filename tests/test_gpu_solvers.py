"""GPU-resident solvers vs the reference (golden vectors) and the oracle.

complex128: trajectory-level parity (identical per-level evaluation counts and
stop reasons, histories / iterates within 1e-9..1e-10 relative).  complex64:
per-sweep / per-eval tolerances (discrete line-search decisions may flip in
fp32, so counts are only required to match in c128; SURVEY.md 7 hard part 7).
"""
import os

import numpy as np
import pytest

from conftest import rand_field, rel_l2

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def _ref_plan(gold, precision="c128"):
    from paper_1810_05628_b200 import Plan
    n, w, s = (int(v) for v in gold["eval_b_geom"])
    return Plan(n, n, w, gold["eval_b_pos"], gold["eval_b_data"], None, precision=precision), n, w, s


def test_pie_ref_mode_vs_reference(gold):
    plan, n, w, s = _ref_plan(gold)
    r = plan.pie(gold["pie_z0"], gamma=0.1, sweeps=3)
    assert rel_l2(r.final_iterate, gold["pie_z"]) <= 1e-10
    np.testing.assert_allclose(r.history, gold["pie_hist"], rtol=1e-10, atol=1e-12)
    assert r.weighted_evals == gold["pie_meta"][1]


def test_lbfgs_ref_mode_vs_reference(gold):
    plan, n, w, s = _ref_plan(gold)
    r = plan.lbfgs(gold["pie_z0"], v=gold["eval_b_v"], max_iters=6)
    assert r.history.shape == gold["lbfgs_hist"].shape
    np.testing.assert_allclose(r.history[:, 0], gold["lbfgs_hist"][:, 0], rtol=0)   # identical eval counts
    np.testing.assert_allclose(r.history[:, 1:], gold["lbfgs_hist"][:, 1:], rtol=1e-9)
    assert rel_l2(r.final_iterate, gold["lbfgs_z"]) <= 1e-9


@pytest.mark.parametrize("depth", [2, 3])
def test_mgopt_ref_mode_vs_reference(gold, depth):
    from paper_1810_05628_b200 import Hierarchy
    plan, n, w, s = _ref_plan(gold)
    h = Hierarchy(plan, depth, coarsest_max_iters=10)
    r = h.driver(gold[f"mg{depth}_z0"], budget=1e9, max_cycles=3)
    meta = gold[f"mg{depth}_meta"]
    assert r.per_level_evals == [int(x) for x in meta[3:]]
    assert r.weighted_evals == meta[1]
    np.testing.assert_allclose(r.history, gold[f"mg{depth}_hist"], rtol=1e-9)
    assert rel_l2(r.final_iterate, gold[f"mg{depth}_z"]) <= 1e-9


@pytest.mark.parametrize("tag", ["a", "b"])
def test_mgopt_default_settings_vs_reference(tag):
    """north_star: identical iteration counts for fixed-iteration runs, here at
    the reference's DEFAULT MG/OPT settings (depth 3 => coarsest solve of 100
    LBFGS iterations, multigrid.cpp:123-128) on noisy data; golden produced by
    the unmodified reference (tests/golden/make_mg_default_golden.py)."""
    from paper_1810_05628_b200 import Hierarchy, Plan
    gold = dict(np.load(os.path.join(os.path.dirname(GOLD), "mg_default_golden.npz")))
    n, w, s, depth = (int(v) for v in gold[f"{tag}_geom"])
    plan = Plan(n, n, w, gold[f"{tag}_pos"], gold[f"{tag}_data"], None, precision="c128")
    h = Hierarchy(plan, depth)
    r = h.driver(gold[f"{tag}_z0"], budget=1e9, max_cycles=3)
    meta = gold[f"{tag}_meta"]
    # identical counts at every level; the trajectory itself (three cycles,
    # ~180 coarsest LBFGS iterations with a 25-pair history) amplifies the
    # 1e-16 differences between FFT summation orders to ~1e-7 (measured
    # 8.5e-8 on case b), so values / iterate are held to 1e-6 here -- the
    # 1e-9..1e-10 bars are pinned by the short-trajectory tests above
    assert r.per_level_evals == [int(x) for x in meta[3:]]
    assert r.weighted_evals == meta[1]
    np.testing.assert_allclose(r.history, gold[f"{tag}_hist"], rtol=1e-6)
    assert rel_l2(r.final_iterate, gold[f"{tag}_z"]) <= 1e-6


def _patch(oracle, precision, cfg=None):
    from paper_1810_05628_b200 import Plan, synth
    cfg = cfg or synth.small_config(precision=precision)
    obj, probe, pos = synth.make_inputs(cfg)
    if precision == "c64":
        obj = obj.astype(np.complex64).astype(np.complex128)
        probe = probe.astype(np.complex64).astype(np.complex128)
    data = oracle.simulate(cfg.n, cfg.M, cfg.w, pos, obj, probe)
    if precision == "c64":
        data = data.astype(np.float32)
    p = oracle.Problem(cfg.n, cfg.M, cfg.w, pos, data.astype(np.float64), probe)
    plan = Plan(cfg.n, cfg.M, cfg.w, pos, data, probe, precision=precision)
    return p, plan, cfg


def test_pie_patch_c128_vs_oracle(oracle):
    p, plan, cfg = _patch(oracle, "c128")
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    want = oracle.pie(p, z0, 0.05, 2)
    got = plan.pie(z0, gamma=0.05, sweeps=2)
    assert rel_l2(got.final_iterate, want.z) <= 1e-10
    np.testing.assert_allclose(got.history, want.history, rtol=1e-10)


def test_pie_config2_c64_vs_oracle(oracle):
    from paper_1810_05628_b200 import synth
    p, plan, cfg = _patch(oracle, "c64", synth.CONFIGS[2])
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    want = oracle.pie(p, z0, 0.0, 1)
    got = plan.pie(z0, gamma=0.0, sweeps=1)
    # 841 strictly sequential fp32 projections: per-projection rounding (~1e-6)
    # accumulates along the sweep, so the iterate tolerance is 3e-4 while the
    # objective values stay within the 1e-5 complex64 bar
    assert rel_l2(got.final_iterate, want.z) <= 3e-4
    np.testing.assert_allclose(got.history[:, 1], want.history[:, 1], rtol=1e-5)


def test_mgopt_patch_c128_vs_oracle(oracle):
    from paper_1810_05628_b200 import Hierarchy
    p, plan, cfg = _patch(oracle, "c128")
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    want = oracle.Hierarchy(p, 2).driver(z0, budget=1e9, max_cycles=3)
    got = Hierarchy(plan, 2).driver(z0, budget=1e9, max_cycles=3)
    assert got.per_level_evals == want.per_level
    np.testing.assert_allclose(got.history, want.history, rtol=1e-8)
    assert rel_l2(got.final_iterate, want.z) <= 1e-8


def test_mgopt_config1_c64_values(oracle):
    """Config-1 geometry in complex64: values track the c128 oracle to 1e-4."""
    from paper_1810_05628_b200 import Hierarchy, synth
    cfg = synth.Config(1, 128, 32, 13, 8, 4.0, 8.0, 0.01, "c64", depth=2)
    p, plan, cfg = _patch(oracle, "c64", cfg)
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    want = oracle.Hierarchy(p, 2).driver(z0, budget=1e9, max_cycles=2)
    got = Hierarchy(plan, 2).driver(z0, budget=1e9, max_cycles=2)
    assert got.history.shape == want.history.shape
    np.testing.assert_allclose(got.history[:, 1], want.history[:, 1], rtol=1e-4)


def test_mgopt_deterministic(oracle):
    from paper_1810_05628_b200 import Hierarchy
    p, plan, cfg = _patch(oracle, "c64")
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    h = Hierarchy(plan, 2)
    a = h.driver(z0, budget=1e9, max_cycles=2)
    b = h.driver(z0, budget=1e9, max_cycles=2)
    assert np.array_equal(a.final_iterate, b.final_iterate)
    assert np.array_equal(a.history, b.history)


def test_depth1_is_lbfgs(oracle):
    """multigrid.cpp:185-189: depth-1 hierarchy == plain LBFGS (bitwise)."""
    from paper_1810_05628_b200 import Hierarchy
    p, plan, cfg = _patch(oracle, "c128")
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    a = Hierarchy(plan, 1).driver(z0, budget=1e9, max_cycles=3)
    b = plan.lbfgs(z0, max_iters=3)
    assert np.array_equal(a.final_iterate, b.final_iterate)
    assert np.array_equal(a.history, b.history)


def test_hierarchy_errors():
    from paper_1810_05628_b200 import ConfigError, Hierarchy, Plan
    n = 16
    plan = Plan(n, n, 8, np.array([[0, 0], [4, 4]], np.int32), np.ones((2, n, n)), None, precision="c128")
    with pytest.raises(ConfigError):
        Hierarchy(plan, 3)   # would coarsen below 8
    with pytest.raises(ConfigError):
        Hierarchy(plan, 0)


def test_lbfgs_budget_and_stall(oracle):
    p, plan, cfg = _patch(oracle, "c128")
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    r = plan.lbfgs(z0, max_iters=50, max_weighted=5.0)
    assert r.reason == "budget" and r.weighted_evals >= 5.0
    w = oracle.lbfgs(p, z0, max_iters=50, max_weighted=5.0)
    assert r.weighted_evals == w.weighted


@pytest.mark.parametrize("precision", ["c64", "c128"])
def test_fused_two_loop_matches_per_op(oracle, monkeypatch, precision):
    """The cooperative two-loop kernel reduces every product over the same
    partition and trees as the kernel-per-op path: identical bits."""
    p, plan, cfg = _patch(oracle, precision)
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    monkeypatch.setenv("PTG_TWO_LOOP", "fused")
    a = plan.lbfgs(z0, max_iters=30, lbfgs_memory=5)
    monkeypatch.setenv("PTG_TWO_LOOP", "ops")
    b = plan.lbfgs(z0, max_iters=30, lbfgs_memory=5)
    assert len(a.history) > 6
    assert np.array_equal(a.final_iterate, b.final_iterate)
    assert np.array_equal(a.history, b.history)


def test_truncated_newton_ref_mode_vs_reference(gold):
    """solvers.cpp:143-227 (Newton-CG, finite-difference Hessian-vector products)."""
    plan, n, w, s = _ref_plan(gold)
    r = plan.truncated_newton(gold["pie_z0"], v=gold["eval_b_v"], max_iters=4, cg_max_iters=5)
    assert r.history.shape == gold["tn_hist"].shape
    np.testing.assert_allclose(r.history[:, 0], gold["tn_hist"][:, 0], rtol=0)   # identical eval counts
    np.testing.assert_allclose(r.history[:, 1:], gold["tn_hist"][:, 1:], rtol=1e-8)
    assert r.weighted_evals == gold["tn_meta"][1]
    assert rel_l2(r.final_iterate, gold["tn_z"]) <= 1e-8


def test_truncated_newton_patch_c128_vs_oracle(oracle):
    p, plan, cfg = _patch(oracle, "c128")
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    want = oracle.truncated_newton(p, z0, max_iters=3, cg_max_iters=6)
    got = plan.truncated_newton(z0, max_iters=3, cg_max_iters=6)
    assert got.weighted_evals == want.weighted
    np.testing.assert_allclose(got.history, want.history, rtol=1e-8)
    assert rel_l2(got.final_iterate, want.z) <= 1e-8


def test_truncated_newton_c64_descends(oracle):
    """complex64: the finite-difference Hessian products are fp32-noisy, so only
    the solver contract is checked (monotone accepted values, accounting)."""
    p, plan, cfg = _patch(oracle, "c64")
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    r = plan.truncated_newton(z0, max_iters=3, cg_max_iters=4)
    vals = r.history[:, 1]
    assert np.all(np.diff(vals) <= 0) and vals[-1] < vals[0]
    assert r.weighted_evals == r.history[-1, 0]


def test_compact_lbfgs_matches_two_loop(oracle, monkeypatch):
    """The compact representation (default) is the same LBFGS matrix as the
    reference's two-loop recursion: c128 trajectories agree to rounding."""
    p, plan, cfg = _patch(oracle, "c128")
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    a = plan.lbfgs(z0, max_iters=25, lbfgs_memory=5)
    monkeypatch.setenv("PTG_TWO_LOOP", "fused")
    b = plan.lbfgs(z0, max_iters=25, lbfgs_memory=5)
    assert a.weighted_evals == b.weighted_evals and a.reason == b.reason
    np.testing.assert_allclose(a.history, b.history, rtol=1e-10)
    assert rel_l2(a.final_iterate, b.final_iterate) <= 1e-10


@pytest.mark.parametrize("precision", ["c64", "c128"])
def test_graph_replayed_lbfgs_matches_eager(oracle, monkeypatch, precision):
    """From the third iteration the compact LBFGS iteration is replayed as a
    CUDA graph (direction with the fused first trial, evaluation, statistics
    and products on a side stream); the trajectory is bitwise the eager one."""
    p, plan, cfg = _patch(oracle, precision)
    z0 = np.ones((cfg.n, cfg.n), np.complex128)
    a = plan.lbfgs(z0, max_iters=30, lbfgs_memory=5)
    monkeypatch.setenv("PTG_LBFGS_GRAPH", "0")
    b = plan.lbfgs(z0, max_iters=30, lbfgs_memory=5)
    assert len(a.history) > 6
    assert a.weighted_evals == b.weighted_evals and a.reason == b.reason
    assert np.array_equal(a.history, b.history)
    assert np.array_equal(a.final_iterate, b.final_iterate)
