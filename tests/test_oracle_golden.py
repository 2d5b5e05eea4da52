"""Pin the CPU oracle (oracle/ptgo.c) to golden vectors produced by the
unmodified reference library (tests/golden/make_golden.py).

In ref mode the restatement keeps the reference's operation order, so every
comparison here is BITWISE (np.array_equal / ==).
"""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


@pytest.mark.parametrize("n", [1, 2, 8, 32])
def test_fft2_bitwise(oracle, gold, n):
    x = gold[f"fft_in_{n}"]
    assert np.array_equal(oracle.fft2(x, False), gold[f"fft_fwd_{n}"])
    assert np.array_equal(oracle.fft2(x, True), gold[f"fft_inv_{n}"])


@pytest.mark.parametrize("tag", ["a", "b"])
@pytest.mark.parametrize("metric", [0, 1])
def test_evaluate_bitwise(oracle, gold, tag, metric):
    n, w, s = (int(v) for v in gold[f"eval_{tag}_geom"])
    p = oracle.Problem(n, n, w, gold[f"eval_{tag}_pos"], gold[f"eval_{tag}_data"], None, metric)
    val, g = oracle.evaluate(p, gold[f"eval_{tag}_z"], gold[f"eval_{tag}_v"])
    assert val == float(gold[f"eval_{tag}_m{metric}_value"])
    assert np.array_equal(g, gold[f"eval_{tag}_m{metric}_grad"])


@pytest.mark.parametrize("tag", ["a", "b"])
def test_project_modulus_bitwise(oracle, gold, tag):
    n, w, s = (int(v) for v in gold[f"eval_{tag}_geom"])
    pos = gold[f"eval_{tag}_pos"]
    p = oracle.Problem(n, n, w, pos, gold[f"eval_{tag}_data"])
    for k in (0, len(pos) // 2, len(pos) - 1):
        got = oracle.project_modulus(p, gold[f"eval_{tag}_z"], k)
        assert np.array_equal(got, gold[f"proj_{tag}_{k}"])


def test_simulate_bitwise(oracle, gold):
    n, w, s = (int(v) for v in gold["eval_b_geom"])
    d = oracle.simulate(n, n, w, gold["eval_b_pos"], gold["eval_b_truth"])
    assert np.array_equal(d, gold["eval_b_data"])


def test_transfers_bitwise(oracle, gold):
    assert np.array_equal(oracle.restrict_field(gold["xfer_fine"]), gold["xfer_restrict"])
    assert np.array_equal(oracle.prolong_field(gold["xfer_restrict"]), gold["xfer_prolong"])
    assert np.array_equal(oracle.restrict_data(gold["xfer_data"]), gold["xfer_restrict_data"])


def _geom(gold):
    n, w, s = (int(v) for v in gold["eval_b_geom"])
    return n, w, s, gold["eval_b_pos"], gold["eval_b_data"]


def test_pie_bitwise(oracle, gold):
    n, w, s, pos, data = _geom(gold)
    r = oracle.pie(oracle.Problem(n, n, w, pos, data), gold["pie_z0"], 0.1, 3)
    assert np.array_equal(r.z, gold["pie_z"])
    assert np.array_equal(r.history, gold["pie_hist"])
    assert [r.value, r.weighted, r.reason] == list(gold["pie_meta"])


def test_lbfgs_bitwise(oracle, gold):
    n, w, s, pos, data = _geom(gold)
    r = oracle.lbfgs(oracle.Problem(n, n, w, pos, data), gold["pie_z0"], v=gold["eval_b_v"], max_iters=6)
    assert np.array_equal(r.z, gold["lbfgs_z"])
    assert np.array_equal(r.history, gold["lbfgs_hist"])
    assert [r.value, r.weighted, r.reason] == list(gold["lbfgs_meta"])


def test_truncated_newton_bitwise(oracle, gold):
    n, w, s, pos, data = _geom(gold)
    r = oracle.truncated_newton(oracle.Problem(n, n, w, pos, data), gold["pie_z0"], v=gold["eval_b_v"],
                                max_iters=4, cg_max_iters=5)
    assert np.array_equal(r.z, gold["tn_z"])
    assert np.array_equal(r.history, gold["tn_hist"])
    assert [r.value, r.weighted, r.reason] == list(gold["tn_meta"])


@pytest.mark.parametrize("depth", [2, 3])
def test_mgopt_bitwise(oracle, gold, depth):
    n, w, s, pos, data = _geom(gold)
    h = oracle.Hierarchy(oracle.Problem(n, n, w, pos, data), depth, coarsest_max_iters=10)
    r = h.driver(gold[f"mg{depth}_z0"], budget=1e9, max_cycles=3)
    assert np.array_equal(r.z, gold[f"mg{depth}_z"])
    assert np.array_equal(r.history, gold[f"mg{depth}_hist"])
    meta = gold[f"mg{depth}_meta"]
    assert [r.value, r.weighted, r.reason] == list(meta[:3])
    assert r.per_level == [int(x) for x in meta[3:]]


MG_DEFAULT = os.path.join(os.path.dirname(__file__), "golden", "mg_default_golden.npz")


@pytest.mark.parametrize("tag", ["a", "b"])
def test_mgopt_default_settings_bitwise(oracle, tag):
    """Depth-3 MG/OPT at the reference's default settings (coarsest solve 100
    LBFGS iterations, multigrid.cpp:123-128) on data with the reference's
    addNoise: golden run by the unmodified reference (make_mg_default_golden.py)."""
    gold = dict(np.load(MG_DEFAULT))
    n, w, s, depth = (int(v) for v in gold[f"{tag}_geom"])
    h = oracle.Hierarchy(oracle.Problem(n, n, w, gold[f"{tag}_pos"], gold[f"{tag}_data"]), depth)
    assert h.coarsest_iters() == 100
    r = h.driver(gold[f"{tag}_z0"], budget=1e9, max_cycles=3)
    meta = gold[f"{tag}_meta"]
    assert np.array_equal(r.z, gold[f"{tag}_z"])
    assert np.array_equal(r.history, gold[f"{tag}_hist"])
    assert [r.value, r.weighted, r.reason] == list(meta[:3])
    assert r.per_level == [int(x) for x in meta[3:]]
