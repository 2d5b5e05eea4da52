"""Patch-model oracle properties (no reference test pins the complex-probe /
M x M-frame generalisation, so it is validated by invariants):

* reduction to ref mode: probe == 1 with M == n equals the binary-window
  full-field model (shift theorem) to ~1e-15;
* finite differences of the value confirm the gradient (acceptance 1 style);
* additivity over scan positions; zero misfit at the truth (noiseless);
* PIE with binary probes and gamma = 0 is a unit descent step
  (solvers.hpp:108-110, test_solvers.cpp:249-298);
* restrict(prolong(u)) == u bitwise and <prolong u, w> = 4 <u, restrict w>.
"""
import numpy as np
import pytest

from conftest import rand_field, rel, rel_l2


def _patch(oracle, n=32, M=8, steps=7, step=4, seed=1, metric=0):
    from paper_1810_05628_b200 import synth
    cfg = synth.Config(0, n, M, steps, step, 2.0, 3.0, 0.03, "c128")
    obj, probe, pos = synth.make_inputs(cfg)
    data = oracle.simulate(n, M, M, pos, obj, probe)
    return oracle.Problem(n, M, M, pos, data, probe, metric), obj


def test_unit_probe_full_frame_equals_ref_mode(oracle):
    n, w, s = 32, 16, 8
    from paper_1810_05628_b200 import synth
    pos = synth.raster(n, w, (n - w) // s + 1, s)
    zt, z = rand_field(n, 1), rand_field(n, 2)
    data = oracle.simulate(n, n, w, pos, zt)
    ref = oracle.evaluate(oracle.Problem(n, n, w, pos, data), z)
    ones = np.ones((n, n), np.complex128)
    ones[w:, :] = 0
    ones[:, w:] = 0
    pat = oracle.evaluate(oracle.Problem(n, n, w, pos, data, ones), z)
    assert rel(pat[0], ref[0]) < 1e-14
    assert rel_l2(pat[1], ref[1]) < 1e-13


@pytest.mark.parametrize("metric", [0, 1])
def test_finite_differences(oracle, metric):
    p, obj = _patch(oracle, metric=metric)
    z = obj + 0.2 * rand_field(p.n, 3)
    val, g = oracle.evaluate(p, z)
    for s in range(4):
        d = rand_field(p.n, 40 + s)
        d /= np.linalg.norm(d)
        h = 1e-6
        fp = oracle.evaluate(p, z + h * d)[0]
        fm = oracle.evaluate(p, z - h * d)[0]
        fd = (fp - fm) / (2 * h)
        an = np.sum(g.real * d.real + g.imag * d.imag)
        assert abs(fd - an) <= 1e-6 * max(1.0, abs(an))


def test_additivity(oracle):
    p, obj = _patch(oracle)
    z = obj + 0.1 * rand_field(p.n, 4)
    whole = oracle.evaluate(p, z)
    tot, gs = 0.0, np.zeros_like(z)
    for k in range(p.N):
        pk = oracle.Problem(p.n, p.M, p.w, p.pos[k:k + 1], p.data[k:k + 1], p.probe)
        v, g = oracle.evaluate(pk, z)
        tot += v
        gs += g
    assert rel(tot, whole[0]) < 1e-12
    assert rel_l2(gs, whole[1]) < 1e-12


def test_zero_at_truth(oracle):
    p, obj = _patch(oracle)
    val, g = oracle.evaluate(p, obj)
    assert 0 <= val < 1e-20
    assert np.linalg.norm(g) < 1e-9


def test_pie_is_unit_descent_step(oracle):
    n, w, s = 16, 8, 4
    from paper_1810_05628_b200 import synth
    pos = synth.raster(n, w, 3, s)
    data = oracle.simulate(n, n, w, pos, rand_field(n, 5))
    z = rand_field(n, 6)
    one = oracle.Problem(n, n, w, pos[:1], data[:1])
    r = oracle.pie(one, z, 0.0, 1)
    _, g = oracle.evaluate(one, z)
    assert np.max(np.abs(r.z - (z - g))) <= 1e-12


def test_transfer_identities(oracle):
    u = rand_field(16, 7)
    wv = rand_field(32, 8)
    assert np.array_equal(oracle.restrict_field(oracle.prolong_field(u)), u)
    lhs = np.sum((oracle.prolong_field(u).conj() * wv).real)
    rhs = 4 * np.sum((u.conj() * oracle.restrict_field(wv)).real)
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_patch_hierarchy_levels(oracle):
    p, obj = _patch(oracle, n=64, M=16, steps=7, step=8)
    h = oracle.Hierarchy(p, 3)
    shapes = [(h.level(l).n, h.level(l).M, h.level(l).w) for l in range(3)]
    assert shapes == [(64, 16, 16), (32, 8, 8), (16, 4, 4)]
    assert h.coarsest_iters() == 100
    assert np.array_equal(h.level(1).pos, p.pos // 2)
    r = h.driver(np.ones((64, 64), np.complex128), budget=1e9, max_cycles=2)
    assert r.history[-1, 1] < r.history[0, 1]
