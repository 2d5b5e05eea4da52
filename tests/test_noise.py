"""Noise: addNoise (forward.cpp:56-86) and the Poisson
photon sampler, oracle pinned against the reference and numpy, GPU against
the oracle / the reference's golden output."""
import os

import numpy as np
import pytest

from conftest import rel_l2

GOLD = os.path.join(os.path.dirname(__file__), "golden", "noise_golden.npz")


# ---------------------------------------------------------------- CPU (oracle)
def test_oracle_philox_matches_numpy(oracle):
    # numpy bumps the 256-bit counter (with carry) before each block: start it one below
    for ctr, key in [((1, 0, 0, 0), (0, 0)), ((11, 2, 3, 4), (5, 7)), ((2**64 - 1, 9, 1, 0), (2**63, 1))]:
        bg = np.random.Philox(counter=np.array([ctr[0] - 1, *ctr[1:]], np.uint64), key=np.array(key, np.uint64))
        want = bg.random_raw(4).astype(np.uint64)
        got = oracle.philox4x64(ctr, key)
        assert np.array_equal(got, want), (ctr, key)


def test_oracle_add_noise_matches_reference_golden(oracle):
    g = np.load(GOLD)
    for tag in ("a", "b"):
        d, (level, seed) = g[f"noise_{tag}_data"], g[f"noise_{tag}_meta"]
        got = oracle.add_noise(d, level, int(seed), uniforms=g[f"noise_{tag}_uniforms"])
        # same arithmetic in the same order as forward.cpp:56-86
        assert np.array_equal(got, g[f"noise_{tag}_out"]), tag


def test_oracle_add_noise_live_reference(reference):
    rng = np.random.default_rng(5)
    d = rng.uniform(0, 2, (4, 8, 8)) ** 2
    u = reference.ref_uniform_stream(99, 2 * d.size)
    assert np.array_equal(reference.add_noise(d, 0.1, 99, uniforms=u), reference.ref_add_noise(d, 0.1, 99))


def test_oracle_add_noise_philox_properties(oracle):
    rng = np.random.default_rng(6)
    d = rng.uniform(1, 2, (3, 32, 32))
    out = oracle.add_noise(d, 0.02, seed=3)
    # no clamping at these levels: ||eps|| / ||d|| == level per pattern
    for j in range(3):
        assert abs(np.linalg.norm(out[j] - d[j]) / np.linalg.norm(d[j]) - 0.02) < 1e-12
    assert np.array_equal(out, oracle.add_noise(d, 0.02, seed=3))
    assert not np.array_equal(out, oracle.add_noise(d, 0.02, seed=4))
    with pytest.raises(oracle.OracleError):
        oracle.add_noise(d, -1.0)


@pytest.mark.parametrize("lam", [0.3, 4.0, 25.0, 400.0])
def test_oracle_poisson_moments(oracle, lam):
    # one pattern of constant intensity: lambda = photons / pixels per pixel
    m = 64
    d = np.ones((4, m, m))
    photons = lam * m * m
    out = oracle.add_poisson(d, photons, seed=4)
    k = out * photons / (m * m)          # back to counts
    assert np.allclose(k, np.round(k), atol=1e-9) and k.min() >= 0
    mean, var = k.mean(), k.var()
    ns = k.size
    assert abs(mean - lam) < 5 * np.sqrt(lam / ns)
    assert abs(var - lam) < 6 * lam * np.sqrt(2.0 / ns) + 1e-3


# ---------------------------------------------------------------------- GPU
def _plan(d, precision="c128"):
    from paper_1810_05628_b200 import Plan
    N, M = d.shape[0], d.shape[1]
    pos = np.zeros((N, 2), np.int32)
    return Plan(M, M, M, pos, d, None, precision=precision, device=0)


@pytest.mark.gpu
def test_gpu_philox_matches_numpy():
    import ctypes as C

    from paper_1810_05628_b200 import _lib
    L = _lib.lib()
    ctr = np.array([5, 2, 3, 4], np.uint64)
    key = np.array([123456789, 987654321], np.uint64)
    out = np.zeros(4 * 1000, np.uint64)
    _lib.check(L.ptg_philox4x64(0, ctr.ctypes.data, key.ctypes.data, C.c_size_t(1000), out.ctypes.data))
    bg = np.random.Philox(counter=np.array([4, 2, 3, 4], np.uint64), key=np.array([123456789, 987654321], np.uint64))
    assert np.array_equal(out, bg.random_raw(4000).astype(np.uint64))


@pytest.mark.gpu
def test_gpu_add_noise_reference_uniforms_matches_reference():
    g = np.load(GOLD)
    for tag in ("a", "b"):
        d, (level, seed) = g[f"noise_{tag}_data"], g[f"noise_{tag}_meta"]
        p = _plan(d)
        p.add_noise(level, int(seed), uniforms=g[f"noise_{tag}_uniforms"])
        got = p.data_host()
        # fixed-tree fp64 norms and the device's log / cos vs the reference's
        # serial sums and libm: rounding-level differences only
        assert rel_l2(got, g[f"noise_{tag}_out"]) < 1e-13, tag
        p.close()


@pytest.mark.gpu
def test_gpu_add_noise_philox_matches_oracle(oracle):
    rng = np.random.default_rng(8)
    d = rng.uniform(0, 3, (5, 64, 64)) ** 2
    p = _plan(d)
    p.add_noise(0.25, seed=21)
    got = p.data_host()
    want = oracle.add_noise(d, 0.25, seed=21)
    assert rel_l2(got, want) < 1e-13
    # amplitudes rebuilt from the noisy data
    assert np.allclose(p.data_host(metric=0), np.sqrt(got), rtol=1e-15, atol=0)
    p.close()


@pytest.mark.gpu
def test_gpu_add_poisson_matches_oracle(oracle):
    rng = np.random.default_rng(9)
    M = 64
    d = (rng.uniform(0, 1, (6, M, M)) ** 4) * 1e3
    d[0, 0, 0] = 5e4                       # a bright DC-like pixel (PTRS branch)
    for precision, photons in (("c128", 1e6), ("c128", 1e4)):
        p = _plan(d, precision)
        p.add_poisson(photons, seed=4)
        got = p.data_host()
        want = oracle.add_poisson(d, photons, seed=4)
        # integer counts: identical except where a libm ulp flips an accept
        # test or an inversion comparison (not seen in practice; bounded here)
        same = np.isclose(got, want, rtol=1e-12, atol=0)
        assert same.mean() > 0.9999, same.mean()
        p.close()
    # complex64 plans: the same counts, rounded to float32
    p = _plan(d, "c64")
    p.add_poisson(1e6, seed=4)
    want = oracle.add_poisson(d.astype(np.float32).astype(np.float64), 1e6, seed=4)
    assert np.isclose(p.data_host(), want.astype(np.float32), rtol=1e-6, atol=0).mean() > 0.9999
    p.close()
