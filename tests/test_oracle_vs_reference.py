"""Live pinning: oracle vs the compiled reference library on fresh seeded
ref-mode problems (skipped where the reference was not built).  Bitwise."""
import numpy as np
import pytest

from conftest import rand_field


@pytest.mark.parametrize("n,w,s", [(8, 4, 2), (16, 8, 4), (32, 16, 8), (64, 32, 16)])
@pytest.mark.parametrize("metric", [0, 1])
def test_evaluate_matches_reference(reference, n, w, s, metric):
    pos = reference.ref_raster(n, w, s)[:, :2].copy()
    data = reference.ref_simulate(n, w, pos, rand_field(n, 3 * n))
    z, v = rand_field(n, 5 * n), rand_field(n, 7 * n, 0.1)
    want = reference.ref_evaluate(metric, n, w, pos, data, z, v)
    got = reference.evaluate(reference.Problem(n, n, w, pos, data, None, metric), z, v)
    assert got[0] == want[0]
    assert np.array_equal(got[1], want[1])


def test_pattern_parallel_is_bitwise_serial(reference):
    """The OpenMP pattern-parallel oracle (CPU baseline) equals the serial loop."""
    n, w, s = 64, 32, 8
    pos = reference.ref_raster(n, w, s)[:, :2].copy()
    data = reference.ref_simulate(n, w, pos, rand_field(n, 1))
    z = rand_field(n, 2)
    p = reference.Problem(n, n, w, pos, data)
    reference.set_threads(1)
    a = reference.evaluate(p, z)
    reference.set_threads(4)
    b = reference.evaluate(p, z)
    reference.use_reference_fft(True)
    c = reference.evaluate(p, z)
    reference.use_reference_fft(False)
    reference.set_threads(1)
    assert a[0] == b[0] == c[0]
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[1], c[1])


def test_errors_match_reference(reference):
    n = 8
    pos = np.array([[0, 0]], np.int32)
    d = np.ones((1, n, n))
    d[0, 1, 1] = -1.0
    with pytest.raises(reference.OracleError) as e1:
        reference.ref_evaluate(0, n, 4, pos, d, rand_field(n, 1))
    with pytest.raises(reference.OracleError) as e2:
        reference.evaluate(reference.Problem(n, n, 4, pos, d), rand_field(n, 1))
    assert e1.value.code == e2.value.code == 12   # DomainError
    with pytest.raises(reference.OracleError) as e3:
        reference.ref_raster(16, 8, 3)
    assert e3.value.code == 11                     # GeometryError
    with pytest.raises(reference.OracleError) as e4:
        reference.fft2(np.zeros((6, 6)))
    assert e4.value.code == 11


@pytest.mark.parametrize("depth,cycles", [(2, 4), (3, 2)])
def test_mgopt_matches_reference(reference, depth, cycles):
    n, w, s = 64, 32, 16
    pos = reference.ref_raster(n, w, s)[:, :2].copy()
    data = reference.ref_simulate(n, w, pos, rand_field(n, 9) + 1.5)
    z0 = np.ones((n, n), np.complex128)
    a = reference.ref_mgopt(0, n, w, s, data, z0, depth, budget=1e9, max_cycles=cycles)
    b = reference.Hierarchy(reference.Problem(n, n, w, pos, data), depth).driver(z0, budget=1e9,
                                                                                  max_cycles=cycles)
    assert np.array_equal(a.z, b.z)
    assert np.array_equal(a.history, b.history)
    assert a.per_level == b.per_level
