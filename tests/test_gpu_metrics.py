"""Device diagnostics (metrics.cpp:67-136) vs golden values produced by the
unmodified reference (tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


@pytest.mark.parametrize("tag,z,zt", [("a", "tn_z", "eval_b_truth"), ("b", "met_za", "met_zb")])
def test_metrics_vs_reference(gold, tag, z, zt):
    from paper_1810_05628_b200 import metrics
    m = metrics(gold[z], gold[zt])
    want = gold[f"met_{tag}"]
    assert m["relative_error"] == pytest.approx(want[0], rel=1e-13)
    assert m["magnitude_rel_error"] == pytest.approx(want[1], rel=1e-13)
    assert m["phase_ssim"] == pytest.approx(want[2], rel=1e-12)


@pytest.mark.parametrize("tag,z", [("a", "tn_z"), ("b", "met_za")])
def test_canonical_phase_vs_reference(gold, tag, z):
    from paper_1810_05628_b200 import canonical_phase
    got = canonical_phase(gold[z])
    np.testing.assert_allclose(got, gold[f"met_phase_{tag}"], rtol=0, atol=1e-14)


def test_metric_identities_and_errors(gold):
    from paper_1810_05628_b200 import DomainError, MetricError, metrics, phase_ssim, relative_error
    z = gold["met_za"]
    m = metrics(z, z)
    assert m["phase_ssim"] == 1.0 and m["relative_error"] == 0.0 and m["magnitude_rel_error"] == 0.0
    with pytest.raises(DomainError):
        relative_error(z, np.zeros_like(z))
    with pytest.raises(MetricError):
        phase_ssim(z[:10, :10], z[:10, :10])
    with pytest.raises(DomainError):
        relative_error(z, z[:20, :20])


def test_metrics_device_complex64(gold):
    import torch
    from paper_1810_05628_b200 import metrics, metrics_device
    z = gold["met_za"].astype(np.complex64)
    zt = gold["met_zb"].astype(np.complex64)
    got = metrics_device(torch.from_numpy(z).cuda(), torch.from_numpy(zt).cuda())
    want = metrics(z.astype(np.complex128), zt.astype(np.complex128))   # fp64 on the widened values
    for k in want:
        assert got[k] == pytest.approx(want[k], rel=1e-14)
