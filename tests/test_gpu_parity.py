"""GPU parity: libptg (through the C-ABI) vs the CPU oracle / compiled reference.

Tolerances (BASELINE.json north_star): complex64 objective 1e-5 relative and
gradient 1e-4 relative L2; complex128 1e-10.  Integer/index work (transfers)
is bit-exact.
"""
import numpy as np
import pytest

from conftest import rand_field, rel, rel_l2

pytestmark = pytest.mark.gpu

C64_VAL, C64_GRAD = 1e-5, 1e-4
C128_TOL = 1e-10


def _round64(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def _patch_case(oracle, cfg, precision, metric=0, with_shift=True, seed=5):
    from paper_1810_05628_b200 import Plan, synth
    obj, probe, pos = synth.make_inputs(cfg)
    z = obj * 0.9 + 0.05 * rand_field(cfg.n, seed)   # an iterate near the truth
    v = 0.01 * rand_field(cfg.n, seed + 1) if with_shift else None
    data = oracle.simulate(cfg.n, cfg.M, cfg.w, pos, obj, probe)
    if precision == "c64":
        z, probe = _round64(z), _round64(probe)
        v = _round64(v) if v is not None else None
        data = data.astype(np.float32)
    p = oracle.Problem(cfg.n, cfg.M, cfg.w, pos, data.astype(np.float64), probe, metric)
    want_v, want_g = oracle.evaluate(p, z, v)
    plan = Plan(cfg.n, cfg.M, cfg.w, pos, data, probe, precision=precision)
    got_v, got_g = plan.evaluate(z, v, metric=metric)
    return got_v, got_g, want_v, want_g, plan, (z, v)


@pytest.mark.parametrize("cid", [1, 2])
def test_config_eval_c64(oracle, cid):
    from paper_1810_05628_b200 import synth
    cfg = synth.CONFIGS[cid]
    gv, gg, wv, wg, _, _ = _patch_case(oracle, cfg, "c64")
    assert rel(gv, wv) <= C64_VAL, (gv, wv)
    assert rel_l2(gg, wg) <= C64_GRAD


def test_config1_eval_c128(oracle):
    from paper_1810_05628_b200 import synth
    gv, gg, wv, wg, _, _ = _patch_case(oracle, synth.CONFIGS[1], "c128")
    assert rel(gv, wv) <= C128_TOL
    assert rel_l2(gg, wg) <= C128_TOL


@pytest.mark.parametrize("precision,tv,tg", [("c64", C64_VAL, C64_GRAD), ("c128", C128_TOL, C128_TOL)])
@pytest.mark.parametrize("M", [1, 2, 4, 8, 16, 32, 64])
def test_frame_sizes(oracle, precision, tv, tg, M):
    from paper_1810_05628_b200 import synth
    n = max(2 * M, 8)
    steps = 3 if M > 1 else 2
    step = max(1, M // 2) if M > 1 else 1
    n = max(n, (steps - 1) * step + M)
    cfg = synth.Config(0, n, M, steps, step, 2.0, max(M / 4, 1.0), 0.01, precision)
    gv, gg, wv, wg, _, _ = _patch_case(oracle, cfg, precision)
    assert rel(gv, wv, floor=1e-12) <= tv
    assert rel_l2(gg, wg) <= tg


@pytest.mark.parametrize("M", [16, 32, 64])
def test_odd_positions_c64(oracle, M):
    """Jittered scans put windows at odd columns/rows (TMA box starts that are
    not 16-B aligned)."""
    from paper_1810_05628_b200 import synth
    cfg = synth.Config(0, 4 * M + 6, M, 5, M // 2 + 1, 3.0, M / 4, 0.01, "c64", jitter=2)
    gv, gg, wv, wg, _, _ = _patch_case(oracle, cfg, "c64")
    assert rel(gv, wv) <= C64_VAL
    assert rel_l2(gg, wg) <= C64_GRAD


def test_frame_128_c64(oracle):
    from paper_1810_05628_b200 import synth
    cfg = synth.Config(0, 256, 128, 3, 64, 6.0, 32.0, 0.0, "c64", jitter=2)
    gv, gg, wv, wg, _, _ = _patch_case(oracle, cfg, "c64")
    assert rel(gv, wv) <= C64_VAL
    assert rel_l2(gg, wg) <= C64_GRAD


@pytest.mark.parametrize("precision", ["c64", "c128"])
def test_intensity_metric(oracle, precision):
    from paper_1810_05628_b200 import synth
    cfg = synth.small_config(precision=precision)
    gv, gg, wv, wg, _, _ = _patch_case(oracle, cfg, precision, metric=1)
    tol = C128_TOL if precision == "c128" else C64_GRAD
    assert rel(gv, wv) <= tol
    assert rel_l2(gg, wg) <= tol


def test_ref_mode_against_reference(reference):
    """Binary window, M == n: the reference library itself is the oracle."""
    from paper_1810_05628_b200 import Plan
    n, w, s = 32, 16, 8
    win = reference.ref_raster(n, w, s)
    pos = win[:, :2]
    zt = rand_field(n, 11)
    z = rand_field(n, 12)
    v = rand_field(n, 13)
    data = reference.ref_simulate(n, w, pos, zt)
    plan = Plan(n, n, w, pos, data, None, precision="c128")
    for metric in (0, 1):
        wv, wg = reference.ref_evaluate(metric, n, w, pos, data, z, v)
        gv, gg = plan.evaluate(z, v, metric=metric)
        assert rel(gv, wv) <= C128_TOL
        assert rel_l2(gg, wg) <= C128_TOL
    # projectModulus returns object coordinates in ref mode
    for k in (0, 4, 8):
        want = reference.ref_project_modulus(n, win[k], data[k], z)
        got = plan.project_modulus(z, k)
        assert rel_l2(got, want) <= C128_TOL


def test_simulate_matches_oracle(oracle):
    from paper_1810_05628_b200 import Plan, synth
    for precision, tol in (("c128", 1e-12), ("c64", 2e-6)):
        cfg = synth.small_config(precision=precision)
        obj, probe, pos = synth.make_inputs(cfg)
        want = oracle.simulate(cfg.n, cfg.M, cfg.w, pos, obj, probe)
        plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision=precision)
        got = plan.simulate(obj)
        assert rel_l2(got, want) <= tol


def test_project_modulus_patch(oracle):
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.small_config(precision="c128")
    obj, probe, pos = synth.make_inputs(cfg)
    data = oracle.simulate(cfg.n, cfg.M, cfg.w, pos, obj, probe)
    z = rand_field(cfg.n, 3)
    p = oracle.Problem(cfg.n, cfg.M, cfg.w, pos, data, probe)
    plan = Plan(cfg.n, cfg.M, cfg.w, pos, data, probe, precision="c128")
    for k in (0, 10, cfg.N - 1):
        assert rel_l2(plan.project_modulus(z, k), oracle.project_modulus(p, z, k)) <= C128_TOL


def test_fixed_point_at_truth():
    """test_objectives.cpp:207-217: Phi ~ 0 and grad ~ 0 at the true object."""
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.small_config(precision="c128")
    obj, probe, pos = synth.make_inputs(cfg)
    plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision="c128")
    plan.simulate(obj, copy_out=False)
    val, g = plan.evaluate(obj)
    assert 0.0 <= val <= 1e-20
    assert np.linalg.norm(g) <= 1e-9


def test_determinism_bitwise(oracle):
    from paper_1810_05628_b200 import synth
    gv, gg, _, _, plan, (z, v) = _patch_case(oracle, synth.CONFIGS[2], "c64")
    for _ in range(3):
        v2, g2 = plan.evaluate(z, v)
        assert v2 == gv
        assert np.array_equal(g2, gg)


def test_empty_scan(oracle):
    from paper_1810_05628_b200 import Plan
    n = 16
    z, v = rand_field(n, 1), rand_field(n, 2)
    plan = Plan(n, 8, 8, np.zeros((0, 2), np.int32), np.zeros((0, 8, 8)), None, precision="c128")
    val, g = plan.evaluate(z, v)
    assert val == pytest.approx(-np.sum(v.real * z.real + v.imag * z.imag), rel=1e-14)
    assert np.array_equal(g, -v)


def test_single_pixel_analytic():
    """test_objectives.cpp:185-205: 1x1 analytic values."""
    from paper_1810_05628_b200 import Plan
    z = np.array([[1.0 + 0j]])
    pos = np.zeros((1, 2), np.int32)
    plan = Plan(1, 1, 1, pos, np.array([[[4.0]]]), None, precision="c128")
    val, g = plan.evaluate(z)
    assert val == pytest.approx(0.5, rel=1e-15)
    assert g[0, 0].real == pytest.approx(-1.0, rel=1e-15)
    plan0 = Plan(1, 1, 1, pos, np.array([[[0.0]]]), None, precision="c128")
    val, g = plan0.evaluate(z, metric=1)
    assert val == pytest.approx(0.5, rel=1e-15)
    assert g[0, 0].real == pytest.approx(2.0, rel=1e-15)


def test_validation_errors():
    from paper_1810_05628_b200 import DomainError, GeometryError, Plan
    pos = np.array([[0, 0]], np.int32)
    d = np.ones((1, 8, 8))
    d[0, 3, 3] = -1e-9
    with pytest.raises(DomainError):
        Plan(8, 8, 4, pos, d, None, precision="c128")
    with pytest.raises(GeometryError):
        Plan(8, 8, 4, np.array([[6, 0]], np.int32), np.ones((1, 8, 8)), None)
    with pytest.raises(GeometryError):
        Plan(12, 12, 4, pos, np.ones((1, 12, 12)), None)
    plan = Plan(8, 8, 4, pos, np.ones((1, 8, 8)), None, precision="c128")
    with pytest.raises(DomainError):
        plan.set_data(d)


def test_transfers_bitexact(oracle):
    from paper_1810_05628_b200 import prolong_field, restrict_data, restrict_field
    f = rand_field(64, 7)
    assert np.array_equal(restrict_field(f), oracle.restrict_field(f))
    c = rand_field(32, 8)
    assert np.array_equal(prolong_field(c), oracle.prolong_field(c))
    assert np.array_equal(restrict_field(prolong_field(c)), c)   # multigrid.hpp:11-13
    d = np.abs(np.random.default_rng(9).normal(size=(5, 32, 32)))
    assert np.array_equal(restrict_data(d), oracle.restrict_data(d))


def test_ptyf_streamed_upload(tmp_path, oracle):
    """loadRawStack (image_io.cpp:184-196) streamed into the plan == in-memory upload;
    the reference's error classes for bad files."""
    from paper_1810_05628_b200 import GeometryError, IoError, Plan, synth, write_ptyf
    cfg = synth.small_config(precision="c64")
    obj, probe, pos = synth.make_inputs(cfg)
    data = oracle.simulate(cfg.n, cfg.M, cfg.w, pos, obj, probe)
    path = tmp_path / "stack.ptyf"
    write_ptyf(path, data)
    a = Plan(cfg.n, cfg.M, cfg.w, pos, data, probe, precision="c64")
    b = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision="c64")
    b.load_ptyf(path)
    z = rand_field(cfg.n, seed=5)
    va, ga = a.evaluate(z)
    vb, gb = b.evaluate(z)
    assert va == vb and np.array_equal(ga, gb)
    bad = tmp_path / "bad.ptyf"
    bad.write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(IoError):
        b.load_ptyf(bad)
    with pytest.raises(IoError):
        b.load_ptyf(tmp_path / "missing.ptyf")
    trunc = tmp_path / "trunc.ptyf"
    trunc.write_bytes(path.read_bytes()[:-8])
    with pytest.raises(IoError):
        b.load_ptyf(trunc)
    other = tmp_path / "other.ptyf"
    write_ptyf(other, data[:-1])
    with pytest.raises(GeometryError):
        b.load_ptyf(other)
    b.load_ptyf(path)   # the plan stays usable after failed loads
    vc, gc = b.evaluate(z)
    assert vc == va


@pytest.mark.parametrize("cfg_id,with_shift", [(2, False), (2, True), (3, False)])
def test_banded_host_eval_equals_device_eval(cfg_id, with_shift):
    """ptg_eval overlaps the PCIe copies with the computation in row bands; the
    gradient and value are bitwise those of the device-resident evaluation."""
    import torch
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.CONFIGS[cfg_id]
    obj, probe, pos = synth.make_inputs(cfg)
    plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision="c64")
    plan.simulate(obj, copy_out=False)
    z = obj * 0.9 + 0.05 * rand_field(cfg.n, 11)
    v = 0.01 * rand_field(cfg.n, 12) if with_shift else None
    val_h, g_h = plan.evaluate(z, v)
    zt = torch.from_numpy(z.astype(np.complex64)).cuda()
    vt = torch.from_numpy(v.astype(np.complex64)).cuda() if v is not None else None
    gt = torch.empty_like(zt)
    val_d = plan.evaluate_device(zt, gt, v=vt)
    assert val_h == val_d
    assert np.array_equal(g_h, gt.cpu().numpy().astype(np.complex128))


@pytest.mark.parametrize("with_shift", [False, True])
def test_graph_replayed_host_eval(with_shift):
    """With pinned host buffers ptg_eval replays the banded sequence as one CUDA
    graph (first call eager, second captured, later calls replayed).  Every call
    sees the current contents of z / v and equals the device evaluation bitwise;
    new buffers (another key) fall back to eager and are captured again."""
    import torch
    from paper_1810_05628_b200 import Plan, synth
    cfg = synth.CONFIGS[2]
    obj, probe, pos = synth.make_inputs(cfg)
    plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision="c64")
    plan.simulate(obj, copy_out=False)
    n = cfg.n
    zp = torch.empty(n, n, dtype=torch.complex128).pin_memory()
    gp = torch.empty(n, n, dtype=torch.complex128).pin_memory()
    vp = torch.empty(n, n, dtype=torch.complex128).pin_memory() if with_shift else None
    for call in range(5):
        if call == 3:   # new pointers: eager again, then re-captured
            zp = torch.empty(n, n, dtype=torch.complex128).pin_memory()
            gp = torch.empty(n, n, dtype=torch.complex128).pin_memory()
        z = (obj * (0.9 - 0.05 * call) + 0.05 * rand_field(n, 20 + call)).astype(np.complex64).astype(np.complex128)
        zp.numpy()[:] = z
        v = None
        if with_shift:
            v = (0.01 * rand_field(n, 40 + call)).astype(np.complex64).astype(np.complex128)
            vp.numpy()[:] = v
        gp.numpy()[:] = np.nan
        val_h, _ = plan.evaluate(zp.numpy(), None if vp is None else vp.numpy(), out=gp.numpy())
        zt = torch.from_numpy(z.astype(np.complex64)).cuda()
        vt = torch.from_numpy(v.astype(np.complex64)).cuda() if v is not None else None
        gt = torch.empty_like(zt)
        val_d = plan.evaluate_device(zt, gt, v=vt)
        assert val_h == val_d, call
        assert np.array_equal(gp.numpy(), gt.cpu().numpy().astype(np.complex128)), call


@pytest.mark.parametrize("precision", ["c64", "c128"])
def test_halo_exchange_kernels(precision):
    """csrc/halo.cu (band exchange): pack every simulated rank's band, concatenate
    the buffers as the all-gather would, unpack on each rank: neighbours' rows
    added to the own rows (bitwise own + received), misfits summed in rank order."""
    import torch
    from paper_1810_05628_b200 import _lib, sharding
    lib = _lib.lib()
    world, n, ov = 3, 64, 16
    cdt = torch.complex64 if precision == "c64" else torch.complex128
    prec = 0 if precision == "c64" else 1
    nb = int(lib.ptg_halo_bytes(prec, n, ov))
    assert nb == sharding.halo_bytes(n, ov, 8 if precision == "c64" else 16)
    rng = np.random.default_rng(5)
    grads = [torch.from_numpy((rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))).astype(
        np.complex64 if precision == "c64" else np.complex128)).cuda() for _ in range(world)]
    vals = [torch.tensor([float(r) + 0.25, 0.0], dtype=torch.float64, device="cuda") for r in range(world)]
    bufs = []
    for r in range(world):
        b = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        assert lib.ptg_halo_pack(prec, grads[r].data_ptr(), n, ov, vals[r].data_ptr(), b.data_ptr(), None) == 0
        bufs.append(b)
    allb = torch.cat(bufs)
    torch.cuda.synchronize()
    for r in range(world):
        g = grads[r].clone()
        v = vals[r].clone()
        assert lib.ptg_halo_unpack(prec, g.data_ptr(), n, ov, allb.data_ptr(), r, world, v.data_ptr(), None) == 0
        torch.cuda.synchronize()
        want = grads[r].cpu().numpy().copy()
        if r > 0:
            want[:ov] = want[:ov] + grads[r - 1].cpu().numpy()[n - ov:]
        if r + 1 < world:
            want[n - ov:] = want[n - ov:] + grads[r + 1].cpu().numpy()[:ov]
        assert np.array_equal(g.cpu().numpy(), want)
        assert float(v[0].cpu()) == sum(float(k) + 0.25 for k in range(world))


def test_transfer_device_kernels_c64_f32():
    """The float4-vectorised complex64 / float32 transfer kernels (transfer.cu)
    against the reference's arithmetic in the same precision and order
    (multigrid.cpp:34-77): bit-exact."""
    import torch
    from paper_1810_05628_b200 import _lib
    lib = _lib.lib()
    rng = np.random.default_rng(9)
    n = 96
    f = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))).astype(np.complex64)
    ft = torch.from_numpy(f).cuda()
    ct = torch.empty(n // 2, n // 2, dtype=torch.complex64, device="cuda")
    assert lib.ptg_restrict_field_device(0, ft.data_ptr(), n, ct.data_ptr(), None) == 0
    a, b, c, d = f[0::2, 0::2], f[0::2, 1::2], f[1::2, 0::2], f[1::2, 1::2]
    want = ((a + b) + (c + d)) * np.float32(0.25)
    torch.cuda.synchronize()
    assert np.array_equal(ct.cpu().numpy(), want)
    pt = torch.empty(n, n, dtype=torch.complex64, device="cuda")
    assert lib.ptg_prolong_field_device(0, ct.data_ptr(), n // 2, pt.data_ptr(), None) == 0
    torch.cuda.synchronize()
    assert np.array_equal(pt.cpu().numpy(), np.repeat(np.repeat(want, 2, 0), 2, 1))
    for M in (16, 32, 64):   # float4 path (M % 16 == 0)
        N = 5
        dd = rng.random((N, M, M)).astype(np.float32)
        dt = torch.from_numpy(dd).cuda()
        ot = torch.empty(N, M // 2, M // 2, dtype=torch.float32, device="cuda")
        assert lib.ptg_restrict_data_device(0, dt.data_ptr(), N, M, ot.data_ptr(), None) == 0
        MH = M // 2
        idx = (((np.arange(MH) + MH // 2) % MH) + 3 * M // 4) % M
        want_d = dd[:, idx][:, :, idx] * np.float32(1.0 / 16.0)
        torch.cuda.synchronize()
        assert np.array_equal(ot.cpu().numpy(), want_d), M
