"""The C-ABI library loads without a GPU and exports every symbol the header
declares; without a device every call fails loudly (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ptg.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ptg_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    from paper_1810_05628_b200 import _lib
    L = _lib.lib()   # loads (no GPU needed)
    names = _declared()
    assert len(names) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(ptg_[a-z0-9_]+)\b", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(_lib.EXPORTS) == set(names)
    for n in names:
        getattr(L, n)


def test_built_for_sm100a():
    from paper_1810_05628_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1810_05628_b200 import CudaError, Plan
    with pytest.raises(CudaError):
        Plan(8, 8, 4, np.zeros((1, 2), np.int32), np.ones((1, 8, 8)))


def test_defaults_match_reference():
    """SolverConfig / MgoptConfig / MgoptDriverConfig defaults (solvers.hpp:56-66,
    multigrid.hpp:39-49, 82-87)."""
    import ctypes as C

    from paper_1810_05628_b200 import _lib
    L = _lib.lib()
    s = _lib.SolverCfg()
    L.ptg_solver_cfg_default(C.byref(s))
    assert (s.max_iters, s.grad_tol_rel, s.grad_tol_abs, s.lbfgs_memory, s.linesearch_max) == (100, 0.0, 1e-13, 25, 50)
    assert s.max_weighted == float("inf")
    m = _lib.MgCfg()
    L.ptg_mg_cfg_default(C.byref(m))
    assert (m.k1, m.k2, m.coarsest_max_iters, m.coarsest_grad_tol_rel, m.intermediate_grad_tol_rel) == (1, 1, 0, 1e-4, 1e-3)
    d = _lib.DriverCfg()
    L.ptg_driver_cfg_default(C.byref(d))
    assert (d.budget, d.grad_tol_rel, d.grad_tol_abs, d.max_cycles) == (100.0, 0.0, 1e-13, 1000000)


def test_synthetic_configs_geometry():
    from paper_1810_05628_b200 import synth
    for cid, cfg in synth.CONFIGS.items():
        pos = synth.raster(cfg.n, cfg.w, cfg.steps, cfg.step, cfg.jitter)
        assert pos.shape == (cfg.N, 2)
        assert pos.min() >= 0 and pos.max() <= cfg.n - cfg.w
    assert synth.CONFIGS[2].N == 841 and synth.CONFIGS[5].N == 27556
