"""Host-side mirror of the reference's public API over the libptg C-ABI.

Names follow /root/reference/proj/include/ptycho/*.hpp:

* ``Plan``               ScanGeometry + DiffractionStack + Objective bound to a
                         B200 (field.hpp:75-85, forward.hpp:22-27, objectives.hpp:18-26)
* ``Plan.evaluate``      evaluate / phiDistance / phiIntensityGaussian (objectives.hpp:38-44)
* ``Plan.project_modulus`` projectModulus (objectives.hpp:32-33)
* ``Plan.simulate``      simulate (forward.hpp:43)
* ``Plan.pie``           pie (solvers.hpp:111-114)
* ``Plan.lbfgs``         lbfgs (solvers.hpp:92-95), GPU-resident
* ``Hierarchy``          buildHierarchy / mgoptDriver / mgoptCycle (multigrid.hpp:61-95)
* ``restrict_field`` / ``prolong_field`` / ``restrict_data`` (multigrid.hpp:15-23)

Host arrays are numpy complex128 / float64 like the reference's value types;
``*_device`` methods take torch CUDA tensors (complex64/complex128) and keep
everything resident.  Every call goes to the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L
from ._lib import (ConfigError, CudaError, DomainError, Error, GeometryError, IoError,  # noqa: F401
                   MetricError, NumericError, check, lib)

DISTANCE, INTENSITY = L.PTG_DISTANCE, L.PTG_INTENSITY
STOP_NAMES = {0: "tolerance", 1: "budget", 2: "maxiters", 3: "stall"}


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _vp(a) -> Optional[int]:
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _prec(p) -> int:
    if p in ("c64", "complex64", L.PTG_C64):
        return L.PTG_C64
    if p in ("c128", "complex128", L.PTG_C128):
        return L.PTG_C128
    raise ConfigError(f"unknown precision {p!r}")


@dataclass
class SolverReport:
    """solvers.hpp:49-54 (+ EvalCounter)."""
    final_iterate: np.ndarray
    final_value: float
    history: np.ndarray            # [iters + 1, 3] = (weighted evals, value, |grad|)
    reason: str
    weighted_evals: float
    per_level_evals: list = field(default_factory=list)
    final_gradient: Optional[np.ndarray] = None


class Plan:
    """One ptychography problem level resident on one B200.

    positions: int [N, 2] (row0, col0) window offsets in scan order.
    probe: complex [M, M] or None for the reference's binary window.
    data: [N, M, M] non-negative intensities (float32 or float64), or None.
    """

    def __init__(self, n: int, M: int, w: int, positions, data=None, probe=None,
                 precision="c64", device: int = 0):
        self.n, self.M, self.w = int(n), int(M), int(w)
        self.rows = self.n   # object rows held (a BANDS shard holds fewer)
        self.positions = np.ascontiguousarray(positions, dtype=np.int32).reshape(-1, 2)
        self.N = self.positions.shape[0]
        self.precision = _prec(precision)
        self.probe = None if probe is None else _c128(probe).reshape(self.M, self.M)
        d = L.PlanDesc()
        d.n, d.M, d.w, d.N = self.n, self.M, self.w, self.N
        d.positions = self.positions.ctypes.data_as(C.POINTER(C.c_int32))
        d.probe = (self.probe.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))
                   if self.probe is not None else None)
        data_arr = None
        if data is not None:
            data_arr = np.ascontiguousarray(data)
            if data_arr.dtype not in (np.float32, np.float64):
                data_arr = data_arr.astype(np.float64)
            d.data = data_arr.ctypes.data
            d.data_dtype = L.PTG_F32 if data_arr.dtype == np.float32 else L.PTG_F64
        d.precision = self.precision
        d.device = int(device)
        self._h = C.c_void_p()
        check(lib().ptg_plan_create(C.byref(d), C.byref(self._h)))

    @classmethod
    def sharded(cls, n: int, M: int, w: int, positions, world: int, rank: int, layout: str = "bands",
                data=None, probe=None, precision="c64", device: int = 0) -> "Plan":
        """This rank's plan of a global problem (ptg_plan_create_sharded).
        positions: ALL N positions (global scan order); data: None or this
        rank's own patterns.  layout "bands" (object rows [row0, row0 + rows))
        or "replicated" (whole object)."""
        lay = {"replicated": L.PTG_SHARD_REPLICATED, "bands": L.PTG_SHARD_BANDS}[layout]
        self = cls.__new__(cls)
        self.n, self.M, self.w = int(n), int(M), int(w)
        allpos = np.ascontiguousarray(positions, dtype=np.int32).reshape(-1, 2)
        info = shard_layout(n, w, allpos, world, rank, layout)
        self.shard = info
        self.rows = info["rows"]
        self.positions = allpos[info["pos_begin"]:info["pos_end"]].copy()
        self.positions[:, 0] -= info["row0"]
        self.N = self.positions.shape[0]
        self.precision = _prec(precision)
        self.probe = None if probe is None else _c128(probe).reshape(self.M, self.M)
        d = L.PlanDesc()
        d.n, d.M, d.w, d.N = self.n, self.M, self.w, allpos.shape[0]
        d.positions = allpos.ctypes.data_as(C.POINTER(C.c_int32))
        d.probe = (self.probe.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))
                   if self.probe is not None else None)
        data_arr = None
        if data is not None:
            data_arr = np.ascontiguousarray(data)
            if data_arr.dtype not in (np.float32, np.float64):
                data_arr = data_arr.astype(np.float64)
            d.data = data_arr.ctypes.data
            d.data_dtype = L.PTG_F32 if data_arr.dtype == np.float32 else L.PTG_F64
        d.precision = self.precision
        d.device = int(device)
        self._h = C.c_void_p()
        check(lib().ptg_plan_create_sharded(C.byref(d), int(world), int(rank), lay, C.byref(self._h)))
        return self

    def bind_comm(self, comm: "Comm"):
        """Evaluations return the global value and this rank's gradient (NCCL inside libptg)."""
        check(lib().ptg_plan_bind_comm(self._h, comm._h))
        self._comm = comm   # keep the communicator alive with the plan

    def sync_halo(self, z):
        """BANDS: fill z's halo rows [own_rows, rows) from the next rank (device tensor)."""
        check(lib().ptg_band_sync_halo(self._h, _vp(z)))

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            lib().ptg_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- configuration
    def set_stream(self, stream_handle: Optional[int]):
        check(lib().ptg_plan_set_stream(self._h, stream_handle))

    def set_data(self, data):
        a = np.ascontiguousarray(data)
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        check(lib().ptg_plan_set_data(self._h, a.ctypes.data,
                                      L.PTG_F32 if a.dtype == np.float32 else L.PTG_F64))

    def load_ptyf(self, path):
        """loadRawStack (image_io.hpp:36) streamed straight into the plan's device data."""
        check(lib().ptg_plan_load_ptyf(self._h, os.fsencode(path)))

    def set_data_device(self, data_tensor):
        import torch
        dt = L.PTG_F32 if data_tensor.dtype == torch.float32 else L.PTG_F64
        check(lib().ptg_plan_set_data_device(self._h, data_tensor.data_ptr(), dt))

    @property
    def device_bytes(self) -> int:
        b = C.c_size_t()
        check(lib().ptg_plan_info(self._h, None, None, None, None, None, C.byref(b)))
        return b.value

    @property
    def launch_count(self) -> int:
        c = C.c_int64()
        check(lib().ptg_plan_launch_count(self._h, C.byref(c)))
        return c.value

    def set_timing(self, enable: bool = True):
        check(lib().ptg_plan_set_timing(self._h, int(enable)))

    def get_timing(self):
        """(frame_ms, frame_launches, gather_ms, gather_launches) since last call."""
        fm, gm = C.c_double(), C.c_double()
        fl, gl = C.c_int64(), C.c_int64()
        check(lib().ptg_plan_get_timing(self._h, C.byref(fm), C.byref(fl), C.byref(gm), C.byref(gl)))
        return fm.value, fl.value, gm.value, gl.value

    # -- objectives (host complex128)
    def evaluate(self, z, v=None, metric: int = DISTANCE, want_grad: bool = True, out=None):
        """(value, gradient); ``out`` may be a preallocated (e.g. pinned) complex128 array."""
        z = _c128(z).reshape(self.rows, self.n)
        v = None if v is None else _c128(v).reshape(self.rows, self.n)
        if out is not None:
            if out.dtype != np.complex128 or not out.flags.c_contiguous or out.size != self.rows * self.n:
                raise ConfigError("out must be a contiguous complex128 array of n*n entries")
            g = out
        else:
            g = np.empty((self.rows, self.n), np.complex128) if want_grad else None
        val = C.c_double()
        check(lib().ptg_eval(self._h, metric, z.ctypes.data, _vp(v), C.byref(val), _vp(g)))
        return val.value, g

    def phi_distance(self, z):
        return self.evaluate(z, None, DISTANCE)

    def phi_intensity_gaussian(self, z):
        return self.evaluate(z, None, INTENSITY)

    def evaluate_device(self, z, grad=None, v=None, metric: int = DISTANCE, value_dev=None,
                        sync_value: bool = True):
        """z, v, grad: torch CUDA tensors (n, n) in the plan precision."""
        val = C.c_double()
        check(lib().ptg_eval_device(self._h, metric, _vp(z), _vp(v), _vp(grad), _vp(value_dev),
                                    C.byref(val) if sync_value else None))
        return val.value if sync_value else None

    def project_modulus(self, z, k: int) -> np.ndarray:
        z = _c128(z).reshape(self.rows, self.n)
        out = np.empty((self.M, self.M), np.complex128)
        check(lib().ptg_project_modulus(self._h, z.ctypes.data, int(k), out.ctypes.data))
        return out

    def simulate(self, z, copy_out: bool = True) -> Optional[np.ndarray]:
        """d_j = |fft2(P o S_j z)|^2 on the GPU; becomes the plan's data."""
        z = _c128(z).reshape(self.rows, self.n)
        out = np.empty((self.N, self.M, self.M), np.float64) if copy_out else None
        check(lib().ptg_simulate(self._h, z.ctypes.data, _vp(out)))
        return out

    def simulate_device(self, z):
        check(lib().ptg_simulate_device(self._h, _vp(z)))

    def add_noise(self, level: float, seed: int = 0, uniforms=None):
        """addNoise (forward.hpp:44-48) on the resident data, on the GPU.
        uniforms: None = Philox4x64-10 stream; else 2 N M^2 uniforms in the
        reference's draw order (its std::mt19937_64 stream)."""
        u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float64)
        check(lib().ptg_add_noise(self._h, float(level), int(seed), _vp(u)))

    def add_poisson(self, photons: float, seed: int = 4):
        """Poisson photon noise at `photons` per pattern, on the GPU."""
        check(lib().ptg_add_poisson(self._h, float(photons), int(seed)))

    def data_host(self, metric: int = INTENSITY) -> np.ndarray:
        """The resident intensities (metric INTENSITY) or amplitudes, as float64 [N, M, M]."""
        out = np.empty((self.N, self.M, self.M), np.float64)
        check(lib().ptg_plan_get_data(self._h, int(metric), out.ctypes.data))
        return out

    # -- solvers
    def pie(self, z0, gamma: float = 0.0, sweeps: int = 1,
            max_weighted: float = float("inf")) -> SolverReport:
        z = _c128(z0).reshape(self.rows, self.n).copy()
        cap = sweeps + 2
        hist = (L.Hist * cap)()
        nh, rs = C.c_int(), C.c_int()
        fv, wt = C.c_double(), C.c_double()
        check(lib().ptg_pie(self._h, z.ctypes.data, float(gamma), int(sweeps), float(max_weighted),
                            C.byref(fv), hist, cap, C.byref(nh), C.byref(wt), C.byref(rs)))
        h = np.array([[hist[i].weighted, hist[i].value, hist[i].gnorm] for i in range(min(nh.value, cap))])
        return SolverReport(z, fv.value, h, STOP_NAMES[rs.value], wt.value, [int(wt.value)])

    def pie_sweep_device(self, z, gamma: float = 0.0):
        check(lib().ptg_pie_sweep_device(self._h, _vp(z), float(gamma)))

    def _solve(self, fn, z0, v, metric, cfg) -> SolverReport:
        c = L.SolverCfg()
        lib().ptg_solver_cfg_default(C.byref(c))
        for k, val in cfg.items():
            setattr(c, k, val)
        z0 = _c128(z0).reshape(self.rows, self.n)
        v = None if v is None else _c128(v).reshape(self.rows, self.n)
        z = np.empty_like(z0)
        g = np.empty_like(z0)
        cap = c.max_iters + 2
        hist = (L.Hist * cap)()
        rep = L.Report()
        check(fn(self._h, metric, _vp(v), z0.ctypes.data, C.byref(c), z.ctypes.data, g.ctypes.data,
                 C.byref(rep), hist, cap))
        h = np.array([[hist[i].weighted, hist[i].value, hist[i].gnorm]
                      for i in range(min(rep.hist_len, cap))])
        return SolverReport(z, rep.final_value, h, STOP_NAMES[rep.reason], rep.weighted,
                            [int(rep.per_level[0])], g)

    def lbfgs(self, z0, v=None, metric: int = DISTANCE, **cfg) -> SolverReport:
        """lbfgs (solvers.hpp:92-95), GPU-resident."""
        return self._solve(lib().ptg_lbfgs, z0, v, metric, cfg)

    def truncated_newton(self, z0, v=None, metric: int = DISTANCE, **cfg) -> SolverReport:
        """truncatedNewton (solvers.hpp:101-104), GPU-resident."""
        return self._solve(lib().ptg_truncated_newton, z0, v, metric, cfg)


class Hierarchy:
    """buildHierarchy + mgoptDriver (multigrid.hpp:61-95), coarse levels built on device."""

    def __init__(self, plan: Plan, depth: int, metric: int = DISTANCE, **mg):
        self.plan = plan
        self.depth = int(depth)
        c = L.MgCfg()
        lib().ptg_mg_cfg_default(C.byref(c))
        for k, val in mg.items():
            setattr(c, k, val)
        self.cfg = c
        self._h = C.c_void_p()
        check(lib().ptg_hier_create(plan._h, metric, self.depth, C.byref(c), C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib().ptg_hier_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def driver(self, z0, budget: float = 100.0, grad_tol_rel: float = 0.0,
               grad_tol_abs: float = 1e-13, max_cycles: int = 1000000) -> SolverReport:
        d = L.DriverCfg(budget, grad_tol_rel, grad_tol_abs, max_cycles)
        n = self.plan.n
        z0 = _c128(z0).reshape(n, n)
        z = np.empty_like(z0)
        cap = min(max_cycles, 100000) + 2
        hist = (L.Hist * cap)()
        rep = L.Report()
        check(lib().ptg_mgopt_driver(self._h, z0.ctypes.data, C.byref(d), z.ctypes.data, C.byref(rep),
                                     hist, cap))
        h = np.array([[hist[i].weighted, hist[i].value, hist[i].gnorm]
                      for i in range(min(rep.hist_len, cap))])
        return SolverReport(z, rep.final_value, h, STOP_NAMES[rep.reason], rep.weighted,
                            [int(rep.per_level[l]) for l in range(self.depth)])

    def level(self, l: int) -> "Plan":
        """Non-owning Plan view of hierarchy level l (0 = the fine plan)."""
        h = C.c_void_p()
        check(lib().ptg_hier_level(self._h, int(l), C.byref(h)))
        if l == 0:
            return self.plan
        v = Plan.__new__(Plan)
        n, M, w, N = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(lib().ptg_plan_info(h, C.byref(n), C.byref(M), C.byref(w), C.byref(N), None, None))
        v.n, v.M, v.w, v.N = n.value, M.value, w.value, N.value
        v.rows = v.n
        v.precision = self.plan.precision
        v._h = h
        v._view_of = self   # keep the hierarchy alive; never destroyed through the view
        v.close = lambda: None
        return v

    def cycle_device(self, z, grad, value: float):
        """One top-level V-cycle in place on device tensors (z, grad); returns
        (new value, weighted evals, per-level eval counts)."""
        val = C.c_double(value)
        rep = L.Report()
        check(lib().ptg_mgopt_cycle_device(self._h, _vp(z), C.byref(val), _vp(grad), C.byref(rep)))
        return val.value, rep.weighted, [int(rep.per_level[l]) for l in range(self.depth)]


# ------------------------------------------------------------------ transfers
def restrict_field(fine) -> np.ndarray:
    f = _c128(fine)
    n = f.shape[0]
    out = np.empty((n // 2, n // 2), np.complex128)
    check(lib().ptg_restrict_field(f.ctypes.data, n, out.ctypes.data))
    return out


def prolong_field(coarse) -> np.ndarray:
    c = _c128(coarse)
    nH = c.shape[0]
    out = np.empty((2 * nH, 2 * nH), np.complex128)
    check(lib().ptg_prolong_field(c.ctypes.data, nH, out.ctypes.data))
    return out


def restrict_data(fine) -> np.ndarray:
    d = np.ascontiguousarray(fine, dtype=np.float64)
    N, M = d.shape[0], d.shape[1]
    out = np.empty((N, M // 2, M // 2), np.float64)
    check(lib().ptg_restrict_data(d.ctypes.data, N, M, out.ctypes.data))
    return out


def shard_layout(n: int, w: int, positions, world: int, rank: int, layout: str = "bands") -> dict:
    """The partition of a global scan over `world` ranks (host only, ptg_shard_layout)."""
    lay = {"replicated": L.PTG_SHARD_REPLICATED, "bands": L.PTG_SHARD_BANDS}[layout]
    pos = np.ascontiguousarray(positions, dtype=np.int32).reshape(-1, 2)
    out = np.zeros(6, np.int32)
    check(lib().ptg_shard_layout(int(n), int(w), pos.shape[0], pos.ctypes.data, int(world), int(rank), lay,
                                 out.ctypes.data))
    keys = ("pos_begin", "pos_end", "row0", "rows", "own_rows", "halo_prev")
    return {k: int(v) for k, v in zip(keys, out)}


class Comm:
    """An NCCL communicator inside libptg (one per process / GPU).  The
    128-byte ncclUniqueId is made on rank 0 and broadcast with `broadcast`
    (e.g. torch.distributed over any backend)."""

    def __init__(self, world: int, rank: int, device: int, broadcast):
        uid = np.zeros(128, np.uint8)
        if rank == 0:
            check(lib().ptg_comm_unique_id(uid.ctypes.data))
        uid = np.ascontiguousarray(broadcast(uid), dtype=np.uint8)
        self._h = C.c_void_p()
        check(lib().ptg_comm_init(uid.ctypes.data, int(world), int(rank), int(device), C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib().ptg_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_count() -> int:
    c = C.c_int()
    check(lib().ptg_device_count(C.byref(c)))
    return c.value


def write_ptyf(path, stack) -> None:
    """saveRawStack (image_io.hpp:37, format :10-20): "PTYF", u32 n, u32 k, u32 0,
    then k row-major float64 n x n planes (little endian)."""
    a = np.ascontiguousarray(stack, dtype="<f8")
    if a.ndim == 2:
        a = a[None]
    k, n, n2 = a.shape
    if n != n2 or k < 1:
        raise ValueError("write_ptyf: expected a stack of square patterns")
    with open(path, "wb") as f:
        f.write(b"PTYF" + np.array([n, k, 0], "<u4").tobytes())
        f.write(a.tobytes())


# ------------------------------------------------------------ diagnostics
def _square_pair(z, z_true):
    z = _c128(z)
    zt = _c128(z_true)
    if z.ndim != 2 or z.shape[0] != z.shape[1]:
        raise GeometryError("metric: fields must be square")
    if z.shape != zt.shape:
        raise DomainError("metric: field sizes differ")   # checkSameSize (metrics.cpp:17-20)
    return z, zt


def metrics(z, z_true, mask: int = L.PTG_METRIC_ALL) -> dict:
    """metrics.hpp:9-24 computed on the GPU (host complex128 fields)."""
    z, zt = _square_pair(z, z_true)
    m = L.Metrics()
    check(lib().ptg_metrics_host(z.ctypes.data, zt.ctypes.data, z.shape[0], mask, C.byref(m)))
    return {"relative_error": m.relative_error, "magnitude_rel_error": m.magnitude_rel_error,
            "phase_ssim": m.phase_ssim}


def metrics_device(z, z_true, mask: int = L.PTG_METRIC_ALL, stream: int = 0) -> dict:
    """The same on device tensors (complex64 or complex128, n x n) — no host copy of the fields."""
    import torch
    if z.shape != z_true.shape or z.dtype != z_true.dtype:
        raise DomainError("metric: field sizes differ")
    prec = {torch.complex64: L.PTG_C64, torch.complex128: L.PTG_C128}[z.dtype]
    m = L.Metrics()
    check(lib().ptg_metrics_device(prec, z.data_ptr(), z_true.data_ptr(), z.shape[0], mask, C.byref(m),
                                   stream or None))
    return {"relative_error": m.relative_error, "magnitude_rel_error": m.magnitude_rel_error,
            "phase_ssim": m.phase_ssim}


def relative_error(z, z_true) -> float:
    return metrics(z, z_true, L.PTG_METRIC_RELATIVE_ERROR)["relative_error"]


def magnitude_rel_error(z, z_true) -> float:
    return metrics(z, z_true, L.PTG_METRIC_MAGNITUDE_REL_ERROR)["magnitude_rel_error"]


def phase_ssim(z, z_true) -> float:
    return metrics(z, z_true, L.PTG_METRIC_PHASE_SSIM)["phase_ssim"]


def canonical_phase(z) -> np.ndarray:
    """canonicalPhase (metrics.hpp:15-18) on the GPU."""
    z = _c128(z)
    out = np.empty(z.shape, np.float64)
    check(lib().ptg_canonical_phase(z.ctypes.data, z.shape[0], out.ctypes.data))
    return out
