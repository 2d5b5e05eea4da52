"""ctypes binding of libptg.so (include/ptg.h) — the product's only compute path.

Loading fails loudly when the in-tree shared library is missing; there is no
CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# PTG_LIB: alternative build of the same library (A/B experiments on kernel variants)
LIB_PATH = os.environ.get("PTG_LIB") or os.path.join(PKG, "lib", "libptg.so")

PTG_OK = 0
PTG_C64, PTG_C128 = 0, 1
PTG_F32, PTG_F64 = 0, 1
PTG_DISTANCE, PTG_INTENSITY = 0, 1
PTG_SHARD_NONE, PTG_SHARD_REPLICATED, PTG_SHARD_BANDS = 0, 1, 2


# --- exception hierarchy mirroring /root/reference/proj/include/ptycho/errors.hpp:12-43
class Error(RuntimeError):
    """ptycho::Error"""


class ConfigError(Error):
    """ptycho::ConfigError"""


class GeometryError(ConfigError):
    """ptycho::GeometryError"""


class DomainError(ConfigError):
    """ptycho::DomainError"""


class MetricError(ConfigError):
    """ptycho::MetricError"""


class IoError(Error):
    """ptycho::IoError"""


class NumericError(Error):
    """ptycho::NumericError"""


class CudaError(Error):
    """CUDA / device failure (no CPU fallback exists)."""


_STATUS = {10: ConfigError, 11: GeometryError, 12: DomainError, 13: MetricError, 2: IoError,
           3: NumericError, 4: CudaError}

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class PlanDesc(C.Structure):
    _fields_ = [("n", C.c_int), ("M", C.c_int), ("w", C.c_int), ("N", C.c_int),
                ("positions", C.POINTER(C.c_int32)), ("probe", _dp), ("data", _vp),
                ("data_dtype", C.c_int), ("precision", C.c_int), ("device", C.c_int)]


class Hist(C.Structure):
    _fields_ = [("weighted", C.c_double), ("value", C.c_double), ("gnorm", C.c_double)]


class Metrics(C.Structure):
    _fields_ = [("relative_error", C.c_double), ("magnitude_rel_error", C.c_double), ("phase_ssim", C.c_double)]


PTG_METRIC_RELATIVE_ERROR, PTG_METRIC_MAGNITUDE_REL_ERROR, PTG_METRIC_PHASE_SSIM, PTG_METRIC_ALL = 1, 2, 4, 7


class SolverCfg(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("grad_tol_rel", C.c_double), ("grad_tol_abs", C.c_double),
                ("lbfgs_memory", C.c_int), ("linesearch_max", C.c_int), ("max_weighted", C.c_double),
                ("cg_max_iters", C.c_int), ("cg_rel_tol", C.c_double)]


class MgCfg(C.Structure):
    _fields_ = [("k1", C.c_int), ("k2", C.c_int), ("coarsest_max_iters", C.c_int),
                ("coarsest_grad_tol_rel", C.c_double), ("intermediate_grad_tol_rel", C.c_double),
                ("lbfgs_memory", C.c_int), ("linesearch_max", C.c_int), ("grad_tol_abs", C.c_double)]


class DriverCfg(C.Structure):
    _fields_ = [("budget", C.c_double), ("grad_tol_rel", C.c_double), ("grad_tol_abs", C.c_double),
                ("max_cycles", C.c_int)]


class Report(C.Structure):
    _fields_ = [("final_value", C.c_double), ("weighted", C.c_double), ("per_level", C.c_long * 16),
                ("reason", C.c_int), ("hist_len", C.c_int)]


# every symbol include/ptg.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "ptg_last_error", "ptg_version", "ptg_device_count",
    "ptg_plan_create", "ptg_plan_destroy", "ptg_plan_set_stream", "ptg_plan_set_data",
    "ptg_plan_set_data_device", "ptg_plan_load_ptyf", "ptg_plan_get_data", "ptg_plan_info", "ptg_plan_launch_count",
    "ptg_plan_set_timing", "ptg_plan_get_timing",
    "ptg_eval", "ptg_eval_device", "ptg_project_modulus", "ptg_simulate", "ptg_simulate_device",
    "ptg_add_noise", "ptg_add_poisson", "ptg_philox4x64", "ptg_uniform01_stream",
    "ptg_pie", "ptg_pie_cb", "ptg_pie_sweep_device", "ptg_fft2",
    "ptg_lbfgs_ex", "ptg_truncated_newton_ex", "ptg_mgopt_driver_ex", "ptg_mgopt_cycle",
    "ptg_restrict_field", "ptg_prolong_field", "ptg_restrict_data",
    "ptg_restrict_field_device", "ptg_prolong_field_device", "ptg_restrict_data_device",
    "ptg_halo_bytes", "ptg_halo_pack", "ptg_halo_unpack",
    "ptg_comm_unique_id", "ptg_comm_init", "ptg_comm_destroy", "ptg_shard_layout", "ptg_plan_create_sharded",
    "ptg_plan_bind_comm", "ptg_band_sync_halo",
    "ptg_solver_cfg_default", "ptg_mg_cfg_default", "ptg_driver_cfg_default",
    "ptg_metrics_device", "ptg_metrics_host", "ptg_canonical_phase",
    "ptg_lbfgs", "ptg_truncated_newton", "ptg_hier_create", "ptg_hier_destroy", "ptg_hier_level",
    "ptg_mgopt_driver", "ptg_mgopt_cycle_device",
]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libptg.so not built at {LIB_PATH}: run `python -m paper_1810_05628_b200._build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.ptg_last_error.restype = C.c_char_p
    L.ptg_plan_create.argtypes = [C.POINTER(PlanDesc), C.POINTER(_vp)]
    L.ptg_plan_destroy.argtypes = [_vp]
    L.ptg_plan_set_stream.argtypes = [_vp, _vp]
    L.ptg_plan_set_data.argtypes = [_vp, _vp, C.c_int]
    L.ptg_plan_set_data_device.argtypes = [_vp, _vp, C.c_int]
    L.ptg_plan_load_ptyf.argtypes = [_vp, C.c_char_p]
    L.ptg_plan_get_data.argtypes = [_vp, C.c_int, _vp]
    L.ptg_metrics_device.argtypes = [C.c_int, _vp, _vp, C.c_int, C.c_uint, C.POINTER(Metrics), _vp]
    L.ptg_metrics_host.argtypes = [_vp, _vp, C.c_int, C.c_uint, C.POINTER(Metrics)]
    L.ptg_canonical_phase.argtypes = [_vp, C.c_int, _vp]
    L.ptg_plan_info.argtypes = [_vp] + [C.POINTER(C.c_int)] * 5 + [C.POINTER(C.c_size_t)]
    L.ptg_plan_launch_count.argtypes = [_vp, C.POINTER(C.c_int64)]
    L.ptg_eval.argtypes = [_vp, C.c_int, _vp, _vp, _dp, _vp]
    L.ptg_eval_device.argtypes = [_vp, C.c_int, _vp, _vp, _vp, _vp, _dp]
    L.ptg_project_modulus.argtypes = [_vp, _vp, C.c_int, _vp]
    L.ptg_simulate.argtypes = [_vp, _vp, _vp]
    L.ptg_simulate_device.argtypes = [_vp, _vp]
    L.ptg_pie.argtypes = [_vp, _vp, C.c_double, C.c_int, C.c_double, _dp, C.POINTER(Hist), C.c_int,
                          C.POINTER(C.c_int), _dp, C.POINTER(C.c_int)]
    L.ptg_pie_sweep_device.argtypes = [_vp, _vp, C.c_double]
    L.ptg_add_noise.argtypes = [_vp, C.c_double, C.c_uint64, _vp]
    L.ptg_add_poisson.argtypes = [_vp, C.c_double, C.c_uint64]
    L.ptg_philox4x64.argtypes = [C.c_int, _vp, _vp, C.c_size_t, _vp]
    L.ptg_uniform01_stream.argtypes = [C.c_uint64, C.c_size_t, _vp]
    L.ptg_restrict_field.argtypes = [_vp, C.c_int, _vp]
    L.ptg_prolong_field.argtypes = [_vp, C.c_int, _vp]
    L.ptg_restrict_data.argtypes = [_vp, C.c_int, C.c_int, _vp]
    L.ptg_restrict_field_device.argtypes = [C.c_int, _vp, C.c_int, _vp, _vp]
    L.ptg_prolong_field_device.argtypes = [C.c_int, _vp, C.c_int, _vp, _vp]
    L.ptg_restrict_data_device.argtypes = [C.c_int, _vp, C.c_int, C.c_int, _vp, _vp]
    L.ptg_comm_unique_id.argtypes = [_vp]
    L.ptg_comm_init.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]
    L.ptg_comm_destroy.argtypes = [_vp]
    L.ptg_shard_layout.argtypes = [C.c_int, C.c_int, C.c_int, _vp, C.c_int, C.c_int, C.c_int, _vp]
    L.ptg_plan_create_sharded.argtypes = [C.POINTER(PlanDesc), C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]
    L.ptg_plan_bind_comm.argtypes = [_vp, _vp]
    L.ptg_band_sync_halo.argtypes = [_vp, _vp]
    L.ptg_halo_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
    L.ptg_halo_bytes.restype = C.c_size_t
    L.ptg_halo_pack.argtypes = [C.c_int, _vp, C.c_int, C.c_int, _vp, _vp, _vp]
    L.ptg_halo_unpack.argtypes = [C.c_int, _vp, C.c_int, C.c_int, _vp, C.c_int, C.c_int, _vp, _vp]
    L.ptg_solver_cfg_default.argtypes = [C.POINTER(SolverCfg)]
    L.ptg_solver_cfg_default.restype = None
    L.ptg_mg_cfg_default.argtypes = [C.POINTER(MgCfg)]
    L.ptg_mg_cfg_default.restype = None
    L.ptg_driver_cfg_default.argtypes = [C.POINTER(DriverCfg)]
    L.ptg_driver_cfg_default.restype = None
    L.ptg_lbfgs.argtypes = [_vp, C.c_int, _vp, _vp, C.POINTER(SolverCfg), _vp, _vp, C.POINTER(Report),
                            C.POINTER(Hist), C.c_int]
    L.ptg_truncated_newton.argtypes = [_vp, C.c_int, _vp, _vp, C.POINTER(SolverCfg), _vp, _vp,
                                       C.POINTER(Report), C.POINTER(Hist), C.c_int]
    L.ptg_hier_create.argtypes = [_vp, C.c_int, C.c_int, C.POINTER(MgCfg), C.POINTER(_vp)]
    L.ptg_hier_destroy.argtypes = [_vp]
    L.ptg_hier_level.argtypes = [_vp, C.c_int, C.POINTER(_vp)]
    L.ptg_mgopt_driver.argtypes = [_vp, _vp, C.POINTER(DriverCfg), _vp, C.POINTER(Report),
                                   C.POINTER(Hist), C.c_int]
    L.ptg_mgopt_cycle_device.argtypes = [_vp, _vp, _dp, _vp, C.POINTER(Report)]
    L.ptg_device_count.argtypes = [C.POINTER(C.c_int)]
    L.ptg_plan_set_timing.argtypes = [_vp, C.c_int]
    L.ptg_plan_get_timing.argtypes = [_vp, _dp, C.POINTER(C.c_int64), _dp, C.POINTER(C.c_int64)]
    _lib = L
    return L


def check(rc: int):
    if rc != PTG_OK:
        msg = lib().ptg_last_error().decode(errors="replace")
        raise _STATUS.get(rc, Error)(f"{msg} (status {rc})")
