"""paper_1810_05628_b200 — B200-native (sm_100a) ptychographic objective/gradient
hot path of MG/OPT phase retrieval (arXiv 1810.05628).

The compute lives in ``lib/libptg.so`` (hand-written CUDA, C-ABI in
``include/ptg.h``); this package is its host-side mirror of the reference's
``ptycho::`` API.  Importing the package does not touch the GPU; the first
call that needs libptg loads it and fails loudly if it is missing.
"""
from .ptycho import (DISTANCE, INTENSITY, ConfigError, CudaError, DomainError, Error,  # noqa: F401
                     GeometryError, Hierarchy, IoError, MetricError, NumericError, Plan,
                     SolverReport, device_count, prolong_field, restrict_data, restrict_field,
                     write_ptyf, metrics, metrics_device, relative_error, magnitude_rel_error,
                     phase_ssim, canonical_phase, Comm, shard_layout)

__all__ = ["Plan", "Hierarchy", "SolverReport", "restrict_field", "prolong_field", "restrict_data",
           "DISTANCE", "INTENSITY", "Error", "ConfigError", "GeometryError", "DomainError",
           "MetricError", "IoError", "NumericError", "CudaError", "device_count", "write_ptyf",
           "metrics", "metrics_device", "relative_error", "magnitude_rel_error", "phase_ssim", "canonical_phase",
           "Comm", "shard_layout"]
