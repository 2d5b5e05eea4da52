"""Seeded synthetic inputs for the BASELINE.json configurations.

The paper's images are not available; BASELINE.json specifies
seeded synthetic objects instead, reproduced here:

* object: magnitude = smooth random field (uniform noise, periodic Gaussian
  filter sigma px) rescaled to [0.5, 1]; phase = independent smooth field in
  [-pi/4, pi/4]
* probe: Gaussian amplitude (sigma px) x exp(i a r^2), r from the frame centre
* scan: serpentine raster (field.cpp:77-83 order), optional seeded uniform
  integer jitter clamped to [0, n - w]
* data: d_j = |fft2(P o S_j x)|^2 (computed by the caller: GPU simulate for the
  product, the oracle in tests), optional Poisson noise at a photon budget

Inputs are generated once on the host and fed byte-identically to the GPU
and to the CPU oracle.  RNG: the reference's std::mt19937_64 +
rng::uniform01 (rng.hpp:14-16, via ptg_uniform01_stream) with fixed seeds
(object magnitude 1 / phase 2, jitter 3); Poisson noise is drawn on the GPU
from Philox4x64-10 keyed by seed 4 (ptg_add_poisson).  A C++ user regenerates
the same fields with the reference's own rng.hpp.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import scipy.fft as sfft


@dataclass(frozen=True)
class Config:
    cid: int
    n: int
    M: int
    steps: int
    step: int
    sigma_obj: float
    sigma_probe: float
    a: float
    precision: str
    jitter: int = 0
    photons: Optional[float] = None
    depth: int = 2

    @property
    def w(self) -> int:
        return self.M

    @property
    def N(self) -> int:
        return self.steps * self.steps

    def describe(self) -> str:
        j = f", jitter +-{self.jitter}px" if self.jitter else ""
        p = f", Poisson {self.photons:g} photons" if self.photons else ", noiseless"
        return (f"config{self.cid}: {self.precision} object {self.n}x{self.n}, probe {self.M}x{self.M} "
                f"(sigma {self.sigma_probe}, a {self.a}), {self.steps}x{self.steps} raster step "
                f"{self.step} ({self.N} patterns){j}{p}")


# BASELINE.json "configs" (index 0 = the CPU-runnable oracle case)
CONFIGS = {
    1: Config(1, 128, 32, 13, 8, 4.0, 8.0, 0.01, "c128", depth=2),
    2: Config(2, 512, 64, 29, 16, 8.0, 16.0, 0.0025, "c64", depth=2),
    3: Config(3, 1024, 128, 29, 32, 8.0, 32.0, 0.0, "c64", jitter=2, depth=3),
    4: Config(4, 4096, 256, 61, 64, 8.0, 64.0, 0.0, "c64", photons=1e6, depth=4),
    5: Config(5, 8192, 256, 166, 48, 8.0, 64.0, 0.0006, "c64", photons=1e5, depth=4),
}


def uniform01(seed: int, count: int) -> np.ndarray:
    """rng::uniform01 draws of std::mt19937_64(seed) (rng.hpp:14-16), row-major."""
    from paper_1810_05628_b200 import _lib
    out = np.empty(count, np.float64)
    _lib.check(_lib.lib().ptg_uniform01_stream(int(seed), count, out.ctypes.data))
    return out


def smooth_field(n: int, sigma: float, seed: int) -> np.ndarray:
    """Uniform noise (mt19937_64(seed), row-major), periodically Gaussian-filtered
    (sigma px), min-max to [0, 1]."""
    u = uniform01(seed, n * n).reshape(n, n)
    f = np.fft.fftfreq(n)
    k = np.exp(-2.0 * np.pi ** 2 * sigma ** 2 * (f[:, None] ** 2 + f[None, :] ** 2))
    # scipy's pocketfft with all host threads (8192^2: 0.3 s vs 4.6 s per
    # transform for numpy's single-threaded one); rows are transformed
    # independently, so the result does not depend on the thread count
    s = np.real(sfft.ifft2(sfft.fft2(u, workers=-1) * k, workers=-1))
    lo, hi = s.min(), s.max()
    return (s - lo) / (hi - lo) if hi > lo else np.zeros_like(s)


def make_object(n: int, sigma: float, seed_mag: int = 1, seed_phase: int = 2) -> np.ndarray:
    mag = 0.5 + 0.5 * smooth_field(n, sigma, seed_mag)
    ph = (2.0 * smooth_field(n, sigma, seed_phase) - 1.0) * (np.pi / 4)
    return (mag * np.exp(1j * ph)).astype(np.complex128)


def make_probe(M: int, sigma: float, a: float) -> np.ndarray:
    c = (M - 1) / 2.0
    y, x = np.mgrid[0:M, 0:M]
    r2 = (y - c) ** 2 + (x - c) ** 2
    return (np.exp(-r2 / (2.0 * sigma ** 2)) * np.exp(1j * a * r2)).astype(np.complex128)


def raster(n: int, w: int, steps: int, step: int, jitter: int = 0, seed: int = 3) -> np.ndarray:
    """Serpentine raster (generateRasterScan order, field.cpp:77-83) + optional jitter."""
    pos = []
    for i in range(steps):
        for j in range(steps):
            jj = j if i % 2 == 0 else steps - 1 - j
            pos.append((i * step, jj * step))
    pos = np.array(pos, dtype=np.int64)
    if jitter:
        # U{-jitter..jitter} per coordinate, (row, col) per position in scan order
        u = uniform01(seed, pos.size).reshape(pos.shape)
        pos = pos + np.floor(u * (2 * jitter + 1)).astype(np.int64) - jitter
    pos = np.clip(pos, 0, n - w)
    return pos.astype(np.int32)


def make_inputs(cfg: Config):
    """(object, probe, positions) for a configuration; data is simulated by the caller."""
    obj = make_object(cfg.n, cfg.sigma_obj)
    probe = make_probe(cfg.M, cfg.sigma_probe, cfg.a)
    pos = raster(cfg.n, cfg.w, cfg.steps, cfg.step, cfg.jitter)
    return obj, probe, pos


def small_config(n=64, M=16, steps=7, step=8, sigma_obj=3.0, sigma_probe=4.0, a=0.02,
                 precision="c128", jitter=0) -> Config:
    return Config(0, n, M, steps, step, sigma_obj, sigma_probe, a, precision, jitter)
