"""MG/OPT at the reference's DEFAULT settings (coarsest solve 100 LBFGS
iterations for depth > 2, multigrid.cpp:123-128) from the UNMODIFIED reference.

Run in the build container:   python tests/golden/make_mg_default_golden.py

reference_golden.npz caps the coarsest solve at 10 iterations because its
noiseless data lets 100 iterations reach the rounding floor, where
accept/reject decisions depend on the FFT's summation order.  Here the data
carries the reference's own addNoise (forward.cpp:56-86), so the objective
stays well above that floor and the default-settings trajectory is
reproducible by any correctly rounded implementation: per-level evaluation
counts must match exactly.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ptgo  # noqa: E402


def rf(n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    return scale * (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n)))


CASES = {"a": (32, 16, 8, 0.2, 3), "b": (64, 16, 8, 0.3, 3)}


def main():
    assert ptgo.has_reference(), "build oracle/_ref/libptycho_ref.so first (make -C oracle)"
    out = {}
    for tag, (n, w, s, level, depth) in CASES.items():
        pos = ptgo.ref_raster(n, w, s)[:, :2].copy()
        truth = 1.0 + rf(n, 11, 0.5)
        data = ptgo.ref_add_noise(ptgo.ref_simulate(n, w, pos, truth), level, 5)
        z0 = 1.0 + rf(n, 41, 0.25)
        r = ptgo.ref_mgopt(0, n, w, s, data, z0, depth, budget=1e9, max_cycles=3)   # coarsest_max_iters = default
        out[f"{tag}_geom"] = np.array([n, w, s, depth])
        out[f"{tag}_pos"], out[f"{tag}_data"], out[f"{tag}_z0"] = pos, data, z0
        out[f"{tag}_z"], out[f"{tag}_hist"] = r.z, r.history
        out[f"{tag}_meta"] = np.array([r.value, r.weighted, r.reason] + r.per_level)
        print(tag, r.per_level, r.weighted, r.value)
    path = os.path.join(HERE, "mg_default_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
