"""Generate tests/golden/noise_golden.npz from the UNMODIFIED reference library.

Run in the build container (needs oracle/_ref/libptycho_ref.so):
    python tests/golden/make_noise_golden.py

addNoise (forward.cpp:56-86) on a small seeded stack, plus the reference
engine's own uniform stream (std::mt19937_64 + rng::uniform01, rng.hpp:14-16)
that produced it, so the GPU's ptg_add_noise can be fed the same uniforms on
the GPU box (where /root/reference does not exist) and checked against the
reference's output.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ptgo  # noqa: E402


def main():
    assert ptgo.has_reference(), "build oracle/_ref/libptycho_ref.so first (make -C oracle)"
    rng = np.random.default_rng(77)
    out = {}
    for tag, (N, m, level, seed) in {"a": (3, 16, 0.05, 11), "b": (2, 32, 0.3, 12345)}.items():
        d = rng.uniform(0, 4, (N, m, m)) ** 2
        d[0, :2, :3] = 0.0            # zeros stay >= 0 after the clamp
        out[f"noise_{tag}_data"] = d
        out[f"noise_{tag}_meta"] = np.array([level, seed], dtype=np.float64)
        out[f"noise_{tag}_uniforms"] = ptgo.ref_uniform_stream(seed, 2 * N * m * m)
        out[f"noise_{tag}_out"] = ptgo.ref_add_noise(d, level, seed)
    path = os.path.join(HERE, "noise_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
