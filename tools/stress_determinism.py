"""Stress: repeated evaluations must be bitwise identical (races show up as
rare differences).  Usage: python tools/stress_determinism.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1810_05628_b200 import Plan, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
cases = [synth.Config(0, 2 * M + 8, M, 3, M // 2 + 3, 8.0, M / 4, 0.0006, "c64", jitter=2) for M in (128, 256)]
cases += [synth.CONFIGS[2], synth.CONFIGS[3]]
for cfg in cases:
    obj, probe, pos = synth.make_inputs(cfg)
    plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision="c64")
    plan.simulate(obj, copy_out=False)
    z = torch.tensor((obj * 0.9 + 0.05).astype(np.complex64), device="cuda")
    for shift in (False, True):
        v = (z * 0.01) if shift else None
        g0 = torch.empty_like(z)
        val0 = plan.evaluate_device(z, g0, v=v)
        bad = 0
        for r in range(reps):
            g = torch.empty_like(z)
            val = plan.evaluate_device(z, g, v=v)
            if val != val0 or not torch.equal(g, g0):
                bad += 1
                if bad <= 3:
                    d = (g - g0).abs().max().item()
                    print(f"  M={cfg.M} n={cfg.n} shift={shift} rep {r}: value {val!r} vs {val0!r}, max |dg| {d:.3e}")
        print(f"M={cfg.M} n={cfg.n} N={cfg.N} shift={shift}: {bad}/{reps} differ", flush=True)
