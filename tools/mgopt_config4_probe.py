"""One 4-level MG/OPT V-cycle on config 4 (n = 4096, M = 256, 3721 patterns,
Poisson data), device-resident (dev tool): wall time, evaluations per level."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_05628_b200 import Hierarchy, Plan, synth  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = synth.CONFIGS[cid]
obj, probe, pos = synth.make_inputs(cfg)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision=cfg.precision)
plan.set_stream(stream.cuda_stream)
host = plan.simulate(obj, copy_out=bool(cfg.photons))
if cfg.photons:
    plan.add_poisson(cfg.photons, seed=4)
h = Hierarchy(plan, cfg.depth)
z = torch.ones(cfg.n, cfg.n, dtype=torch.complex64, device="cuda")
g = torch.empty_like(z)
v = plan.evaluate_device(z, g)
print(f"config {cid}: depth {cfg.depth}, initial value {v:.6e}", flush=True)
for c in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, wt, per = h.cycle_device(z, g, v)
    torch.cuda.synchronize()
    print(f"cycle {c}: {1e3 * (time.perf_counter() - t0):.1f} ms, value {v:.6e}, weighted evals {wt}, per level {per}",
          flush=True)
print("device memory (GB):", torch.cuda.max_memory_allocated() / 1e9)
