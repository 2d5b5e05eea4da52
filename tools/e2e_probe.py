"""e2e probe (dev tool): PCIe floor for 4 MiB pinned copies, and ptg_eval wall time."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_05628_b200 import Plan, synth  # noqa: E402

cfg = synth.CONFIGS[2]
obj, probe, pos = synth.make_inputs(cfg)
plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision="c64")
plan.simulate(obj, copy_out=False)
zh = torch.ones(cfg.n, cfg.n, dtype=torch.complex128).pin_memory()
gh = torch.empty(cfg.n, cfg.n, dtype=torch.complex128).pin_memory()
zd = torch.empty(cfg.n, cfg.n, dtype=torch.complex128, device="cuda")
for name, fn in [("h2d 4MiB", lambda: zd.copy_(zh)), ("d2h 4MiB", lambda: gh.copy_(zd)),
                 ("h2d+d2h concurrent", None)]:
    if fn is None:
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        zd2 = torch.empty_like(zd)
        def fn():
            with torch.cuda.stream(s1):
                zd.copy_(zh, non_blocking=True)
            with torch.cuda.stream(s2):
                gh.copy_(zd2, non_blocking=True)
            torch.cuda.synchronize()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us")
zn, gn = zh.numpy(), gh.numpy()
for _ in range(3):
    plan.evaluate(zn, out=gn)
t0 = time.perf_counter()
for _ in range(50):
    plan.evaluate(zn, out=gn)
print(f"ptg_eval: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us")
