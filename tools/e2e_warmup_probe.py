"""e2e (ptg_eval, pinned buffers) in consecutive blocks of 50 calls: how long
until a fresh process / fresh buffers reach steady state (dev tool)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1810_05628_b200 import Plan, synth  # noqa: E402

cfg = synth.CONFIGS[2]
obj, probe, pos = synth.make_inputs(cfg)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision="c64")
plan.set_stream(stream.cuda_stream)
plan.simulate(obj, copy_out=False)
zh = torch.ones(cfg.n, cfg.n, dtype=torch.complex128).pin_memory().numpy()
gh = torch.empty(cfg.n, cfg.n, dtype=torch.complex128).pin_memory().numpy()
for blk in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        plan.evaluate(zh, out=gh)
    print(f"block {blk}: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us", flush=True)
