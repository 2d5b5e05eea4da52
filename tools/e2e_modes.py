"""e2e (ptg_eval, pinned host buffers) measured at several points of a
bench-like sequence (dev tool): after creation, after flushed device
evaluations, after the timing-attribution loop."""
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


def e2e(tag):
    for _ in range(3):
        plan.evaluate(zh, out=gh)
    torch.cuda.synchronize()
    ts = []
    for _ in range(200):
        t0 = time.perf_counter()
        plan.evaluate(zh, out=gh)
        ts.append((time.perf_counter() - t0) * 1e6)
    ts.sort()
    print(f"{tag}: mean {sum(ts) / len(ts):.1f} us  p10 {ts[20]:.1f} p50 {ts[100]:.1f} p90 {ts[180]:.1f} max {ts[-1]:.1f}",
          flush=True)


e2e("fresh")
flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
fo = torch.empty(1, dtype=torch.float32, device="cuda")
z = torch.ones(cfg.n, cfg.n, dtype=torch.complex64, device="cuda")
g = torch.empty_like(z)
for _ in range(50):
    torch.amax(flush, dim=0, out=fo[0])
    plan.evaluate_device(z, g, sync_value=False)
torch.cuda.synchronize()
e2e("after flushed loop")
plan.set_timing(True)
for _ in range(50):
    torch.amax(flush, dim=0, out=fo[0])
    plan.evaluate_device(z, g, sync_value=False)
plan.get_timing()
plan.set_timing(False)
torch.cuda.synchronize()
e2e("after timing loop")
del flush
torch.cuda.empty_cache()
e2e("after freeing the flush buffer")
