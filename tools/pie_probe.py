"""PIE sweep time on config 2 (dev tool): python tools/pie_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1810_05628_b200 import Plan, synth  # noqa: E402

cfg = synth.CONFIGS[2]
obj, probe, pos = synth.make_inputs(cfg)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision="c64")
plan.set_stream(stream.cuda_stream)
plan.simulate(obj, copy_out=False)
z = torch.ones(cfg.n, cfg.n, dtype=torch.complex64, device="cuda")
plan.pie_sweep_device(z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(5):
    plan.pie_sweep_device(z)
e1.record(stream)
torch.cuda.synchronize()
print(f"PIE sweep {e0.elapsed_time(e1) / 5:.3f} ms ({e0.elapsed_time(e1) / 5 / cfg.N * 1e3:.2f} us per position)")
