"""Per-level objective+gradient time of a config's MG/OPT hierarchy (dev tool):
python tools/level_probe.py [config]   (PTG_RMW / PTG_NO_RMW select the overlap-add)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1810_05628_b200 import Hierarchy, Plan, synth  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
obj, probe, pos = synth.make_inputs(cfg)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision=cfg.precision)
plan.set_stream(stream.cuda_stream)   # the plan's kernels on the stream the events see
plan.simulate(obj, copy_out=False)
if cfg.photons:
    plan.add_poisson(cfg.photons, seed=4)
h = Hierarchy(plan, cfg.depth)
for l in range(cfg.depth):
    pl = h.level(l)
    pl.set_stream(stream.cuda_stream)
    z = torch.ones(pl.n, pl.n, dtype=torch.complex64, device="cuda")
    g = torch.empty_like(z)
    for _ in range(3):
        pl.evaluate_device(z, g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        pl.evaluate_device(z, g, sync_value=False)
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"level {l}: n={pl.n} M={pl.M} N={pl.N}: {e0.elapsed_time(e1) / 10:.3f} ms per evaluation", flush=True)
