import sys, time, os
import torch
sys.path.insert(0, ".")
from paper_1810_05628_b200 import Plan, synth
mode = sys.argv[1]
cfg = synth.CONFIGS[2]
obj, probe, pos = synth.make_inputs(cfg)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision="c64")
plan.set_stream(stream.cuda_stream)
plan.simulate(obj, copy_out=False)
z = torch.ones(cfg.n, cfg.n, dtype=torch.complex64, device="cuda"); g = torch.empty_like(z)
val = torch.zeros(4, dtype=torch.float64, device="cuda")
if "nvml" in mode:
    import pynvml; pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
    for _ in range(100): pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
for _ in range(50):
    if "valdev" in mode: plan.evaluate_device(z, g, value_dev=val, sync_value=False)
    else: plan.evaluate_device(z, g, sync_value=False)
torch.cuda.synchronize()
if "timing" in mode:
    plan.set_timing(True)
    for _ in range(50): plan.evaluate_device(z, g, value_dev=val, sync_value=False)
    plan.get_timing(); plan.set_timing(False)
    torch.cuda.synchronize()
zh = torch.ones(cfg.n, cfg.n, dtype=torch.complex128).pin_memory().numpy()
gh = torch.empty(cfg.n, cfg.n, dtype=torch.complex128).pin_memory().numpy()
for _ in range(10): plan.evaluate(zh, out=gh)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100): plan.evaluate(zh, out=gh)
print(mode, f"{(time.perf_counter() - t0) / 100 * 1e6:.1f} us")
