"""H2D / D2H of a 4 MiB pinned buffer with and without binding the process to
the GPU's NUMA-local CPUs (dev tool)."""
import os
import time

import torch


def bw(tag):
    zh = torch.ones(512, 512, dtype=torch.complex128).pin_memory()
    zd = torch.empty_like(zh, device="cuda")
    for _ in range(5):
        zd.copy_(zh)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        zd.copy_(zh)
    torch.cuda.synchronize()
    h2d = (time.perf_counter() - t0) / 50 * 1e6
    t0 = time.perf_counter()
    for _ in range(50):
        zh.copy_(zd)
    torch.cuda.synchronize()
    d2h = (time.perf_counter() - t0) / 50 * 1e6
    print(f"{tag}: h2d {h2d:.1f} us, d2h {d2h:.1f} us, cpus {len(os.sched_getaffinity(0))}", flush=True)


torch.cuda.init()
bw("default")
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    n = (os.cpu_count() + 63) // 64
    masks = pynvml.nvmlDeviceGetCpuAffinity(h, n)
    cpus = set()
    for w, m in enumerate(masks):
        for b in range(64):
            if m >> b & 1:
                cpus.add(w * 64 + b)
    print("gpu-local cpus", sorted(cpus))
    if cpus:
        os.sched_setaffinity(0, cpus)
        bw("bound")
except Exception as e:
    print("nvml affinity failed:", e)
