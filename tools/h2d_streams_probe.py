"""H2D of a 4 MiB pinned buffer split over 1 / 2 / 4 concurrent streams (dev tool)."""
import time

import torch

zh = torch.ones(512, 512, dtype=torch.complex128).pin_memory()
zd = torch.empty_like(zh, device="cuda")
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    parts_h = zh.view(-1).chunk(k)
    parts_d = zd.view(-1).chunk(k)

    def go():
        for s, a, b in zip(streams, parts_d, parts_h):
            with torch.cuda.stream(s):
                a.copy_(b, non_blocking=True)
        torch.cuda.synchronize()
    for _ in range(5):
        go()
    t0 = time.perf_counter()
    for _ in range(50):
        go()
    print(f"{k} streams: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us per 4 MiB H2D", flush=True)
