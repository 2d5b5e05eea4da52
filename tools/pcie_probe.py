"""PCIe probe (dev tool): 1 GiB pinned host <-> device, H2D alone, D2H alone and
both at once (16 chunks alternating over two streams per direction)."""
import time

import torch

N = 1 << 27   # complex128 elements = 2 GiB? no: 2^27 * 8 B = 1 GiB of float64
h_in = torch.empty(N, dtype=torch.float64).pin_memory()
h_out = torch.empty(N, dtype=torch.float64).pin_memory()
d_in = torch.empty(N, dtype=torch.float64, device="cuda")
d_out = torch.empty(N, dtype=torch.float64, device="cuda")
s = [torch.cuda.Stream() for _ in range(4)]
K = 16
c = N // K


def run(h2d, d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        if h2d:
            with torch.cuda.stream(s[k & 1]):
                d_in[k * c:(k + 1) * c].copy_(h_in[k * c:(k + 1) * c], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s[2 + (k & 1)]):
                h_out[k * c:(k + 1) * c].copy_(d_out[k * c:(k + 1) * c], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for name, a, b in (("h2d", 1, 0), ("d2h", 0, 1), ("both", 1, 1)):
    run(a, b)
    ts = [run(a, b) for _ in range(5)]
    t = min(ts)
    gb = (a + b) * N * 8 / 1e9
    print(f"{name}: {t * 1e3:.2f} ms, {gb / t:.1f} GB/s aggregate")
