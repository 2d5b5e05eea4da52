"""One warm MG/OPT V-cycle on config 3 (dev tool: run under ncu for a kernel
time breakdown; prints the wall time of the measured cycles)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_05628_b200 import Hierarchy, Plan, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c3 = synth.CONFIGS[3]
o3, p3, s3 = synth.make_inputs(c3)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
plan3 = Plan(c3.n, c3.M, c3.w, s3, None, p3, precision=c3.precision)
plan3.set_stream(stream.cuda_stream)
plan3.simulate(o3, copy_out=False)
h3 = Hierarchy(plan3, c3.depth)
z3 = torch.ones(c3.n, c3.n, dtype=torch.complex64, device="cuda")
g3 = torch.empty_like(z3)
v3 = plan3.evaluate_device(z3, g3)
v3, _, _ = h3.cycle_device(z3, g3, v3)
torch.cuda.synchronize()
for _ in range(reps):
    t0 = time.perf_counter()
    v3, wt, per = h3.cycle_device(z3, g3, v3)
    torch.cuda.synchronize()
    print(f"cycle {1e3 * (time.perf_counter() - t0):.2f} ms evals {per} value {v3}")
