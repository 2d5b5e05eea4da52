"""Per-frame phase timeline of the persistent RMW kernel (diagnostic build only).

Build:  tools/build_variant.sh tl "-DABL_TIMELINE"
Run:    PTG_LIB=paper_1810_05628_b200/lib/variants/libptg_tl.so python tools/rmw_timeline.py [config]
Stamps (globaltimer ns, thread 0 of the first 64 CTAs, first 128 frames each):
0 loop top, 1 item known (after the full cluster barrier), 2 gather issued,
3 gather landed (mbarrier), 4 row FFT done (pass 1, before the spectral op),
5 spectral op done, 6 row DIT combine done, 7 inverse column pushes issued,
8 after the cluster barrier (pushes landed), 9 contributions formed,
10 dependencies acquired, 11 gradient updated + released.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1810_05628_b200 import Plan, synth, _lib  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
obj, probe, pos = synth.make_inputs(cfg)
plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision=cfg.precision)
plan.simulate(obj, copy_out=False)
z = torch.ones(cfg.n, cfg.n, dtype=torch.complex64, device="cuda")
g = torch.empty_like(z)
for _ in range(3):
    plan.evaluate_device(z, g)
torch.cuda.synchronize()
C, F, S = 64, 128, 12
buf = np.zeros(C * F * S, np.uint64)
L = _lib.lib()
L.ptg_debug_rmw_timeline.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.ptg_debug_rmw_timeline(buf.ctypes.data, buf.nbytes) == 0
t = buf.reshape(C, F, S).astype(np.int64)
ok = (t > 0).all(axis=2)
d = np.diff(t, axis=2)[ok]          # [frames, 11] phase durations (ns)
names = ["barrier/item", "gather issue", "gather land", "pass0+rowDIF+rowFFT", "spectral", "rowDIT",
         "colFFT+push", "cluster sync", "contrib", "deps", "RMW+release"]
tot = np.diff(t[:, :, [0, 11]], axis=2)[ok][:, 0]
print(f"{ok.sum()} frames sampled; frame time median {np.median(tot) / 1e3:.2f} us "
      f"(p10 {np.percentile(tot, 10) / 1e3:.2f}, p90 {np.percentile(tot, 90) / 1e3:.2f})")
for i, nm in enumerate(names):
    col = d[:, i]
    print(f"  {nm:22s} median {np.median(col) / 1e3:7.2f} us  p90 {np.percentile(col, 90) / 1e3:7.2f} us  "
          f"share {np.median(col) / np.median(tot) * 100:5.1f} %")
# loop-top to the previous frame's end: the gap between frames
gap = (t[:, 1:, 0] - t[:, :-1, 11])[ok[:, 1:] & ok[:, :-1]]
print(f"  inter-frame gap median {np.median(gap) / 1e3:.2f} us")
