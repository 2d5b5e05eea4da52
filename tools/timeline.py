"""Per-CTA timeline of the config-2 frame kernel (diagnostic build only).

Build:  tools/build_variant.sh tl "-DABL_TIMELINE"
Run:    PTG_LIB=paper_1810_05628_b200/lib/variants/libptg_tl.so python tools/timeline.py
Stamps (globaltimer ns, thread 0 of each CTA): 0 start, 1 object tile landed,
2 row FFT done (before the spectral operator), 3 all four passes + misfit done,
4 contribution stored.  Prints phase-duration percentiles and the spread of
start / end times across CTAs, relative to the earliest start.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1810_05628_b200 import Plan, synth, _lib  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
obj, probe, pos = synth.make_inputs(cfg)
plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision=cfg.precision)
plan.simulate(obj, copy_out=False)
z = torch.ones(cfg.n, cfg.n, dtype=torch.complex64, device="cuda")
g = torch.empty_like(z)
flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
for _ in range(5):
    plan.evaluate_device(z, g)
torch.cuda.synchronize()
torch.amax(flush)
torch.cuda.synchronize()
plan.evaluate_device(z, g)
torch.cuda.synchronize()
lib = _lib.lib()
buf = np.zeros(8192 * 8, dtype=np.uint64)
lib.ptg_debug_timeline(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
if cfg.M <= 64:
    nb, K = cfg.N, 5
    names = ["start", "obj landed", "rows FFT done", "passes done", "stored"]
else:
    nb, K = min(8192, cfg.N * (cfg.M // 32)), 6
    names = ["start", "gather+sync", "spectral done", "pushes done", "cluster sync", "stored"]
t = buf.reshape(8192, 8)[:nb].astype(np.int64)
t0 = t[:, 0].min()
rel = (t[:, :K] - t0) / 1e3
for k in range(K):
    print(f"{names[k]:14s} min {rel[:, k].min():7.2f}  p50 {np.median(rel[:, k]):7.2f}  max {rel[:, k].max():7.2f} us")
for k in range(1, K):
    d = rel[:, k] - rel[:, k - 1]
    print(f"phase {names[k-1]:>14s} -> {names[k]:14s}: p10 {np.percentile(d, 10):6.2f} p50 {np.median(d):6.2f} p90 {np.percentile(d, 90):6.2f} us")
sm = t[:, 7]
last = {}
for i in range(nb):
    last[sm[i]] = max(last.get(sm[i], 0), rel[i, K - 1])
v = np.array(list(last.values()))
life = rel[:, K - 1] - rel[:, 0]
print(f"CTA lifetime p10 {np.percentile(life, 10):.2f} p50 {np.median(life):.2f} p90 {np.percentile(life, 90):.2f} us")
print(f"per-SM finish: min {v.min():.2f} p50 {np.median(v):.2f} max {v.max():.2f} us over {len(v)} SMs")
