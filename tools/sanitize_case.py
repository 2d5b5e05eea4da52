"""Smallest cases of the hand-rolled mbarrier / TMA / st.async / DSMEM kernels,
for compute-sanitizer (dev tool; one tool per run):
    compute-sanitizer --tool memcheck  python tools/sanitize_case.py
    compute-sanitizer --tool racecheck python tools/sanitize_case.py
frame_tma_kernel<64> (TMA tensor loads + mbarriers), frame_cl_kernel<4,32>
(cluster DSMEM, st.async gather, split cluster barriers), frame_rmw_kernel<8,32>
(persistent, dependency flags, read-modify-write), each checked against the
CPU oracle so a silent corruption also fails."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ptgo  # noqa: E402
from paper_1810_05628_b200 import Plan, synth  # noqa: E402


def case(M, steps, step, env):
    for k, v in env.items():
        os.environ[k] = v
    n = (steps - 1) * step + M + 4
    cfg = synth.Config(0, n, M, steps, step, 5.0, M / 4, 0.002, "c64", jitter=1)
    obj, probe, pos = synth.make_inputs(cfg)
    probe = probe.astype(np.complex64).astype(np.complex128)
    obj = obj.astype(np.complex64).astype(np.complex128)
    data = ptgo.simulate(n, M, M, pos, obj, probe).astype(np.float32)
    z = (obj * 0.9).astype(np.complex64).astype(np.complex128)
    plan = Plan(n, M, M, pos, data, probe, precision="c64")
    gv, gg = plan.evaluate(z)
    wv, wg = ptgo.evaluate(ptgo.Problem(n, M, M, pos, data.astype(np.float64), probe), z)
    rv, rg = abs(gv - wv) / abs(wv), np.linalg.norm(gg - wg) / np.linalg.norm(wg)
    print(f"M={M} N={len(pos)} env={env}: value rel {rv:.2e}, grad rel L2 {rg:.2e}", flush=True)
    assert rv <= 1e-5 and rg <= 1e-4
    plan.close()
    for k in env:
        os.environ.pop(k)


if __name__ == "__main__":
    case(64, 3, 24, {})                           # frame_tma_kernel<64> + plane reduce
    case(128, 3, 40, {})                          # frame_cl_kernel<4,32> (planes)
    case(256, 3, 64, {"PTG_NO_PLANES": "1"})      # frame_rmw_kernel<8,32>
    print("sanitize cases ok")
