"""Where does the config-2 evaluation step spend its time?

Times the production objective+gradient step (Plan.evaluate_device) under
several cache conditions on one GPU, CUDA events on the launch stream:
  flush   : 512 MiB read between steps (bench.py's timed loop)
  warm    : back-to-back steps, L2 warm
  attr    : per-kernel events (frame kernel / reduce) with flush
Usage: python tools/step_probe.py [--config 2] [--steps 200]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1810_05628_b200 import Plan, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--custom", default="", help="n,M,scan_steps,step: complex64 raster instead of a config")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    if args.custom:
        n, M, ss, st = map(int, args.custom.split(","))
        cfg = synth.Config(0, n, M, ss, st, 8.0, M / 4, 0.0025, "c64")
    obj, probe, pos = synth.make_inputs(cfg)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    plan = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision=cfg.precision)
    plan.set_stream(stream.cuda_stream)
    plan.simulate(obj, copy_out=False)
    cdt = torch.complex64 if cfg.precision == "c64" else torch.complex128
    z = torch.ones(cfg.n, cfg.n, dtype=cdt, device="cuda")
    grad = torch.empty_like(z)
    val = torch.zeros(4, dtype=torch.float64, device="cuda")
    flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
    fo = torch.empty(1, dtype=torch.float32, device="cuda")

    def step():
        plan.evaluate_device(z, grad, value_dev=val, sync_value=False)

    for _ in range(10):
        step()
    torch.cuda.synchronize()

    def loop(do_flush, k=args.steps, per=1):
        s = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        e = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        torch.cuda.synchronize()
        for i in range(k):
            if do_flush:
                torch.amax(flush, dim=0, out=fo[0])
            s[i].record(stream)
            for _ in range(per):
                step()
            e[i].record(stream)
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) * 1e3 / per for a, b in zip(s, e))
        return {"mean_us": sum(t) / len(t), "median_us": t[len(t) // 2], "min_us": t[0]}

    out = {"config": args.custom or args.config}
    out["flush"] = loop(True)
    out["warm_single"] = loop(False)
    out["warm_x20"] = loop(False, k=max(args.steps // 10, 10), per=20)
    plan.set_timing(True)
    plan.get_timing()
    out["attr_flush"] = loop(True)
    fm, fn, gm, gn = plan.get_timing()
    out["attr_flush"].update(frame_us=fm / max(fn, 1) * 1e3, reduce_us=gm / max(gn, 1) * 1e3)
    plan.get_timing()
    out["attr_warm"] = loop(False)
    fm, fn, gm, gn = plan.get_timing()
    out["attr_warm"].update(frame_us=fm / max(fn, 1) * 1e3, reduce_us=gm / max(gn, 1) * 1e3)
    plan.set_timing(False)
    # CUDA-graph replay of 20 steps (launch overhead removed)
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(20):
                step()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(10):
            g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        out["graph_warm_us"] = a.elapsed_time(b) * 1e3 / 200
    except Exception as ex:  # noqa: BLE001
        out["graph_warm_us"] = f"capture failed: {ex}"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
