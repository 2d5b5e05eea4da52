#!/usr/bin/env python
"""bench.py — batched ptychographic objective+gradient throughput on B200.

Headline workload (BASELINE.json configs[1] = "config 2"): complex64 object
512x512, 64x64 complex probe, 29x29 serpentine raster at step 16 (841
diffraction patterns), noiseless data.  One step = one objective+gradient
evaluation (the reference's evaluate/phiDistance, objectives.cpp:52-118) over
all 841 patterns; metric = diffraction patterns per second.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU), default --scaling weak: band
decomposition of one scanned object — rank r owns the config-2
problem on an n x n band of a tall object whose bands overlap by w - step
rows (the scan continues across bands); each rank evaluates its band, the
shared gradient rows are summed with the neighbours (NCCL point-to-point, the
path's real exchange step) and the misfit with a scalar allreduce.  Per-GPU
work is fixed; value = all ranks' patterns per second.  --scaling strong:
config 2's scan rows split over ranks with the object replicated and the full
gradient allreduced (north_star's baseline layout).

--impl reference: the reference's own CPU path on the host cores (rank 0
only): the patch-model restatement over the reference's compiled OpenMP
kernels::fft2_inplace (oracle/_ref), same config/metric/unit.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

NPROC = os.cpu_count() or 1
os.environ.setdefault("OMP_NUM_THREADS", str(NPROC))

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "diffraction patterns/sec per objective+gradient eval"
UNIT = "patterns/s"
FP32_LANES_PER_SM = 128
N_SM = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-extras", action="store_true", help="skip V-cycle / PIE / CPU legs")
    ap.add_argument("--dist-selftest", action="store_true",
                    help="run the multi-rank (NCCL) code path with one rank (1-GPU check)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="multi-GPU layout: weak = object bands + halo exchange, strong = replicated object + allreduce")
    return ap.parse_args()


def algorithmic(cfg, N):
    """bytes and FLOPs of one objective+gradient evaluation."""
    M, n = cfg.M, cfg.n
    bd, bz = (4, 8) if cfg.precision == "c64" else (8, 16)
    log2 = int(np.log2(M * M)) if M > 1 else 0
    flops = N * (10 * M * M * log2 + 24 * M * M)
    bytes_ = N * M * M * bd + 2 * n * n * bz
    return bytes_, flops


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def load_traffic(key):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.002):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            # NVML numbers GPUs physically; CUDA_VISIBLE_DEVICES renumbers them
            # for CUDA -- look the device up by its PCI bus id
            try:
                import torch
                pr = torch.cuda.get_device_properties(index)
                bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _reasons(self):
        nv = self.nv
        for fn in ("nvmlDeviceGetCurrentClocksEventReasons", "nvmlDeviceGetCurrentClocksThrottleReasons"):
            if hasattr(nv, fn):
                return getattr(nv, fn)(self.h)
        return 0

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                bits = self._reasons()
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "samples": len(s),
                "reasons": sorted(self.reasons - {"gpu_idle"})}


# ------------------------------------------------------------ CPU baseline
def cpu_reference_eval_rate(cfg, obj, probe, pos, data, seconds: float):
    """Reference CPU path: patch-model restatement (oracle/ptgo.c) whose 2-D FFTs
    are the reference's own OpenMP kernels::fft2_inplace (kernels.cpp:126)."""
    from oracle import ptgo
    kind = "port"
    if ptgo.has_reference():
        ptgo.use_reference_fft(True)
        kind = "reference"
    ptgo.set_threads(NPROC)
    cores = NPROC
    p = ptgo.Problem(cfg.n, cfg.M, cfg.w, pos, data.astype(np.float64), probe.astype(np.complex128))
    z = np.ones((cfg.n, cfg.n), np.complex128)
    times = []
    t_end = time.perf_counter() + seconds
    while True:
        t0 = time.perf_counter()
        ptgo.evaluate(p, z)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() >= t_end and len(times) >= 1:
            break
    med = float(np.median(times))
    ptgo.use_reference_fft(False) if kind == "reference" else None
    sample = (f"{len(times)} full objective+gradient evals of {cfg.N} patterns (median {med * 1e3:.1f} ms); "
              + ("patch-model restatement (oracle/ptgo.c) over the reference's compiled "
                 f"kernels::fft2_inplace, scan positions spread over {cores} OpenMP threads "
                 "(results identical to the serial loop)" if kind == "reference" else
                 f"oracle port, pattern-parallel OpenMP ({cores} threads)"))
    return cfg.N / med, cores, kind, sample, med


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from paper_1810_05628_b200 import synth
    from oracle import ptgo
    cfg = synth.CONFIGS[args.config]
    obj, probe, pos = synth.make_inputs(cfg)
    if cfg.precision == "c64":
        obj = obj.astype(np.complex64).astype(np.complex128)
        probe = probe.astype(np.complex64).astype(np.complex128)
    data = ptgo.simulate(cfg.n, cfg.M, cfg.w, pos, obj, probe)
    if cfg.photons:
        data = synth.poisson(data, cfg.photons)
    if cfg.precision == "c64":
        data = data.astype(np.float32).astype(np.float64)
    kind = "port"
    if ptgo.has_reference():
        ptgo.use_reference_fft(True)
        kind = "reference"
    ptgo.set_threads(NPROC)
    cores = NPROC
    p = ptgo.Problem(cfg.n, cfg.M, cfg.w, pos, data, probe)
    z = np.ones((cfg.n, cfg.n), np.complex128)
    for _ in range(max(args.warmup, 0)):
        ptgo.evaluate(p, z)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ptgo.evaluate(p, z)
    dt = time.perf_counter() - t0
    value = cfg.N * args.steps / dt
    sample = (f"{args.steps} full evals x {cfg.N} patterns, "
              + (f"patch-model restatement over the reference's compiled kernels::fft2_inplace, "
                 f"positions over {cores} OpenMP threads" if kind == "reference"
                 else "oracle port, pattern-parallel"))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg.describe(), "global_batch": cfg.N, "parallelism": "cpu"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- ours
def transfer_rooflines(stream):
    """restrictField / prolongField (n = 4096 complex64) and restrictData
    (N = 3721, M = 256 float32): achieved GB/s over SURVEY 8(d)'s algorithmic
    bytes (1.25 * 8 n^2, 1.25 * 8 n^2, 2 N (M/2)^2 4), 10 launches each."""
    import ctypes as C

    import torch

    from paper_1810_05628_b200 import _lib
    lib = _lib.lib()
    peaks, _ = load_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    n, N, M = 4096, 3721, 256
    fine = torch.ones(n, n, dtype=torch.complex64, device="cuda")
    coarse = torch.empty(n // 2, n // 2, dtype=torch.complex64, device="cuda")
    dfine = torch.ones(N, M, M, dtype=torch.float32, device="cuda")
    dcoarse = torch.empty(N, M // 2, M // 2, dtype=torch.float32, device="cuda")
    st = C.c_void_p(stream.cuda_stream)
    ops = {
        "restrict_field": (lambda: lib.ptg_restrict_field_device(0, C.c_void_p(fine.data_ptr()), n,
                                                                  C.c_void_p(coarse.data_ptr()), st),
                           1.25 * 8 * n * n),
        "prolong_field": (lambda: lib.ptg_prolong_field_device(0, C.c_void_p(coarse.data_ptr()), n // 2,
                                                                C.c_void_p(fine.data_ptr()), st),
                          1.25 * 8 * n * n),
        "restrict_data": (lambda: lib.ptg_restrict_data_device(0, C.c_void_p(dfine.data_ptr()), N, M,
                                                                C.c_void_p(dcoarse.data_ptr()), st),
                          2.0 * N * (M // 2) ** 2 * 4),
    }
    out = {}
    for name, (fn, nbytes) in ops.items():
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(10):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 10 * 1e3
        gbs = nbytes / (us * 1e-6) / 1e9
        out[name] = {"us": us, "bytes": nbytes, "achieved_gbs": gbs, "frac_hbm": gbs / hbm}
    return out


def run_ours(args):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    # --dist-selftest: the multi-rank code path (NCCL, band layout, exchange,
    # max-over-ranks timing) with one rank, for checking it on a 1-GPU box
    multi = world > 1 or args.dist_selftest
    if multi:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1810_05628_b200 import Hierarchy, Plan, synth

    from paper_1810_05628_b200 import sharding

    cfg = synth.CONFIGS[args.config]
    obj, probe, pos = synth.make_inputs(cfg)
    banded = multi and args.scaling == "weak"
    overlap = cfg.w - cfg.step if banded else 0
    if banded:
        # rank r: the config's scan on rows [r (n - overlap), + n) of a tall object
        H = world * (cfg.n - overlap) + overlap
        off = sharding.band_offset(rank, cfg.n, overlap)
        big = synth.make_object(H, cfg.sigma_obj)
        obj = np.ascontiguousarray(big[off:off + cfg.n, :cfg.n])
        del big
        pos_shard = pos
    else:
        rows_per = -(-cfg.steps // world)
        lo, hi = min(rank * rows_per, cfg.steps) * cfg.steps, min((rank + 1) * rows_per, cfg.steps) * cfg.steps
        pos_shard = pos[lo:hi]
    Nr = pos_shard.shape[0]

    cdt = torch.complex64 if cfg.precision == "c64" else torch.complex128
    # a real (non-legacy) stream shared by torch and libptg so CUDA events see our kernels
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    plan = Plan(cfg.n, cfg.M, cfg.w, pos_shard, None, probe, precision=cfg.precision, device=local)
    plan.set_stream(stream.cuda_stream)
    # data: our GPU forward operator (forward.cpp:40-54 restated), + Poisson if configured
    host_data = plan.simulate(obj, copy_out=bool(cfg.photons))
    if cfg.photons:
        plan.set_data(synth.poisson(host_data, cfg.photons, seed=4 + rank))
    z = torch.ones(cfg.n, cfg.n, dtype=cdt, device="cuda")
    grad = torch.empty_like(z)
    val = torch.zeros(4, dtype=torch.float64, device="cuda")
    # L2 eviction between timed steps: READ 512 MiB (> 126 MB L2) so no dirty
    # lines are left whose write-back would land inside the timed kernels
    flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
    flush_out = torch.empty(1, dtype=torch.float32, device="cuda")

    halo = sharding.HaloExchange(cfg.n, overlap, cdt, "cuda") if (dist is not None and banded) else None

    def exchange(g, v):
        if dist is None:
            return
        if banded:
            # shared band rows + misfit: pack kernel, ONE all-gather, unpack kernel
            halo(g, v)
            return
        dist.all_reduce(torch.view_as_real(g))
        dist.all_reduce(v[:1])

    def step():
        plan.evaluate_device(z, grad, value_dev=val, sync_value=False)
        exchange(grad, val)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # multi-rank: the evaluation + band exchange (our kernels and the NCCL
    # all-gather) captured once as a CUDA graph and replayed per step -- the
    # eager sequence costs ~20 us of stream hand-offs and host work per step
    step_graph = None
    if dist is not None and banded and os.environ.get("PTG_BENCH_GRAPH", "1") != "0":
        try:
            g_step = torch.cuda.CUDAGraph()
            lc0 = plan.launch_count
            with torch.cuda.graph(g_step, stream=stream):
                plan.set_stream(torch.cuda.current_stream().cuda_stream)
                step()
            plan.set_stream(stream.cuda_stream)
            # our kernels per replay: the plan's (counted while captured) + halo pack/unpack
            graph_launches = plan.launch_count - lc0 + 2
            step_graph = g_step
        except Exception as ex:   # noqa: BLE001
            plan.set_stream(stream.cuda_stream)
            print(f"[bench] step graph capture failed, eager steps: {ex}", file=sys.stderr)
        ok = torch.tensor([1 if step_graph is not None else 0], dtype=torch.int32, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)   # every rank replays, or none does
        if int(ok.item()) == 0:
            step_graph = None
        torch.cuda.synchronize()
    eager_step = step
    if step_graph is not None:
        def step():
            step_graph.replay()
        for _ in range(3):
            step()
        torch.cuda.synchronize()

    def timed_loop():
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            torch.amax(flush, dim=0, out=flush_out[0])   # evict L2 between timed steps (read-only, not timed)
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        return sum(s.elapsed_time(e) for s, e in zip(starts, ends))

    # headline: the production launch sequence (PDL-chained kernels, no probes)
    sampler = ClockSampler(torch.cuda.current_device())
    l0 = plan.launch_count
    sampler.start()
    t_ms = timed_loop()
    clocks = sampler.stop()
    launches = plan.launch_count - l0
    if step_graph is not None:   # replays do not pass through the plan's launch counter
        launches = args.steps * graph_launches
    # attribution: same loop again with per-kernel CUDA events on the launch stream
    step = eager_step   # per-kernel events need the eager launch sequence
    plan.set_timing(True)
    plan.get_timing()
    t_attr_ms = timed_loop()
    frame_ms, frame_n, gather_ms, gather_n = plan.get_timing()
    plan.set_timing(False)
    if dist is not None:
        t = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())

    total_patterns = cfg.N * world if banded else cfg.N
    value = total_patterns * args.steps / (t_ms / 1e3)
    ms_per_step = t_ms / args.steps

    # roofline of the dominant kernel (frame kernel), live CUDA-event durations
    peaks, peak_src = load_peaks()
    B, F = algorithmic(cfg, Nr)
    # per evaluation: a large problem launches the frame kernel once per stash
    # chunk, so the algorithmic work of one evaluation is set against the
    # summed duration of its launches (= per-launch work / per-launch time)
    launches_per_eval = max(frame_n, 1) / max(args.steps, 1)
    avg_frame_s = (frame_ms / max(args.steps, 1)) / 1e3
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved_gbs = B / avg_frame_s / 1e9
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = N_SM * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12
    if cfg.precision == "c128":   # complex128 frames compute in FP64: 64 FP64 lanes per SM on B200
        fp32_peak /= 2
    achieved_tf = F / avg_frame_s / 1e12
    traffic = load_traffic(f"config{cfg.cid}_frame_kernel")
    kname = (f"frame_tma_kernel<{cfg.M}> (TMA-fed register FFT, one CTA per scan position)" if cfg.M <= 64 and cfg.precision == "c64"
             else f"frame_cl_kernel<{cfg.M // 32},32> (cluster of {cfg.M // 32} CTAs per scan position)" if cfg.precision == "c64"
             else f"frame_kernel<double,{cfg.M}> (shared-memory Stockham, one CTA per scan position)")
    roofline_hbm = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved_gbs / hbm_peak, "traffic": traffic,
                    "algorithmic_bytes_per_launch": B / launches_per_eval,
                    "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)"}
    roofline_fp32 = {"bound": "fp32" if cfg.precision == "c64" else "fp64", "achieved": achieved_tf, "peak": fp32_peak,
                     "unit": "TFLOP/s",
                     "frac": achieved_tf / fp32_peak, "algorithmic_flops_per_launch": F / launches_per_eval,
                     "convention": "F(M)=10 M^2 log2(M^2) + 24 M^2 per pattern (SURVEY 8d)",
                     "peak_source": (f"nominal 148 SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz (no measured FP32 figure; "
                                     "tools/fp32_tput.cu measures 116-124 lane-ops/SM/clk for FFMA/FFMA2/FADD2)")
                     if cfg.precision == "c64" else f"nominal 148 SM x 64 FP64 lanes x 2 x {sm_mhz:.0f} MHz"}
    # the headline roofline is the binding one of SURVEY 8(d): attainable time
    # = max(B / BW_HBM, F / P_FP32); the frame kernel is FP32-bound at every
    # configuration (no tensor cores on this path), the HBM view is kept beside it
    binding = roofline_fp32 if F / (fp32_peak * 1e12) >= B / (hbm_peak * 1e9) else roofline_hbm
    roofline = dict(binding)
    roofline.update({"traffic": traffic, "kernel": kname,
                     "avg_launch_us": avg_frame_s * 1e6 / launches_per_eval, "launches_per_eval": launches_per_eval,
                     "attainable_us": max(F / (fp32_peak * 1e12), B / (hbm_peak * 1e9)) * 1e6 / launches_per_eval})
    eval_share = {"frame_kernel_ms": frame_ms / max(args.steps, 1), "gather_ms": gather_ms / max(args.steps, 1),
                  "frame_share_of_step": frame_ms / max(t_attr_ms, 1e-12),
                  "attribution_loop_ms_per_step": t_attr_ms / max(args.steps, 1)}

    # ---- e2e through the public host API: pinned host z in, value + grad out
    e2e = None
    zh = torch.ones(cfg.n, cfg.n, dtype=torch.complex128).pin_memory().numpy()
    gh = torch.empty(cfg.n, cfg.n, dtype=torch.complex128).pin_memory().numpy()
    h2d = zh.nbytes
    d2h = gh.nbytes + 8
    # warm-up: the first call with these buffers runs eagerly, the second
    # captures the replay graph; then ~0.4 s of calls: a fresh process's
    # per-call time falls from ~350 to ~210 us over its first ~500 calls
    # (tools/e2e_warmup_probe.py) as the mostly idle GPU / link ramps up --
    # the steady state is what a solver calling ptg_eval in a loop sees
    if not multi:
        t_w = time.perf_counter()
        nw = 0
        while nw < 10 or time.perf_counter() - t_w < 0.4:
            plan.evaluate(zh, out=gh)
            nw += 1
    e2e_steps = max(args.steps, 100)
    if not multi:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            plan.evaluate(zh, out=gh)
        e2e_s = time.perf_counter() - t0
    else:
        # per rank: pinned complex128 band in (H2D), device conversion, the
        # evaluation and the band exchange, conversion back, pinned complex128
        # gradient out (D2H) and the value read -- the host API's data path
        zt = torch.empty_like(z)
        z128 = torch.empty(cfg.n, cfg.n, dtype=torch.complex128, device="cuda")
        g128 = torch.empty_like(z128)
        zh_t, gh_t = torch.from_numpy(zh), torch.from_numpy(gh)

        def e2e_step():
            z128.copy_(zh_t, non_blocking=True)
            zt.copy_(z128)
            plan.evaluate_device(zt, grad, value_dev=val, sync_value=False)
            exchange(grad, val)
            g128.copy_(grad)
            gh_t.copy_(g128, non_blocking=True)
            float(val[0].item())
        for _ in range(300):   # a fixed count on every rank (collectives inside)
            e2e_step()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        e2e_s = time.perf_counter() - t0
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e = {"value": total_patterns * e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s / e2e_steps * 1e3, "steps": e2e_steps,
           "api": "Plan.evaluate (ptg_eval): pinned complex128 z in, value + complex128 gradient out"}

    extras = {}
    cpu = None
    if rank == 0 and world == 1 and not args.no_extras:
        # PIE sweep (solvers.cpp:229-265), config-2 geometry
        try:
            zp = torch.ones_like(z)
            plan.pie_sweep_device(zp)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(3):
                plan.pie_sweep_device(zp)
            e1.record(stream)
            torch.cuda.synchronize()
            extras["pie_sweep_ms"] = e0.elapsed_time(e1) / 3
        except Exception as ex:   # noqa: BLE001
            extras["pie_sweep_error"] = str(ex)
        # MG/OPT V-cycle on config 3 (3 levels, M=128, jittered raster)
        try:
            c3 = synth.CONFIGS[3]
            o3, p3, s3 = synth.make_inputs(c3)
            plan3 = Plan(c3.n, c3.M, c3.w, s3, None, p3, precision=c3.precision, device=local)
            plan3.set_stream(stream.cuda_stream)
            plan3.simulate(o3, copy_out=False)
            h3 = Hierarchy(plan3, c3.depth)
            z3 = torch.ones(c3.n, c3.n, dtype=torch.complex64, device="cuda")
            g3 = torch.empty_like(z3)
            v3 = plan3.evaluate_device(z3, g3)
            v3, _, _ = h3.cycle_device(z3, g3, v3)   # warm-up cycle
            torch.cuda.synchronize()
            cyc = []
            per = None
            for _ in range(7):   # wall-clock (one host sync per coarse LBFGS iteration): median of 7
                t0 = time.perf_counter()
                v3, wt, per = h3.cycle_device(z3, g3, v3)
                torch.cuda.synchronize()
                cyc.append((time.perf_counter() - t0) * 1e3)
            extras["vcycle"] = {"config": 3, "levels": c3.depth, "ms": float(np.median(cyc)),
                                "weighted_evals_per_cycle": wt, "evals_per_level_per_cycle": per,
                                "value_after": v3}
            h3.close()
            plan3.close()
        except Exception as ex:   # noqa: BLE001
            extras["vcycle_error"] = str(ex)
        # MG/OPT grid transfers (multigrid.cpp:34-77) at config 4's sizes, HBM
        # rooflines with SURVEY 8(d)'s byte counts; inputs > L2, CUDA events
        try:
            extras["transfers"] = transfer_rooflines(stream)
        except Exception as ex:   # noqa: BLE001
            extras["transfers_error"] = str(ex)
        # CPU baseline on a bounded sample of the same workload
        try:
            host_data = plan.simulate(obj, copy_out=True)
            rate, cores, kind, sample, _ = cpu_reference_eval_rate(
                cfg, obj.astype(np.complex64).astype(np.complex128) if cfg.precision == "c64" else obj,
                probe, pos, host_data, args.cpu_seconds)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
        except Exception as ex:   # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": NPROC, "kind": "reference", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak" if banded else "strong", "vs_baseline": None,
                "dtype": "f32" if cfg.precision == "c64" else "f64",
                "data": "synthetic (seeded smooth object, Gaussian x quadratic-phase probe, data by our GPU forward operator)",
                "config": {"workload": cfg.describe() if not banded else
                           (f"{cfg.describe()} per GPU: {world} bands of a {world * (cfg.n - overlap) + overlap}x{cfg.n} "
                            f"object, consecutive bands sharing {overlap} rows (one continuous raster)"),
                           "global_batch": total_patterns, "patterns_per_rank": Nr,
                           "parallelism": (f"object bands x{world}: per evaluation one NCCL all-gather of every rank's "
                                           f"{overlap} halo rows + misfit (pack/unpack kernels)"
                                           if banded else f"scan-row sharding x{world} + NCCL allreduce")
                           if multi else "single GPU",
                           "l2": "flushed between timed steps (512 MiB read)"},
                "roofline": roofline, "roofline_fp32": roofline_fp32, "roofline_hbm": roofline_hbm, "step_breakdown": eval_share,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks}
        line.update(extras)
        print(json.dumps(line), flush=True)
    plan.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
