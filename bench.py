#!/usr/bin/env python
"""bench.py — batched ptychographic objective+gradient throughput on B200.

Headline workload (BASELINE.json configs[4] = "config 5", the largest
single-GPU configuration): complex64 object 8192x8192, 256x256 Gaussian x
quadratic-phase probe, 166x166 serpentine raster at step 48 (27,556
diffraction patterns, 7.2 GB of fp32 intensities) with Poisson noise at 1e5
photons per pattern.  One step = one objective+gradient evaluation (the
reference's evaluate/phiDistance, objectives.cpp:52-118) over all patterns;
metric = diffraction patterns per second.  `--config K` selects another
BASELINE configuration (1..5).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU), --scaling strong (default): the
config's scan rows are split into contiguous blocks over the ranks with the
object replicated (north_star's layout); each rank evaluates its
rows and the partial gradients + misfits are summed by ONE NCCL allreduce
issued from inside libptg (a communicator bound to the plan with
ptg_plan_bind_comm).  value = all N patterns per max-over-ranks evaluation
time.  --scaling weak: rank r owns a band of a taller object with its own copy
of the config's scan (band decomposition, halo rows exchanged), per-GPU work
fixed.

--impl reference: the reference's own CPU path on the host cores (rank 0
only): the patch-model restatement over the reference's compiled OpenMP
kernels::fft2_inplace (oracle/_ref), same metric/unit, on a bounded sample of
the same workload (configs 4-5: the config's probe / step / noise on the
top-left 2048 x 2048 object window -- config 5: 38 x 38 = 1,444 patterns).
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
N_SM = 148
CPU_SAMPLE_SIDE = 2048   # object side of the bounded CPU sample for configs 4-5


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-extras", action="store_true", help="skip other configs / V-cycle / PIE / CPU legs")
    ap.add_argument("--dist-selftest", action="store_true",
                    help="run the multi-rank (NCCL) code path with one rank (1-GPU check)")
    ap.add_argument("--layout", default=None, choices=["bands", "replicated"],
                    help="strong-scaling layout (default: bands for complex64 M >= 128, else replicated)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="multi-GPU layout: strong = scan rows split, object replicated, gradient allreduce; "
                         "weak = object bands + halo exchange")
    return ap.parse_args()


def algorithmic(cfg, N, n=None):
    """bytes and FLOPs of one objective+gradient evaluation."""
    M = cfg.M
    n = cfg.n if n is None else n
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


def load_profile(key):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def fp32_peak_tflops(sm_mhz):
    """FP32 peak: the measured FMA-pipe rate (profiles/traffic.json "fp32_peak",
    tools/fp32_tput.cu on a B200: lane-FMAs per SM per clock) x 2 flops x 148
    SMs x clock; the nominal 128 lanes when absent."""
    prof = load_profile("fp32_peak") or {}
    lanes = prof.get("lane_fma_per_sm_clk")
    if lanes:
        return N_SM * lanes * 2 * sm_mhz * 1e6 / 1e12, (
            f"measured: {lanes:.1f} FP32 lane-FMAs/SM/clk ({prof.get('source', 'tools/fp32_tput.cu')}) "
            f"x 2 x 148 SM x {sm_mhz:.0f} MHz")
    return N_SM * 128 * 2 * sm_mhz * 1e6 / 1e12, f"nominal 148 SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz"


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
def cpu_sample_problem(cfg, obj):
    """The bounded CPU sample of a configuration: the full problem up to n =
    2048, else the config's probe / step / noise on the top-left 2048 x 2048
    window of its object with the raster that fits it (config 5: 38 x 38 =
    1,444 patterns; config 4: 29 x 29 = 841)."""
    from paper_1810_05628_b200 import synth
    if cfg.n <= CPU_SAMPLE_SIDE:
        return cfg.n, obj, synth.raster(cfg.n, cfg.w, cfg.steps, cfg.step, cfg.jitter), "full problem"
    S = CPU_SAMPLE_SIDE
    steps = (S - cfg.w) // cfg.step + 1
    pos = synth.raster(S, cfg.w, steps, cfg.step, cfg.jitter)
    return S, np.ascontiguousarray(obj[:S, :S]), pos, (f"the config's probe/step/noise on the top-left {S}x{S} "
                                                       f"object window, {steps}x{steps} raster ({steps * steps} "
                                                       "patterns)")


def cpu_problem(cfg, obj, probe):
    """(ptgo.Problem, n, sample description): oracle-simulated (+ Poisson,
    the GPU's sampler restated) data of the CPU sample, fp32-rounded in c64."""
    from oracle import ptgo
    n, o, pos, desc = cpu_sample_problem(cfg, obj)
    if cfg.precision == "c64":
        o = o.astype(np.complex64).astype(np.complex128)
        probe = probe.astype(np.complex64).astype(np.complex128)
    data = ptgo.simulate(n, cfg.M, cfg.w, pos, o, probe)
    if cfg.photons:
        data = ptgo.add_poisson(data, cfg.photons, seed=4)
    if cfg.precision == "c64":
        data = data.astype(np.float32).astype(np.float64)
    return ptgo.Problem(n, cfg.M, cfg.w, pos, data, probe), n, desc


def cpu_reference_on():
    """Route the oracle's 2-D FFTs through the reference's compiled
    kernels::fft2_inplace (kernels.cpp:126) when oracle/_ref has it."""
    from oracle import ptgo
    ptgo.set_threads(NPROC)
    if ptgo.has_reference():
        ptgo.use_reference_fft(True)
        return "reference"
    return "port"


def _how(kind):
    return ("patch-model restatement (oracle/ptgo.c) over the reference's compiled kernels::fft2_inplace, "
            f"scan positions over {NPROC} OpenMP threads (results identical to the serial loop)"
            if kind == "reference" else f"oracle port, pattern-parallel OpenMP ({NPROC} threads)")


def cpu_eval_rate(cfg, obj, probe, seconds: float, min_evals: int = 3):
    from oracle import ptgo
    kind = cpu_reference_on()
    p, n, desc = cpu_problem(cfg, obj, probe)
    z = np.ones((n, n), np.complex128)
    ptgo.evaluate(p, z)   # warm
    times = []
    t_end = time.perf_counter() + seconds
    while len(times) < min_evals or time.perf_counter() < t_end:
        t0 = time.perf_counter()
        ptgo.evaluate(p, z)
        times.append(time.perf_counter() - t0)
    med = float(np.median(times))
    sample = f"{len(times)} objective+gradient evals (median {med * 1e3:.1f} ms) of {p.N} patterns, {desc}; {_how(kind)}"
    return {"value": p.N / med, "unit": UNIT, "cores": NPROC, "kind": kind, "sample": sample,
            "ms_per_eval": med * 1e3, "patterns": p.N}


def cpu_one_thread_rate(cfg, obj, probe):
    """The same CPU sample on ONE thread (nproc and 1 thread)."""
    from oracle import ptgo
    kind = cpu_reference_on()
    ptgo.set_threads(1)
    try:
        p, n, desc = cpu_problem(cfg, obj, probe)
        z = np.ones((n, n), np.complex128)
        t0 = time.perf_counter()
        ptgo.evaluate(p, z)
        dt = time.perf_counter() - t0
    finally:
        ptgo.set_threads(NPROC)
    return {"value": p.N / dt, "unit": UNIT, "cores": 1, "kind": kind, "ms_per_eval": dt * 1e3,
            "sample": f"1 objective+gradient eval of {p.N} patterns on one thread, {desc}"}


def cpu_pie_sweep_ms(cfg, obj, probe):
    """PIE (solvers.cpp:229-265) on the host, ms per sweep: (t(3 sweeps) -
    t(1 sweep)) / 2 minus one evaluation (the uncounted diagnostic
    evaluation each sweep is followed by), i.e. the sweep the GPU's
    pie_sweep_device times."""
    from oracle import ptgo
    kind = cpu_reference_on()
    p, n, desc = cpu_problem(cfg, obj, probe)
    z = np.ones((n, n), np.complex128)
    t1 = time.perf_counter()
    ptgo.pie(p, z, 0.0, 1)
    t2 = time.perf_counter()
    ptgo.pie(p, z, 0.0, 3)
    t3 = time.perf_counter()
    ptgo.evaluate(p, z)
    t4 = time.perf_counter()
    per = ((t3 - t2) - (t2 - t1)) / 2 - (t4 - t3)
    return {"ms": per * 1e3, "cores": NPROC, "kind": kind,
            "sample": f"(pie 3 sweeps - pie 1 sweep) / 2 - one evaluation, {desc}; {_how(kind)}"}


def cpu_vcycle_ms(cfg, obj, probe, cycles: int = 2):
    """One top-level mgoptCycle (multigrid.cpp:207-222) on the host (oracle hierarchy)."""
    from oracle import ptgo
    kind = cpu_reference_on()
    p, n, desc = cpu_problem(cfg, obj, probe)
    h = ptgo.Hierarchy(p, cfg.depth)
    z = np.ones((n, n), np.complex128)
    v0 = np.zeros_like(z)
    val, g = ptgo.evaluate(p, z)
    t = []
    for _ in range(cycles):
        t0 = time.perf_counter()
        z, val, g, _ = h.cycle(0, z, v0, warm=(val, g))
        t.append(time.perf_counter() - t0)
    out = {"ms": float(np.median(t)) * 1e3, "cores": NPROC, "kind": kind, "levels": cfg.depth, "patterns": p.N,
           "sample": f"median of {cycles} cycle(s) after the x0 = 1 evaluation, {desc}; {_how(kind)}"}
    if p.N < cfg.N:   # bounded sample: the work of a cycle is linear in the pattern count
        out["scaled_to_full_ms"] = out["ms"] * cfg.N / p.N
        out["scaling_note"] = (f"the sample has {p.N} of the workload's {cfg.N} patterns (same probe, step, noise, "
                               "levels); scaled_to_full_ms = ms x N / N_sample")
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from paper_1810_05628_b200 import synth
    from oracle import ptgo
    cfg = synth.CONFIGS[args.config]
    obj, probe, _ = synth.make_inputs(cfg)
    kind = cpu_reference_on()
    p, n, desc = cpu_problem(cfg, obj, probe)
    z = np.ones((n, n), np.complex128)
    for _ in range(max(args.warmup, 0)):
        ptgo.evaluate(p, z)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ptgo.evaluate(p, z)
    dt = time.perf_counter() - t0
    value = p.N * args.steps / dt
    sample = f"{args.steps} objective+gradient evals x {p.N} patterns, {desc}; {_how(kind)}"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg.describe(), "global_batch": cfg.N, "parallelism": "cpu",
                       "cpu_sample": desc, "cpu_sample_patterns": p.N},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": NPROC, "kind": kind, "sample": sample},
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
    del fine, coarse, dfine, dcoarse
    return out


class GpuProblem:
    """A configuration resident on this GPU: plan, device data (our forward
    operator + device Poisson noise), iterate / gradient buffers."""

    def __init__(self, cfg, obj, probe, pos, stream, device, plan=None):
        import torch

        from paper_1810_05628_b200 import Plan
        self.cfg = cfg
        self.stream = stream
        self.cdt = torch.complex64 if cfg.precision == "c64" else torch.complex128
        self.plan = plan if plan is not None else Plan(cfg.n, cfg.M, cfg.w, pos, None, probe,
                                                       precision=cfg.precision, device=device)
        self.plan.set_stream(stream.cuda_stream)
        # data: our GPU forward operator (forward.cpp:40-54 restated) + device
        # Poisson noise; `obj` holds the plan's object rows
        self.plan.simulate(obj, copy_out=False)
        if cfg.photons:
            self.plan.add_poisson(cfg.photons, seed=4)
        self.bands = getattr(self.plan, "shard", {}).get("rows", cfg.n) != cfg.n
        self.z = torch.ones(self.plan.rows, cfg.n, dtype=self.cdt, device="cuda")
        self.grad = torch.empty_like(self.z)
        self.val = torch.zeros(4, dtype=torch.float64, device="cuda")

    def step(self):
        if self.bands:
            self.plan.sync_halo(self.z)   # the iterate's halo rows from the next rank (NCCL)
        self.plan.evaluate_device(self.z, self.grad, value_dev=self.val, sync_value=False)

    def close(self):
        self.plan.close()


def timed_loop(step, stream, steps, flush, flush_out, dist=None):
    import torch
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        torch.amax(flush, dim=0, out=flush_out[0])   # evict L2 between timed steps (read-only, not timed)
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    return sum(s.elapsed_time(e) for s, e in zip(starts, ends))


def roofline_for(cfg, N, frame_ms, frame_n, steps):
    """Roofline of the dominant kernel (frame kernel): SURVEY 8(d)'s
    algorithmic work per evaluation over its live CUDA-event duration."""
    peaks, peak_src = load_peaks()
    B, F = algorithmic(cfg, N)
    launches_per_eval = max(frame_n, 1) / max(steps, 1)
    avg_frame_s = (frame_ms / max(steps, 1)) / 1e3
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved_gbs = B / avg_frame_s / 1e9
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak, fp32_src = fp32_peak_tflops(sm_mhz)
    if cfg.precision == "c128":   # complex128 frames compute in FP64: 64 FP64 lanes per SM on B200
        fp32_peak, fp32_src = N_SM * 64 * 2 * sm_mhz * 1e6 / 1e12, f"nominal 148 SM x 64 FP64 lanes x 2 x {sm_mhz:.0f} MHz"
    achieved_tf = F / avg_frame_s / 1e12
    prof = load_profile(f"config{cfg.cid}_frame_kernel")
    traffic = prof.get("dram_bytes_per_launch") if isinstance(prof, dict) else prof
    if cfg.M <= 64 and cfg.precision == "c64":
        kname = f"frame_tma_kernel<{cfg.M}> (TMA-fed register FFT, one CTA per scan position)"
    elif cfg.precision == "c64" and cfg.M == 256 and N >= 2000:
        kname = ("frame_rmw_kernel<8,32> (persistent clusters of 8 CTAs, one scan position per cluster at a time, "
                 "dependency-ordered in-place overlap-add, probe rows + next object window in tensor memory)")
    elif cfg.precision == "c64":
        kname = f"frame_cl_kernel<{cfg.M // 32},32> (cluster of {cfg.M // 32} CTAs per scan position)"
    else:
        kname = f"frame_kernel<double,{cfg.M}> (shared-memory Stockham, one CTA per scan position)"
    roofline_hbm = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved_gbs / hbm_peak, "traffic": traffic,
                    "algorithmic_bytes_per_launch": B / launches_per_eval,
                    "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)"}
    roofline_fp32 = {"bound": "fp32" if cfg.precision == "c64" else "fp64", "achieved": achieved_tf,
                     "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved_tf / fp32_peak,
                     "algorithmic_flops_per_launch": F / launches_per_eval,
                     "convention": "F(M)=10 M^2 log2(M^2) + 24 M^2 per pattern (SURVEY 8d)",
                     "peak_source": fp32_src}
    binding = roofline_fp32 if F / (fp32_peak * 1e12) >= B / (hbm_peak * 1e9) else roofline_hbm
    roofline = dict(binding)
    roofline.update({"traffic": traffic, "kernel": kname,
                     "avg_launch_us": avg_frame_s * 1e6 / launches_per_eval, "launches_per_eval": launches_per_eval,
                     "attainable_us": max(F / (fp32_peak * 1e12), B / (hbm_peak * 1e9)) * 1e6 / launches_per_eval})
    if isinstance(prof, dict) and prof.get("source"):
        roofline["traffic_source"] = prof["source"]
    return roofline, roofline_fp32, roofline_hbm


def gpu_config_rate(cfg, stream, steps, flush, flush_out):
    """Device-timed patterns/s of one configuration (extras)."""
    from paper_1810_05628_b200 import synth
    obj, probe, pos = synth.make_inputs(cfg)
    gp = GpuProblem(cfg, obj, probe, pos, stream, 0)
    for _ in range(3):
        gp.step()
    t = timed_loop(gp.step, stream, steps, flush, flush_out)
    gp.plan.set_timing(True)
    gp.plan.get_timing()
    timed_loop(gp.step, stream, steps, flush, flush_out)
    fm, fn, _, _ = gp.plan.get_timing()
    gp.plan.set_timing(False)
    gp.close()
    roof, _, _ = roofline_for(cfg, cfg.N, fm, fn, steps)
    return {"workload": cfg.describe(), "value": cfg.N * steps / (t / 1e3), "ms_per_eval": t / steps,
            "frame_kernel_ms": fm / steps, "roofline_frac": roof["frac"], "roofline_bound": roof["bound"]}, (obj, probe)


def gpu_vcycle(cfg, stream, cycles=5):
    """MG/OPT V-cycle (one top-level mgoptCycle, multigrid.cpp:207-222) on the GPU, ms."""
    import torch

    from paper_1810_05628_b200 import Hierarchy, synth
    obj, probe, pos = synth.make_inputs(cfg)
    gp = GpuProblem(cfg, obj, probe, pos, stream, 0)
    h = Hierarchy(gp.plan, cfg.depth)
    z, g = gp.z, gp.grad
    v = gp.plan.evaluate_device(z, g)
    v, _, _ = h.cycle_device(z, g, v)   # warm-up cycle
    torch.cuda.synchronize()
    cyc, per, wt = [], None, None
    for _ in range(cycles):   # wall clock (host decisions inside the cycle): median
        t0 = time.perf_counter()
        v, wt, per = h.cycle_device(z, g, v)
        torch.cuda.synchronize()
        cyc.append((time.perf_counter() - t0) * 1e3)
    h.close()
    gp.close()
    return {"config": cfg.cid, "levels": cfg.depth, "ms": float(np.median(cyc)), "cycles_timed": cycles,
            "weighted_evals_per_cycle": wt, "evals_per_level_per_cycle": per, "value_after": v}, (obj, probe)


def run_ours(args):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    multi = world > 1 or args.dist_selftest
    if multi:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1810_05628_b200 import sharding, synth

    from paper_1810_05628_b200 import Comm, Plan

    cfg = synth.CONFIGS[args.config]
    obj, probe, pos = synth.make_inputs(cfg)
    banded = multi and args.scaling == "weak"
    overlap = cfg.w - cfg.step if banded else 0
    comm = None
    splan = None
    layout = args.layout or ("bands" if (cfg.precision == "c64" and cfg.M >= 128) else "replicated")
    if banded:
        # rank r: the config's scan on rows [r (n - overlap), + n) of a tall object
        H = world * (cfg.n - overlap) + overlap
        off = sharding.band_offset(rank, cfg.n, overlap)
        big = synth.make_object(H, cfg.sigma_obj)
        obj = np.ascontiguousarray(big[off:off + cfg.n, :cfg.n])
        del big
        Nr = cfg.N
    elif multi:
        # strong scaling of ONE problem: this rank's share (libptg's partition)
        # and libptg's own NCCL communicator -- every evaluation ends with the
        # library's exchange (BANDS: halo rows send/recv + scalar allreduce;
        # REPLICATED: allreduce of gradient + value)
        def bcast(a):
            t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
            dist.broadcast(t, 0)
            return t.cpu().numpy()
        comm = Comm(world, rank, local, bcast)
        splan = Plan.sharded(cfg.n, cfg.M, cfg.w, pos, world, rank, layout, probe=probe,
                             precision=cfg.precision, device=local)
        splan.bind_comm(comm)
        r0, rows = splan.shard["row0"], splan.rows
        obj = np.ascontiguousarray(obj[r0:r0 + rows])
        Nr = splan.N
    else:
        Nr = cfg.N

    # a real (non-legacy) stream shared by torch and libptg so CUDA events see our kernels
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    gp = GpuProblem(cfg, obj, probe, pos, stream, local, plan=splan)
    plan = gp.plan
    # L2 eviction between timed steps: READ 512 MiB (> 126 MB L2) so no dirty
    # lines are left whose write-back would land inside the timed kernels
    flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
    flush_out = torch.empty(1, dtype=torch.float32, device="cuda")
    halo = sharding.HaloExchange(cfg.n, overlap, gp.cdt, "cuda") if (dist is not None and banded) else None

    def step():
        gp.step()
        if halo is not None:
            halo(gp.grad, gp.val)   # shared band rows + misfit: pack kernel, ONE all-gather, unpack kernel

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(torch.cuda.current_device())
    l0 = plan.launch_count
    sampler.start()
    t_ms = timed_loop(step, stream, args.steps, flush, flush_out, dist)
    clocks = sampler.stop()
    launches = plan.launch_count - l0 + (2 * args.steps if halo is not None else 0)
    # attribution: same loop again with per-kernel CUDA events on the launch stream
    plan.set_timing(True)
    plan.get_timing()
    t_attr_ms = timed_loop(step, stream, args.steps, flush, flush_out, dist)
    frame_ms, frame_n, gather_ms, gather_n = plan.get_timing()
    plan.set_timing(False)
    if dist is not None:
        t = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())

    total_patterns = cfg.N * world if banded else cfg.N
    value = total_patterns * args.steps / (t_ms / 1e3)
    ms_per_step = t_ms / args.steps
    roofline, roofline_fp32, roofline_hbm = roofline_for(cfg, Nr, frame_ms, frame_n, args.steps)
    eval_share = {"frame_kernel_ms": frame_ms / max(args.steps, 1), "overlap_add_ms": gather_ms / max(args.steps, 1),
                  "frame_share_of_step": frame_ms / max(t_attr_ms, 1e-12),
                  "attribution_loop_ms_per_step": t_attr_ms / max(args.steps, 1)}

    # ---- e2e through the public host API: pinned host z in, value + grad out
    zh = torch.ones(plan.rows, cfg.n, dtype=torch.complex128).pin_memory().numpy()
    gh = torch.empty(plan.rows, cfg.n, dtype=torch.complex128).pin_memory().numpy()
    h2d, d2h = zh.nbytes, gh.nbytes + 8
    e2e_steps = max(args.steps, 100 if cfg.n <= 1024 else 10)
    if not multi:
        # warm-up: a fresh process's per-call time falls over its first calls
        # as the mostly idle GPU / link ramps up (tools/e2e_warmup_probe.py)
        t_w, nw = time.perf_counter(), 0
        while nw < 3 or time.perf_counter() - t_w < 0.4:
            plan.evaluate(zh, out=gh)
            nw += 1
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            plan.evaluate(zh, out=gh)
        e2e_s = time.perf_counter() - t0
    elif comm is not None:
        # the host API on every rank: its object rows in, the global value and
        # its gradient rows out (libptg's exchange inside ptg_eval)
        def e2e_step():
            plan.evaluate(zh, out=gh)
        for _ in range(3):   # a fixed count on every rank (collectives inside)
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
    else:
        z128 = torch.empty(cfg.n, cfg.n, dtype=torch.complex128, device="cuda")
        g128 = torch.empty_like(z128)
        zh_t, gh_t = torch.from_numpy(zh), torch.from_numpy(gh)

        def e2e_step():
            z128.copy_(zh_t, non_blocking=True)
            gp.z.copy_(z128)
            step()
            g128.copy_(gp.grad)
            gh_t.copy_(g128, non_blocking=True)
            float(gp.val[0].item())
        for _ in range(5):   # a fixed count on every rank (collectives inside)
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
    del zh, gh
    gp.close()
    torch.cuda.empty_cache()

    extras = {}
    cpu = None
    if rank == 0 and world == 1 and not args.no_extras:
        # CPU baseline on a bounded sample of the same workload
        try:
            cpu = cpu_eval_rate(cfg, obj, probe, args.cpu_seconds)
            cpu["one_thread"] = cpu_one_thread_rate(cfg, obj, probe)
        except Exception as ex:   # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": NPROC, "kind": "reference", "sample": f"failed: {ex}"}
        # the other BASELINE configurations, each beside its CPU reference rate
        others = {}
        for cid in (2, 3, 4, 5):
            if cid == cfg.cid:
                continue
            try:
                c = synth.CONFIGS[cid]
                r, (o, pr) = gpu_config_rate(c, stream, 10, flush, flush_out)
                r["cpu_baseline"] = cpu_eval_rate(c, o, pr, 3.0)
                others[f"config{cid}"] = r
            except Exception as ex:   # noqa: BLE001
                others[f"config{cid}"] = {"error": str(ex)}
            torch.cuda.empty_cache()
        extras["configs"] = others
        # PIE sweep (solvers.cpp:229-265), config-2 geometry, GPU + CPU
        try:
            c2 = synth.CONFIGS[2]
            o2, p2, s2 = synth.make_inputs(c2)
            g2 = GpuProblem(c2, o2, p2, s2, stream, 0)
            zp = torch.ones_like(g2.z)
            g2.plan.pie_sweep_device(zp)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(3):
                g2.plan.pie_sweep_device(zp)
            e1.record(stream)
            torch.cuda.synchronize()
            g2.close()
            extras["pie_sweep"] = {"config": 2, "ms": e0.elapsed_time(e1) / 3,
                                   "cpu_baseline": cpu_pie_sweep_ms(c2, o2, p2)}
        except Exception as ex:   # noqa: BLE001
            extras["pie_sweep_error"] = str(ex)
        # MG/OPT V-cycles: config 3 (3 levels, GPU + CPU) and config 5 (4 levels, GPU)
        vc = {}
        for cid in (3, 5):
            try:
                r, (o, pr) = gpu_vcycle(synth.CONFIGS[cid], stream, cycles=5 if cid == 3 else 3)
                # config 5: one cycle on the bounded 1,444-pattern sample (~15-30 s of host time)
                r["cpu_baseline"] = cpu_vcycle_ms(synth.CONFIGS[cid], o, pr, cycles=2 if cid == 3 else 1)
                vc[f"config{cid}"] = r
            except Exception as ex:   # noqa: BLE001
                vc[f"config{cid}"] = {"error": str(ex)}
            torch.cuda.empty_cache()
        extras["vcycle"] = vc
        # MG/OPT grid transfers (multigrid.cpp:34-77) at config 4's sizes
        try:
            extras["transfers"] = transfer_rooflines(stream)
        except Exception as ex:   # noqa: BLE001
            extras["transfers_error"] = str(ex)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak" if banded else "strong", "vs_baseline": None,
                "dtype": "f32" if cfg.precision == "c64" else "f64",
                "data": ("synthetic (seeded smooth object from std::mt19937_64 uniforms, Gaussian x quadratic-phase "
                         "probe, data by our GPU forward operator" + (", GPU Poisson noise)" if cfg.photons else ")")),
                "config": {"workload": cfg.describe() if not banded else
                           (f"{cfg.describe()} per GPU: {world} bands of a {world * (cfg.n - overlap) + overlap}x{cfg.n} "
                            f"object, consecutive bands sharing {overlap} rows (one continuous raster)"),
                           "global_batch": total_patterns, "patterns_per_rank": Nr,
                           "parallelism": (f"weak: object bands x{world}, halo rows + misfit all-gathered per evaluation"
                                           if banded else
                                           (f"scan-row blocks x{world}, object row bands (libptg BANDS: halo gradient "
                                            "rows NCCL send/recv + scalar allreduce, iterate halo sync)"
                                            if layout == "bands" else
                                            f"scan-row blocks x{world}, object replicated (libptg REPLICATED: NCCL "
                                            "allreduce of gradient + value)"))
                           if multi else "single GPU",
                           "l2": "flushed between timed steps (512 MiB read)"},
                "roofline": roofline, "roofline_fp32": roofline_fp32, "roofline_hbm": roofline_hbm,
                "step_breakdown": eval_share, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks}
        line.update(extras)
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
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
