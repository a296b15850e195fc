#!/usr/bin/env python
"""Benchmark of the B200 twofold hot path (driver contract: one JSON line on rank 0).

Headline workload: BASELINE.json configs[4] ("cfg5"), the largest config and the
one BASELINE.json shards over 1/2/4/8 GPUs.  One STEP = texp and tlog over 2^30
binary64 twofolds each (x0 ~ U[-700, 700] for texp, 2^e*m log-uniform stand-in
for tlog, x1 = x0*u*2^-53, plus 1% special values -- +-0, +-inf, NaN,
subnormals, exp thresholds -- at seeded positions).  The 2^30 elements of each
function are sharded contiguously over the ranks (rank r of G owns global
elements [r*2^30/G, (r+1)*2^30/G): strong scaling, no collective on the hot
path).  Inputs are generated on the device by the shard-invariant generator;
16 GiB of inputs per function per step exceed the 126 MB L2 (no flush needed).

  value    = elements evaluated per second, whole job (2 * 2^30 / step time),
             CUDA events on the launching stream, max over ranks; the step's two
             independent launches run on two streams so one's tail overlaps the
             other's ramp;
  e2e      = the same metric through the public API, api(64).texp / .tlog on
             pinned HOST tensors (out= pinned host tensors): H2D + kernel + D2H
             inside the timed region (tf_eval_host pipeline), max over ranks;
  roofline = the dominant kernel (tlog): algorithmic FP64 ops per launch over its
             CUDA-event duration, against this GPU's FP64 pipe peak measured in
             the same run (tf_fma_peak; MEASURED_PEAKS.json has no FP64 figure);
             traffic = ncu dram bytes of the same kernel (profiles/);
  cpu_baseline = the CPU port of the reference algorithm (oracle/, "dv" backend,
             bit-exact to the reference package) on all host threads, timed over
             rank 0's whole slice in 2^24-element chunks (~20 s); its outputs are
             also the parity reference of every element (parity_cfg5);
  per_function = the eight (function, width) kernels at the north-star size
             2^28 on their own configs' distributions;
  parity_f32 = config 4 samples vs the reference-equivalent oracle (numpy libm)
             and vs the CR-sim oracle (correctly rounded libm).

`--impl reference` times the CPU port alone (rank 0; the reference package is
pure Python and ~2000x slower still -- it is timed too, on a small sample, when
baseline/_ref holds it) on the same workload and config.
`--gpus N` without torchrun relaunches itself under torch.distributed.run.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# algorithmic FP ops per element (reference op sequence,
# config branch mix), the roofline numerators.  cfg5: the general-path count
# over the 99% non-special elements, specials counted as 0 ops (conservative:
# zeros, subnormals and the thresholds do run the full path in the reference).
ALG_OPS = {("texp", 64): 123.0, ("texpm1", 64): 111.1, ("tlog", 64): 151.4,
           ("tlog1p", 64): 142.1, ("texp", 32): 66.0, ("texpm1", 32): 73.9,
           ("tlog", 32): 106.0, ("tlog1p", 32): 110.0}
ALG_OPS_CFG5 = {"texp": 0.99 * 123.0, "tlog": 0.99 * 152.0}
HEADLINE = (("texp", "exp64s"), ("tlog", "logu64s"))
N_TOTAL = 1 << 30          # elements per function (BASELINE.json configs[4])
# per-function kernels at the north-star size 2^28 (BASELINE.json north_star)
PER_FN = (("texp", 64, "exp64"), ("texpm1", 64, "pow10_64"), ("tlog", 64, "log64"),
          ("tlog1p", 64, "pow10c_64"), ("texp", 32, "exp32"), ("texpm1", 32, "exp32"),
          ("tlog", 32, "log32"), ("tlog1p", 32, "log32"))
N_PER_FN = 1 << 28
SEED = 2024
METRIC = "twofold evals/sec (cfg5: texp+tlog float64, 2^30 each, 1% specials)"
# input arrays each tf_eft op streams (a0 + a1/b0/b1 as the op needs them)
EFT_ARRAYS_IN = {"fast_two_sum": 2, "two_sum": 2, "two_diff": 2, "two_prod": 2, "split": 1,
                 "renorm_fast": 2, "renorm": 2, "t_add": 4, "t_add_d": 3, "t_mul": 4,
                 "t_mul_d": 3, "t_div": 4, "t_sqrt": 2}
EFT_BACKEND_OPS = ("two_prod", "t_mul", "t_mul_d", "t_div", "t_sqrt")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


def config_for(world: int) -> dict:
    """The workload description both arms print (identical for the same N)."""
    return {"workload": "cfg5: texp + tlog over 2^30 float64 twofolds each, 1% specials",
            "elements_per_function": N_TOTAL, "elements_per_function_per_gpu": N_TOTAL // world,
            "global_elements_per_step": 2 * N_TOTAL,
            "parallelism": f"contiguous shards x{world}, no collective on the hot path",
            "l2": "inputs 16 GiB per function per step > 126 MB L2 (no flush needed)"}


class ClockSampler:
    """NVML sampler of SM clock and throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001 -- clocks are reported as unavailable
            self.ok = False

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "sm_min_mhz": min(self.samples), "reasons": names, "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _r(x, nd=4):
    """Compact floats for the JSON line (the driver keeps its tail)."""
    if x is None:
        return None
    return float(f"{x:.{nd}g}")


# ---------------------------------------------------------------- reference arm
def _py_ref_worker(args):
    """Time the reference package itself (scalar calls, its own convention,
    audit.py:343-349) on one chunk of the cfg5 stream."""
    path, fn, dist, start, count = args
    sys.path.insert(0, path)
    from twofold import api

    from paper_1502_05216_b200 import workloads

    x0, x1 = workloads.generate(dist, start, count, seed=SEED)
    f = getattr(api(64), fn)
    pairs = list(zip(x0.tolist(), x1.tolist()))
    t = time.perf_counter()
    for p in pairs:
        f(p)
    return time.perf_counter() - t


def python_reference(nt: int, per_proc: int) -> dict | None:
    """The reference package (pkg/src/twofold, installed in baseline/_ref) on
    a small sample: nt processes, each evaluating per_proc elements of each
    function in a loop of scalar calls."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "twofold")):
        return {"unavailable": "baseline/_ref not installed"}
    import multiprocessing as mp

    jobs = [(path, fn, dist, k * per_proc, per_proc) for fn, dist in HEADLINE for k in range(nt)]
    ctx = mp.get_context("spawn")
    with ctx.Pool(nt) as pool:
        pool.map(_py_ref_worker, [(path, fn, dist, 0, 64) for fn, dist in HEADLINE] * nt)
        t = time.perf_counter()
        busy = pool.map(_py_ref_worker, jobs)
        wall = time.perf_counter() - t
    n = len(jobs) * per_proc
    return {"value": _r(n / wall), "unit": "elements/s", "processes": nt,
            "us_per_call_1core": _r(sum(busy) / n * 1e6),
            "sample": f"{per_proc} elements x {nt} processes per function, scalar calls",
            "backend": "dv (no gmpy2 / math.fma on the box)"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """CPU port of the reference algorithm (oracle/, kind "port"), all host
    threads, on rank 0; other ranks exit without work."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1502_05216_b200 import workloads

    O.build()
    nt = O.default_threads()
    sample = min(args.ref_sample, N_TOTAL)
    data = {fn: workloads.generate(dist, 0, sample, seed=SEED) for fn, dist in HEADLINE}
    times = []
    for it in range(args.warmup + args.steps):
        t = time.perf_counter()
        for fn, _ in HEADLINE:
            O.evaluate(fn, 64, *data[fn], backend="dv", nthreads=nt)
        if it >= args.warmup:
            times.append(time.perf_counter() - t)
    per_step = statistics.median(times)
    value = 2 * sample / per_step
    pyref = python_reference(nt, args.py_ref_sample) if args.py_ref_sample > 0 else None
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg-5 generator)",
        "config": config_for(world),
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": nt, "kind": "port",
                         "cpu": cpu_model(),
                         "sample": f"{sample} elements per function per step (prefix of the "
                                   f"2^30-element cfg-5 stream), C port of the reference "
                                   f"algorithm, {nt} threads"},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_python": pyref,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    from paper_1502_05216_b200 import Twofold, _lib, api, workloads

    rank, world, local = dist_env()
    if args.dist_backend == "gloo":
        # code-path check of the N > 1 arm on a box with fewer GPUs: ranks may
        # share a device (their kernels never wait on one another; the timings
        # of such a run mean nothing)
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    L = _lib.ensure_device(local)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    f64 = api(64)
    peaks = _peaks()

    def gen(dist_name, n, dt, start):
        x0 = torch.empty(n, dtype=dt, device=dev)
        x1 = torch.empty(n, dtype=dt, device=dev)
        _lib.check(L.tf_generate(_lib.DIST_CODES[dist_name], SEED, start, n, x0.data_ptr(),
                                 x1.data_ptr(), sp), "tf_generate")
        return x0, x1

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist

        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def events():
        return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    # ---- headline step: texp + tlog over this rank's cfg-5 slice
    start, n = shard(N_TOTAL, rank, world)
    ins, outs = {}, {}
    for fn, dname in HEADLINE:
        ins[fn] = gen(dname, n, torch.float64, start)
        outs[fn] = (torch.empty(n, dtype=torch.float64, device=dev),
                    torch.empty(n, dtype=torch.float64, device=dev))
    torch.cuda.synchronize()
    streams = [stream] + [torch.cuda.Stream(dev) for _ in range(args.streams - 1)]

    def step(evs=None):
        if len(streams) > 1:
            go = torch.cuda.Event()
            go.record(stream)
            for s in streams[1:]:
                s.wait_event(go)
        for k, (fn, _) in enumerate(HEADLINE):
            st = streams[k % len(streams)]
            if evs is not None:
                evs[k][0].record(st)
            a0, a1 = ins[fn]
            z0, z1 = outs[fn]
            f64._launch(fn, a0, a1, z0, z1, n, st.cuda_stream)
            if evs is not None:
                evs[k][1].record(st)
        for s in streams[1:]:
            done = torch.cuda.Event()
            done.record(s)
            stream.wait_event(done)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launch_ev = [[events() for _ in HEADLINE] for _ in range(args.steps)]
    t0, t1 = events()
    with ClockSampler(local) as clk:
        t0.record(stream)
        for s in range(args.steps):
            step(launch_ev[s])
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = max_over_ranks(t0.elapsed_time(t1))
    ms_step = ms_total / args.steps
    value = 2 * N_TOTAL / (ms_step * 1e-3)
    # per-kernel durations (roofline) from the same steps run serialised on one
    # stream (overlapped launches stretch each other's events)
    streams[1:] = []
    torch.cuda.synchronize()
    for s in range(args.steps):
        step(launch_ev[s])
    torch.cuda.synchronize()
    kern_ms = {fn: max_over_ranks(statistics.mean(
                   launch_ev[s][k][0].elapsed_time(launch_ev[s][k][1]) for s in range(args.steps)))
               for k, (fn, _) in enumerate(HEADLINE)}
    # share of the slice the exact path evaluated, counted in one extra launch
    exact_frac = {}
    cnt = ctypes.c_ulonglong(0)
    for fn, _ in HEADLINE:
        _lib.check(L.tf_exact_count(ctypes.byref(cnt), 1), "tf_exact_count")
        f64._launch(fn, *ins[fn], *outs[fn], n, sp, flags=_lib.FLAG_COUNT_EXACT)
        torch.cuda.synchronize()
        _lib.check(L.tf_exact_count(ctypes.byref(cnt), 1), "tf_exact_count")
        exact_frac[fn] = _r(cnt.value / n, 3)

    # ---- FP64 / FP32 pipe peak of this GPU (roofline denominator)
    peak, peak_by_op = {}, {}
    buf = torch.zeros(4, dtype=torch.float64, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    for width in (64, 32):
        blocks, iters = sms * 8, 4096 if width == 64 else 8192
        for op, name in ((0, "fma"), (1, "add"), (2, "mul")):
            code = width + 100 * op
            _lib.check(L.tf_fma_peak(code, buf.data_ptr(), blocks, iters, sp), "peak")
            e0, e1 = events()
            e0.record(stream)
            _lib.check(L.tf_fma_peak(code, buf.data_ptr(), blocks, iters, sp), "peak")
            e1.record(stream)
            torch.cuda.synchronize()
            peak_by_op[f"f{width}_{name}"] = blocks * 256 * iters * 8 / (e0.elapsed_time(e1) * 1e-3)
        peak[width] = max(peak_by_op[f"f{width}_{k}"] for k in ("fma", "add", "mul"))

    # ---- roofline of the dominant kernel
    dom = max(kern_ms, key=kern_ms.get)
    dom_ms = kern_ms[dom]
    ops = ALG_OPS_CFG5[dom] * n / (dom_ms * 1e-3)
    gbs = 32 * n / (dom_ms * 1e-3) / 1e9
    roof = {"bound": "fp64", "kernel": f"k_eval<double,{dom}>", "achieved": ops / 1e12,
            "peak": peak[64] / 1e12, "unit": "TFLOP/s", "frac": ops / peak[64],
            "traffic": _traffic(dom, n), "ops_per_element": ALG_OPS_CFG5[dom],
            "elements_per_launch": n, "launch_ms": dom_ms,
            "peak_source": "measured in this run: tf_fma_peak, best of DADD/DMUL/DFMA chains",
            "hbm_gbs": gbs, "hbm_frac": gbs / peaks["hbm_gbs"]}

    # ---- parity of this rank's slice prefix against the CPU port (which is
    # also the timed cpu_baseline on rank 0); one small merge over the ranks
    from oracle import oracle as O

    O.build()
    nt = O.default_threads()
    # the sample is split over the ranks: the merged counts cover the same number
    # of elements at every N, and the CPU port's time per rank shrinks with N
    m = min(max(1, args.parity_sample // world), n)
    cpu = None
    parity5 = {}
    for fn, _ in HEADLINE:
        parity5[fn] = _parity_chunked(L, dev, sp, O, fn, ins[fn], outs[fn], m, args.parity_host,
                                      nt)
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu_s = sum(parity5[fn].pop("cpu_s") for fn, _ in HEADLINE)
        cpu = {"value": _r(2 * m / cpu_s), "unit": "elements/s", "cores": nt, "kind": "port",
               "cpu": cpu_model(),
               "sample": f"{m} elements of each function ({'all' if m == n else 'a prefix'} "
                         f"of the cfg-5 slice, in 2^24-element chunks), C port of the reference "
                         f"algorithm ('dv' backend), {nt} threads"}
    for fn, _ in HEADLINE:
        parity5[fn].pop("cpu_s", None)
        parity5[fn] = _reduce(parity5[fn], dev)

    # ---- config 1 at its own size (2^20 texp f64): launch-overhead regime,
    # eager launches vs one CUDA graph of 100 launches
    small = None
    if not args.headline_only:
        ms_ = 1 << 20
        a0, a1 = gen("exp64", ms_, torch.float64, rank * ms_)
        z0, z1 = torch.empty_like(a0), torch.empty_like(a0)
        for _ in range(5):
            f64._launch("texp", a0, a1, z0, z1, ms_, sp)
        reps = 100
        e0, e1 = events()
        e0.record(stream)
        for _ in range(reps):
            f64._launch("texp", a0, a1, z0, z1, ms_, sp)
        e1.record(stream)
        torch.cuda.synchronize()
        eager_ms = max_over_ranks(e0.elapsed_time(e1) / reps)
        g = torch.cuda.CUDAGraph()
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        with torch.cuda.stream(gs):
            with torch.cuda.graph(g, stream=gs):
                for _ in range(reps):
                    f64._launch("texp", a0, a1, z0, z1, ms_, gs.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        graph_ms = max_over_ranks(e0.elapsed_time(e1) / reps)
        small = {"n": ms_, "eager_gps": _r(ms_ * world / (eager_ms * 1e-3) / 1e9),
                 "graph_gps": _r(ms_ * world / (graph_ms * 1e-3) / 1e9)}
        del a0, a1, z0, z1, g

    # ---- the reference's own calling convention: one scalar twofold per call
    # (audit.py:343-349), through api(64) on Python floats
    scalar = None
    if not args.headline_only:
        from paper_1502_05216_b200 import workloads as W

        scalar = {}
        for fn, dname in HEADLINE:
            x0s, x1s = W.generate(dname, 0, 512, seed=SEED)
            pairs = list(zip(x0s.tolist(), x1s.tolist()))
            f = getattr(f64, fn)
            for p_ in pairs[:64]:
                f(p_)
            t = time.perf_counter()
            for p_ in pairs:
                f(p_)
            scalar[fn] = _r((time.perf_counter() - t) / len(pairs) * 1e6)
        scalar["unit"] = "us per call (api(64).fn((x0, x1)) on Python floats)"

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        del outs
        torch.cuda.empty_cache()
        host = {}
        for fn, _ in HEADLINE:
            a0, a1 = ins[fn]
            h0 = torch.empty(n, dtype=torch.float64, pin_memory=True)
            h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
            h0.copy_(a0)
            h1.copy_(a1)
            host[fn] = (h0, h1)
        del ins
        torch.cuda.empty_cache()
        hout = (torch.empty(n, dtype=torch.float64, pin_memory=True),
                torch.empty(n, dtype=torch.float64, pin_memory=True))
        for _ in range(min(args.warmup, 2)):
            for fn, _ in HEADLINE:
                getattr(f64, fn)(Twofold(*host[fn]), out=hout)
        barrier()
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        tw = time.perf_counter()
        for _ in range(e2e_steps):
            for fn, _ in HEADLINE:
                z = getattr(f64, fn)(Twofold(*host[fn]), out=hout)
                _ = float(z.value[n - 1])          # the step's result is on the host
        t_e2e = max_over_ranks((time.perf_counter() - tw) / e2e_steps)
        e2e = {"value": 2 * N_TOTAL / t_e2e, "unit": "elements/s",
               "h2d_bytes_per_step": 2 * 2 * n * 8, "d2h_bytes_per_step": 2 * 2 * n * 8,
               "ms_per_step": _r(t_e2e * 1e3), "steps": e2e_steps,
               "path": "api(64).texp/tlog(Twofold(pinned host tensors), out=pinned host tensors)"}
        del host, hout
    else:
        del ins, outs
    torch.cuda.empty_cache()

    # ---- per-function kernel rates at 2^28 (north-star size)
    per_fn = {}
    if not args.headline_only:
        for fn, width, dname in PER_FN:
            mm = N_PER_FN
            dt = torch.float64 if width == 64 else torch.float32
            a0, a1 = gen(dname, mm, dt, rank * mm)
            z0, z1 = torch.empty_like(a0), torch.empty_like(a1)
            lib = api(width)
            for _ in range(max(3, args.warmup)):
                lib._launch(fn, a0, a1, z0, z1, mm, sp)
            reps = max(5, min(args.steps, 20))
            e0, e1 = events()
            e0.record(stream)
            for _ in range(reps):
                lib._launch(fn, a0, a1, z0, z1, mm, sp)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = max_over_ranks(e0.elapsed_time(e1) / reps)
            fp = ALG_OPS[(fn, width)] * mm / (ms * 1e-3) / peak[width]
            hbm = (32 if width == 64 else 16) * mm / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"]
            # bound = the slower of the two rooflines (north_star)
            bound = "fp" if ALG_OPS[(fn, width)] / peak[width] > \
                (32 if width == 64 else 16) / (peaks["hbm_gbs"] * 1e9) else "hbm"
            per_fn[f"{fn}{width}"] = [_r(mm * world / (ms * 1e-3) / 1e9), bound,
                                      _r(fp if bound == "fp" else hbm, 3), _r(fp, 3), _r(hbm, 3)]
            del a0, a1, z0, z1
        torch.cuda.empty_cache()

    # ---- binary32 parity (config 4 samples) vs the reference and CR-sim oracles
    par32 = {}
    if not args.headline_only and args.parity32_sample > 0:
        m32 = max(1, args.parity32_sample // world)
        for fn, width, dname in PER_FN:
            if width != 32:
                continue
            a0, a1 = gen(dname, m32, torch.float32, rank * m32)
            z = getattr(api(32), fn)((a0, a1))
            torch.cuda.synchronize()
            z0, z1 = z.value.cpu().numpy(), z.error.cpu().numpy()
            x0, x1 = a0.cpu().numpy(), a1.cpu().numpy()
            ref = O.evaluate(fn, 32, x0, x1, backend="dv", nthreads=nt)
            crs = O.evaluate(fn, 32, x0, x1, backend="fma", libm32="cr", nthreads=nt)
            par32[fn] = {"ref": _compact(_reduce(_host_compare(z0, z1, *ref, 32), dev)),
                         "crsim": _compact(_reduce(_host_compare(z0, z1, *crs, 32), dev))}

    if args.extended and rank == 0:
        _extended(args, L, dev, stream, sp, gen, peaks)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded shard-invariant cfg-5 generator, on device)",
            "config": config_for(world),
            "gpu_launches": len(HEADLINE) * args.steps,
            "kernel_ms": {k: _r(v) for k, v in kern_ms.items()},
            "exact_path_frac": exact_frac,
            "clocks": clk.summary(),
            "roofline": {k: (_r(v) if isinstance(v, float) else v) for k, v in roof.items()},
            "fp_peak_tops": {k: _r(v / 1e12) for k, v in peak_by_op.items()},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "cfg1_small": small,
            "scalar_call_us": scalar,
            "parity_legend": PARITY_LEGEND,
            "parity_cfg5": {fn: _compact(v) for fn, v in parity5.items()},
            "per_function_legend": "G elem/s, bound, frac of bound, fp frac, hbm frac (2^28)",
            "parity_f32_legend": "vs the reference (numpy libm) / vs CR-sim, 2^22 of cfg 4",
            "per_function": per_fn,
            "parity_f32": par32,
        }
        print(json.dumps(line, separators=(",", ":")), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def _extended(args, L, dev, stream, sp, gen, peaks):
    """--extended PATH: the sixteen sibling kernels on their family's 2^28-element
    inputs and the element-wise EFT / twofold-arithmetic ops at 2^25, written to
    PATH as JSON (kept out of the driver's bench line)."""
    import torch

    from paper_1502_05216_b200 import DOTTED_ARG, FAMILIES, _lib, api, family_of

    def timed(go, reps):
        for _ in range(3):
            go()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            go()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out = {"siblings": {}, "eft_ops": {}}
    for fn, width, dname in PER_FN:
        m = N_PER_FN
        dt = torch.float64 if width == 64 else torch.float32
        a0, a1 = gen(dname, m, dt, 0)
        z0, z1 = torch.empty_like(a0), torch.empty_like(a1)
        lib = api(width)
        base = timed(lambda: lib._launch(fn, a0, a1, z0, z1, m, sp), 5)
        for name in FAMILIES[family_of(fn)]:
            if name == fn:
                continue
            b1 = a0 if name in DOTTED_ARG else a1
            ms = timed(lambda: lib._launch(name, a0, b1, z0, z1, m, sp), 5)
            out["siblings"][f"{name}_f{width}"] = {
                "config_dist": dname, "elements": m, "ms": ms,
                "elements_per_s": m / (ms * 1e-3), "vs_" + fn: base / ms}
        del a0, a1, z0, z1
    m = 1 << 25
    for width in (64, 32):
        dt = torch.float64 if width == 64 else torch.float32
        sz = 8 if width == 64 else 4
        ops_in = [torch.empty(m, dtype=dt, device=dev).uniform_(1.0, 2.0) for _ in range(4)]
        z0, z1 = torch.empty_like(ops_in[0]), torch.empty_like(ops_in[0])
        ptrs = [a.data_ptr() for a in ops_in]
        for op, code in _lib.OP_CODES.items():
            for backend in ((0, 1) if op in EFT_BACKEND_OPS else (0,)):
                def go(code=code, backend=backend):
                    _lib.check(L.tf_eft(code, width, backend, *ptrs, z0.data_ptr(), z1.data_ptr(),
                                        m, sp), "tf_eft")
                ms = timed(go, 10)
                gbs = (EFT_ARRAYS_IN[op] + 2) * sz * m / (ms * 1e-3) / 1e9
                out["eft_ops"][f"{op}{'_dv' if backend else ''}_f{width}"] = {
                    "elements_per_s": m / (ms * 1e-3), "ms": ms, "hbm_gbs": gbs,
                    "hbm_frac": gbs / peaks["hbm_gbs"]}
        del ops_in, z0, z1
    with open(args.extended, "w") as f:
        json.dump(out, f, indent=1)


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """This rank's contiguous slice [start, start + n) of the global index
    range (paper_1502_05216_b200.dist.shard_range)."""
    from paper_1502_05216_b200.dist import shard_range

    return shard_range(total, rank, world)


def _traffic(fn, n):
    """ncu dram read+write bytes per launch of k_eval<double,fn> on the cfg-5
    inputs, from the committed `ncu --set full` capture (profiles/), scaled
    to this launch's element count (traffic per element is size-independent
    for a streaming kernel); None without a capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            rec = json.load(f).get(f"cfg5_{fn}_f64")
        if rec:
            return rec["traffic_bytes"] * n / rec["elements"]
    except (OSError, ValueError, KeyError):
        pass
    return None


def _parity_chunked(L, dev, sp, O, fn, xin, zout, m, host_n, nt, chunk=1 << 24):
    """Parity of the first m elements of a binary64 slice against the CPU port
    (the reference algorithm, "dv" backend), chunk by chunk: counters on the
    device (tf_compare) over all m, the host comparator's finer statistics over
    the first host_n.  Also returns the port's total time ("cpu_s")."""
    import torch

    from paper_1502_05216_b200 import _lib

    st = torch.zeros(6, dtype=torch.int64, device=dev)
    cpu_s, fine = 0.0, {}
    for lo in range(0, m, chunk):
        k = min(chunk, m - lo)
        x0 = xin[0][lo:lo + k].cpu().numpy()
        x1 = xin[1][lo:lo + k].cpu().numpy()
        tc = time.perf_counter()
        r0, r1 = O.evaluate(fn, 64, x0, x1, backend="dv", nthreads=nt)
        cpu_s += time.perf_counter() - tc
        t0, t1 = torch.from_numpy(r0).to(dev), torch.from_numpy(r1).to(dev)
        _lib.check(L.tf_compare(64, zout[0][lo:].data_ptr(), zout[1][lo:].data_ptr(),
                                t0.data_ptr(), t1.data_ptr(), k, 2.0 ** -95, 2 * 2.0 ** -1074,
                                st.data_ptr(), sp), "tf_compare")
        if lo == 0 and host_n:
            h = min(host_n, k)
            fine = _host_compare(zout[0][:h].cpu().numpy(), zout[1][:h].cpu().numpy(), r0[:h],
                                 r1[:h], 64)
            fine = {"host_n": h} | {key: fine[key] for key in (
                "tol_violations_given_z0_match", "z1_bit_mismatch_given_z0_match",
                "worst_rel_log2", "z0_ulp_hist")}
    torch.cuda.synchronize()
    c = st.tolist()
    return {"n": c[0], "z0_mismatch": c[1], "z0_gt1ulp": c[2], "tol_violations": c[3],
            "class_mismatch": c[4], "z1_bit_mismatch": c[5], **fine, "cpu_s": cpu_s}


def _host_compare(z0, z1, r0, r1, width):
    from oracle.compare import compare

    return compare(z0, z1, r0, r1, width)


def _reduce(stats, dev):
    """Merge a rank's parity record over all ranks (the one small collective
    of the run: an 80-byte all-gather merged by tf_reduce_stats)."""
    from paper_1502_05216_b200.dist import reduce_stats

    s = dict(stats)
    s.pop("bad_idx", None)
    return reduce_stats(s, device=dev)


PARITY_LEGEND = ("n, z0 mismatches, z0 beyond 1 ulp, tol violations, tol violations given "
                 "z0 match, class mismatches, worst log2 rel, z0 ulp histogram")


def _compact(s):
    """One parity record as a short list (PARITY_LEGEND order)."""
    hist = s.get("z0_ulp_hist")
    return [s.get("n"), s.get("z0_mismatch"), s.get("z0_gt1ulp"), s.get("tol_violations"),
            s.get("tol_violations_given_z0_match"), s.get("class_mismatch"),
            _r(s.get("worst_rel_log2")),
            {str(a): b for a, b in hist.items()} if isinstance(hist, dict) else None]


def relaunch(args) -> int:
    """--gpus N outside torchrun: run this script under torch.distributed.run
    with one rank per GPU (the driver's own launch for N > 1)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--ref-sample", type=int, default=1 << 25,
                    help="reference arm: elements per function per step (prefix of the stream)")
    ap.add_argument("--py-ref-sample", type=int, default=2048,
                    help="reference arm: elements per process per function for the Python package")
    ap.add_argument("--parity-sample", type=int, default=1 << 30,
                    help="cfg-5 elements per function checked against the CPU port (default: "
                         "all of them)")
    ap.add_argument("--parity-host", type=int, default=1 << 22,
                    help="of those, elements also run through the host comparator")
    ap.add_argument("--parity32-sample", type=int, default=1 << 22)
    ap.add_argument("--e2e-steps", type=int, default=1 << 30)
    ap.add_argument("--headline-only", action="store_true")
    ap.add_argument("--extended", default=None, metavar="PATH",
                    help="also time the sibling kernels and the EFT ops, JSON to PATH")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=("nccl", "gloo"),
                    help="gloo: exercise the N > 1 code path with ranks sharing GPUs (tests)")
    ap.add_argument("--streams", type=int, default=2, choices=(1, 2),
                    help="run the step's two functions on 1 or 2 streams")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        return relaunch(args)
    if world is not None and int(world) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
