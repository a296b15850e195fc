#!/usr/bin/env python
"""Benchmark of the B200 twofold hot path (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], the single-GPU config the metric is quoted
on): one STEP = texpm1 and tlog1p over the cfg-2 float64 twofolds, N = 2^24
each (x0 = +-s*10^-e, s~U[1,10), e~U{0..300}; tlog1p clamped to
[-1+2^-52, 1e300]; x1 = x0*u*2^-53).  Inputs are generated on the device by
the shard-invariant generator (rank r of G owns global elements
[r*N, (r+1)*N) -- weak scaling, no collective on the hot path).  The 512 MiB
of inputs per step exceed the 126 MB L2, so no flush is needed.

  value  = elements evaluated per second, whole job (sum over ranks), CUDA
           events on the launching stream, max over ranks; the step's two
           independent functions run on two streams (--streams 2), so one
           launch's tail overlaps the next one's ramp;
  e2e    = the same metric through the public API with pinned HOST buffers
           (H2D + kernels + D2H inside the timed region, wall clock);
  per_function = every (function, width) kernel at its own config and size
           (2^24 / 2^26 binary64, 2^28 binary32; config 1 at 2^26, its 2^20
           launch-overhead regime separately as cfg1_small), same timing rules;
  roofline = the dominant kernel's algorithmic FP64 op rate vs the measured
           FP64 FMA-pipe peak of this GPU (tf_fma_peak), plus its HBM rate;
  cpu_baseline = the CPU oracle (C port of the reference algorithm, all host
           threads) on a bounded sample of the same workload.

`--impl reference` times that CPU port alone (rank 0) on the same workload.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# algorithmic FP ops per element (reference op sequence,
# config branch mix), the roofline numerators.
ALG_OPS = {("texp", 64): 123.0, ("texpm1", 64): 111.1, ("tlog", 64): 151.4,
           ("tlog1p", 64): 142.1, ("texp", 32): 66.0, ("texpm1", 32): 73.9,
           ("tlog", 32): 106.0, ("tlog1p", 32): 110.0}
HEADLINE = (("texpm1", "cfg2_texpm1_f64"), ("tlog1p", "cfg2_tlog1p_f64"))
PER_FN = {
    ("texp", 64): "cfg1_texp_f64", ("texpm1", 64): "cfg2_texpm1_f64",
    ("tlog", 64): "cfg3_tlog_f64", ("tlog1p", 64): "cfg2_tlog1p_f64",
    ("texp", 32): "cfg4_texp_f32", ("texpm1", 32): "cfg4_texpm1_f32",
    ("tlog", 32): "cfg4_tlog_f32", ("tlog1p", 32): "cfg4_tlog1p_f32",
}
# input arrays each tf_eft op streams (a0 + a1/b0/b1 as the op needs them)
EFT_ARRAYS_IN = {"fast_two_sum": 2, "two_sum": 2, "two_diff": 2, "two_prod": 2, "split": 1,
                 "renorm_fast": 2, "renorm": 2, "t_add": 4, "t_add_d": 3, "t_mul": 4,
                 "t_mul_d": 3, "t_div": 4, "t_sqrt": 2}
EFT_BACKEND_OPS = ("two_prod", "t_mul", "t_mul_d", "t_div", "t_sqrt")
N_HEAD = 1 << 24
# per-function sizes: each config's own N (BASELINE.json), except config 1's
# 2^20 (the launch-overhead regime, measured separately as cfg1_small)
N_CFG = {"cfg1_texp_f64": 1 << 26}
SEED = 2024


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


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
                "reasons": names, "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    """CPU port of the reference algorithm (oracle/, kind "port"), all host threads."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1502_05216_b200 import workloads

    O.build()
    nt = O.default_threads()
    sample = args.ref_sample
    data = {}
    for fn, cfg in HEADLINE:
        _, width, dist, _ = workloads.CONFIGS[cfg]
        data[fn] = workloads.generate(dist, 0, sample, seed=SEED)
    times = []
    for it in range(args.warmup + args.steps):
        t = time.perf_counter()
        for fn, _ in HEADLINE:
            O.evaluate(fn, 64, *data[fn], backend="dv", nthreads=nt)
        if it >= args.warmup:
            times.append(time.perf_counter() - t)
    per_step = statistics.median(times)
    value = 2 * sample / per_step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg-2 generator)",
        "config": {"workload": "cfg2: texpm1 + tlog1p over float64 twofolds",
                   "elements_per_function": sample, "sample_of": N_HEAD},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": nt, "kind": "port",
                         "sample": f"{sample} elements per function per step "
                                   f"(bounded sample of the 2^24-element cfg-2 step)"},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "twofold evals/sec (cfg2: texpm1+tlog1p float64, N=2^24 each)"


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    from paper_1502_05216_b200 import DOTTED_ARG, FAMILIES, Twofold, _lib, api, family_of, workloads

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    L = _lib.ensure_device(local)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    f64 = api(64)

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

    # ---- headline step: texpm1 + tlog1p over cfg-2, N per rank
    n = args.n
    start = rank * n
    ins, outs = {}, {}
    for fn, cfg in HEADLINE:
        _, width, dname, _ = workloads.CONFIGS[cfg]
        ins[fn] = gen(dname, n, torch.float64, start)
        outs[fn] = (torch.empty(n, dtype=torch.float64, device=dev),
                    torch.empty(n, dtype=torch.float64, device=dev))
    torch.cuda.synchronize()

    # The step's two functions are independent: with --streams 2 the second
    # runs on its own stream, so its CTAs take each SM as soon as the first
    # kernel's CTA there retires (the two launches' ramp and tail overlap).
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
    launch_ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in HEADLINE] for _ in range(args.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for s in range(args.steps):
            step(launch_ev[s])
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = max_over_ranks(t0.elapsed_time(t1))
    ms_step = ms_total / args.steps
    value = 2 * n * world / (ms_step * 1e-3)
    if len(streams) > 1:
        # overlapped launches stretch each other's events: the per-kernel
        # durations (roofline) come from the same steps run serialised
        streams[1:] = []
        torch.cuda.synchronize()
        for s in range(args.steps):
            step(launch_ev[s])
        torch.cuda.synchronize()
    kern_ms = {fn: max_over_ranks(statistics.mean(
                   launch_ev[s][k][0].elapsed_time(launch_ev[s][k][1]) for s in range(args.steps)))
               for k, (fn, _) in enumerate(HEADLINE)}

    # ---- FP64 / FP32 FMA-pipe peak of this GPU (roofline denominator)
    peak = {}
    buf = torch.zeros(4, dtype=torch.float64, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_by_op = {}
    for width in (64, 32):
        blocks, iters = sms * 8, 4096 if width == 64 else 8192
        for op, name in ((0, "fma"), (1, "add"), (2, "mul")):
            code = width + 100 * op
            _lib.check(L.tf_fma_peak(code, buf.data_ptr(), blocks, iters, sp), "peak")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _lib.check(L.tf_fma_peak(code, buf.data_ptr(), blocks, iters, sp), "peak")
            e1.record(stream)
            torch.cuda.synchronize()
            peak_by_op[f"f{width}_{name}"] = blocks * 256 * iters * 8 / (e0.elapsed_time(e1) * 1e-3)
        # the roofline denominator: the fastest of add / mul / fma (conservative)
        peak[width] = max(peak_by_op[f"f{width}_{n}"] for n in ("fma", "add", "mul"))

    # ---- per-function kernel rates at their configs
    per_fn, siblings = {}, {}
    if not args.headline_only:
        for (fn, width), cfg in PER_FN.items():
            _, _, dname, _ = workloads.CONFIGS[cfg]
            m = N_CFG.get(cfg, workloads.CONFIGS[cfg][3])
            dt = torch.float64 if width == 64 else torch.float32
            a0, a1 = gen(dname, m, dt, rank * m)
            z0, z1 = torch.empty_like(a0), torch.empty_like(a1)
            lib = api(width)

            def time_fn(name, reps):
                b1 = a0 if name in DOTTED_ARG else a1      # plain argument: x1 unused
                for _ in range(max(3, args.warmup)):
                    lib._launch(name, a0, b1, z0, z1, m, sp)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(reps):
                    lib._launch(name, a0, b1, z0, z1, m, sp)
                e1.record(stream)
                torch.cuda.synchronize()
                return max_over_ranks(e0.elapsed_time(e1) / reps)

            ms = time_fn(fn, max(5, min(args.steps, 50)))
            rate = m * world / (ms * 1e-3)
            ops = ALG_OPS[(fn, width)] * m / (ms * 1e-3)
            gbs = (32 if width == 64 else 16) * m / (ms * 1e-3) / 1e9
            per_fn[f"{fn}_f{width}"] = {
                "config": cfg, "elements": m, "ms": ms, "elements_per_s": rate,
                "alg_gops": ops / 1e9, "fp_pipe_frac": ops / peak[width],
                "hbm_gbs": gbs, "hbm_frac": gbs / _peaks()["hbm_gbs"]}
            if not args.no_siblings:
                # the other four functions of the family, same inputs (a dotted
                # function reads x0 only)
                for name in FAMILIES[family_of(fn)]:
                    if name == fn:
                        continue
                    sms = time_fn(name, 5)
                    siblings[f"{name}_f{width}"] = {
                        "config": cfg, "elements": m, "ms": sms,
                        "elements_per_s": m * world / (sms * 1e-3),
                        "vs_" + fn: ms / sms}
            del a0, a1, z0, z1

    # ---- config 1 at its own size (2^20 texp f64): the launch-overhead regime,
    # eager launches vs one CUDA graph of 100 launches
    small = None
    if not args.headline_only:
        m = 1 << 20
        a0, a1 = gen("exp64", m, torch.float64, rank * m)
        z0, z1 = torch.empty_like(a0), torch.empty_like(a0)
        f = api(64)
        for _ in range(5):
            f._launch("texp", a0, a1, z0, z1, m, sp)
        reps = 100
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            f._launch("texp", a0, a1, z0, z1, m, sp)
        e1.record(stream)
        torch.cuda.synchronize()
        eager_ms = max_over_ranks(e0.elapsed_time(e1) / reps)
        g = torch.cuda.CUDAGraph()
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        with torch.cuda.stream(gs):
            with torch.cuda.graph(g, stream=gs):
                for _ in range(reps):
                    f._launch("texp", a0, a1, z0, z1, m, gs.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        graph_ms = max_over_ranks(e0.elapsed_time(e1) / reps)
        small = {"config": "cfg1_texp_f64", "elements": m,
                 "eager_ms": eager_ms, "eager_elements_per_s": m * world / (eager_ms * 1e-3),
                 "graph_ms": graph_ms, "graph_elements_per_s": m * world / (graph_ms * 1e-3),
                 "graph_launches": reps}
        del a0, a1, z0, z1, g

    # ---- config 5: texp and tlog over 2^30 binary64 twofolds with 1% special
    # values, sharded contiguously across the ranks (strong scaling: the total is
    # fixed, each rank evaluates its 2^30 / N slice; no collective on the path)
    cfg5 = {}
    if not args.headline_only and not args.no_cfg5:
        for cname in ("cfg5_texp_f64", "cfg5_tlog_f64"):
            fn, _, dname, total = workloads.CONFIGS[cname]
            per = total // world
            a0, a1 = gen(dname, per, torch.float64, rank * per)
            z0, z1 = torch.empty_like(a0), torch.empty_like(a0)
            for _ in range(max(3, args.warmup)):
                f64._launch(fn, a0, a1, z0, z1, per, sp)
            reps = max(3, min(args.steps, 10))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record(stream)
            for _ in range(reps):
                f64._launch(fn, a0, a1, z0, z1, per, sp)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = max_over_ranks(e0.elapsed_time(e1) / reps)
            # share of the slice the exact path evaluated (the specials and the
            # rare fast-path rejects), counted in one extra launch
            cnt = ctypes.c_ulonglong(0)
            _lib.check(L.tf_exact_count(ctypes.byref(cnt), 1), "tf_exact_count")
            f64._launch(fn, a0, a1, z0, z1, per, sp, flags=2)   # TF_FLAG_COUNT_EXACT
            torch.cuda.synchronize()
            _lib.check(L.tf_exact_count(ctypes.byref(cnt), 1), "tf_exact_count")
            cfg5[cname] = {"elements_total": per * world, "elements_per_rank": per, "ms": ms,
                           "elements_per_s": per * world / (ms * 1e-3), "scaling": "strong",
                           "exact_path_fraction_rank0": cnt.value / per}
            del a0, a1, z0, z1
        torch.cuda.empty_cache()

    # ---- element-wise EFT / twofold arithmetic ops (HBM-bound streaming)
    eft_rates = {}
    if not args.headline_only and not args.no_eft:
        m = 1 << 25
        for width in (64, 32):
            dt = torch.float64 if width == 64 else torch.float32
            sz = 8 if width == 64 else 4
            ops_in = [torch.empty(m, dtype=dt, device=dev).uniform_(1.0, 2.0) for _ in range(4)]
            z0, z1 = torch.empty_like(ops_in[0]), torch.empty_like(ops_in[0])
            ptrs = [a.data_ptr() for a in ops_in]
            for op, code in _lib.OP_CODES.items():
                for backend in ((0, 1) if op in EFT_BACKEND_OPS else (0,)):
                    def go():
                        _lib.check(L.tf_eft(code, width, backend, *ptrs, z0.data_ptr(),
                                            z1.data_ptr(), m, sp), "tf_eft")
                    for _ in range(3):
                        go()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    for _ in range(10):
                        go()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms = max_over_ranks(e0.elapsed_time(e1) / 10)
                    gbs = (EFT_ARRAYS_IN[op] + 2) * sz * m / (ms * 1e-3) / 1e9
                    name = f"{op}{'_dv' if backend else ''}_f{width}"
                    eft_rates[name] = {"elements_per_s": m * world / (ms * 1e-3), "ms": ms,
                                       "hbm_gbs": gbs, "hbm_frac": gbs / _peaks()["hbm_gbs"]}
            del ops_in, z0, z1
    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        host, hout = {}, {}
        for fn, _ in HEADLINE:
            a0, a1 = ins[fn]
            host[fn] = (a0.cpu().pin_memory(), a1.cpu().pin_memory())
            hout[fn] = (torch.empty(n, dtype=torch.float64).pin_memory(),
                        torch.empty(n, dtype=torch.float64).pin_memory())
        # warm the pipeline (ring buffers, pinned-page mappings)
        for _ in range(2):
            for fn, _ in HEADLINE:
                getattr(f64, fn)(Twofold(*host[fn]), out=hout[fn])
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        barrier()
        tw = time.perf_counter()
        for _ in range(e2e_steps):
            for fn, _ in HEADLINE:
                z = getattr(f64, fn)(Twofold(*host[fn]), out=hout[fn])
        torch.cuda.synchronize()
        t_e2e = max_over_ranks((time.perf_counter() - tw) / e2e_steps)
        _ = float(z.value[0])  # the result is on the host
        e2e = {"value": 2 * n * world / t_e2e, "unit": "elements/s",
               "h2d_bytes_per_step": 2 * 2 * n * 8, "d2h_bytes_per_step": 2 * 2 * n * 8,
               "ms_per_step": t_e2e * 1e3, "path": "api(64).texpm1/tlog1p(Twofold(pinned CPU tensors), out=pinned CPU tensors)"}

    # ---- parity sample + the one small NCCL reduce of error statistics
    stats = parity_sample(args, ins, outs, n, rank, world, dev)

    # ---- roofline of the dominant kernel
    dom = max(kern_ms, key=kern_ms.get)
    dom_ms = kern_ms[dom]
    ops = ALG_OPS[(dom, 64)] * n / (dom_ms * 1e-3)
    gbs = 32 * n / (dom_ms * 1e-3) / 1e9
    traffic = args.traffic
    if traffic is None:
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                rec = json.load(f).get(f"k_eval<double,{dom}>")
            if rec:  # per launch of the same size (ncu --set full capture)
                traffic = rec["traffic_bytes"] * n / rec["elements"]
        except (OSError, ValueError, KeyError):
            traffic = None
    roof = {"bound": "fp64", "kernel": f"k_eval<double,{dom}>",
            "achieved": ops / 1e12, "peak": peak[64] / 1e12, "unit": "TFLOP/s",
            "frac": ops / peak[64], "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)",
            "algorithmic_bytes": 32 * n,
            "ops_per_element": ALG_OPS[(dom, 64)], "elements_per_launch": n,
            "launch_ms": dom_ms, "peak_source": "measured tf_fma_peak, best of DADD/DMUL/DFMA chains (this GPU, this run)",
            "hbm_achieved_gbs": gbs, "hbm_peak_gbs": _peaks()["hbm_gbs"],
            "hbm_frac": gbs / _peaks()["hbm_gbs"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded shard-invariant cfg-2 generator, on device)",
            "config": {"workload": "cfg2: texpm1 + tlog1p over float64 twofolds",
                       "elements_per_function_per_gpu": n, "global_elements_per_step": 2 * n * world,
                       "parallelism": f"contiguous shards x{world}, no collective on the hot path",
                       "l2": "inputs 512 MiB/step > 126 MB L2 (no flush needed)",
                       "streams": args.streams,
                       "kernel_ms": "per-kernel launch durations from the same steps run on one stream"},
            "gpu_launches": len(HEADLINE) * args.steps,
            "kernel_ms": kern_ms,
            "clocks": clk.summary(),
            "roofline": roof,
            "fp_peak_tops": {k: v / 1e12 for k, v in peak_by_op.items()},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "per_function": per_fn,
            "siblings": siblings,
            "eft_ops": eft_rates, "cfg5": cfg5,
            "cfg1_small": small,
            "parity_sample": stats,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def parity_sample(args, ins, outs, n, rank, world, dev):
    """Check a seeded sample of each rank's outputs against the CPU oracle, then
    combine the per-rank counters with the one small all-reduce of the run
    (paper_1502_05216_b200.dist.reduce_stats; NCCL here, gloo in the tests)."""
    from oracle import oracle as O
    from oracle.compare import compare
    from paper_1502_05216_b200.dist import reduce_stats

    m = min(args.parity_sample, n)
    out = {}
    for fn, _ in HEADLINE:
        x0 = ins[fn][0][:m].cpu().numpy()
        x1 = ins[fn][1][:m].cpu().numpy()
        z0 = outs[fn][0][:m].cpu().numpy()
        z1 = outs[fn][1][:m].cpu().numpy()
        r0, r1 = O.evaluate(fn, 64, x0, x1, backend="dv")
        r = compare(z0, z1, r0, r1, 64)
        out[fn] = reduce_stats(r, device=dev)
        out[fn].pop("bad_idx", None)
        out[fn].pop("z0_ulp_hist", None)
    out["oracle"] = "CPU port, dv backend (bit-exact vs reference goldens)"
    return out


def cpu_baseline(args):
    from oracle import oracle as O
    from paper_1502_05216_b200 import workloads

    O.build()
    nt = O.default_threads()
    sample = args.ref_sample
    data = {fn: workloads.generate(workloads.CONFIGS[cfg][2], 0, sample, seed=SEED)
            for fn, cfg in HEADLINE}
    for fn, _ in HEADLINE:
        O.evaluate(fn, 64, *data[fn], backend="dv", nthreads=nt)
    t = time.perf_counter()
    for fn, _ in HEADLINE:
        O.evaluate(fn, 64, *data[fn], backend="dv", nthreads=nt)
    dt = time.perf_counter() - t
    return {"value": 2 * sample / dt, "unit": "elements/s", "cores": nt, "kind": "port",
            "sample": f"{sample} elements each of texpm1 and tlog1p (cfg-2 generator), "
                      f"C port of the reference algorithm (oracle/), {nt} threads"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--n", type=int, default=N_HEAD, help="elements per function per GPU")
    ap.add_argument("--ref-sample", type=int, default=1 << 21)
    ap.add_argument("--parity-sample", type=int, default=1 << 16)
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel (profiles/)")
    ap.add_argument("--headline-only", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the 2^30 config-5 section")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-siblings", action="store_true")
    ap.add_argument("--no-eft", action="store_true")
    ap.add_argument("--streams", type=int, default=2, choices=(1, 2),
                    help="run the step's two functions on 1 or 2 streams")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
