"""Scalar-call latency breakdown (the reference's one-element convention,
audit.py:343-349): the public API call, the bare ctypes tf_eval_host call, a
device-pointer tf_eval + synchronise, the tiny kernel's own duration, and a
one-element torch op + synchronise as the launch floor.

    python tools/scalar_probe.py            (GPU box)
"""

from __future__ import annotations

import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1502_05216_b200 import _lib, api  # noqa: E402


def per_call_us(f, reps=4000):
    for _ in range(200):
        f()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    return (time.perf_counter() - t) / reps * 1e6


def main():
    out = {}
    dev = torch.device("cuda", 0)
    L = _lib.ensure_device(0)
    args = {"texp": (1.25, 1e-17), "tlog": (3.5, 2e-17), "texpm1": (0.3, 1e-18),
            "tlog1p": (0.7, 1e-17)}
    for fn, (a, b) in args.items():
        f = getattr(api(64), fn)
        out[f"api_{fn}"] = per_call_us(lambda: f((a, b)))
        code = _lib.FN_CODES[fn]
        c0, c1, r0, r1 = (ctypes.c_double(a), ctypes.c_double(b), ctypes.c_double(),
                          ctypes.c_double())
        p0, p1, q0, q1 = (ctypes.byref(c0), ctypes.byref(c1), ctypes.byref(r0),
                          ctypes.byref(r1))
        out[f"host_{fn}"] = per_call_us(
            lambda: L.tf_eval_host(code, 64, p0, p1, q0, q1, 1, 0, None, 0))
        x0 = torch.full((1,), a, dtype=torch.float64, device=dev)
        x1 = torch.full((1,), b, dtype=torch.float64, device=dev)
        z0, z1 = torch.empty_like(x0), torch.empty_like(x1)
        s = torch.cuda.current_stream().cuda_stream

        def dev_call():
            L.tf_eval(code, 64, x0.data_ptr(), x1.data_ptr(), z0.data_ptr(), z1.data_ptr(), 1,
                      s, 0)
            torch.cuda.synchronize()

        out[f"dev_sync_{fn}"] = per_call_us(dev_call)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(50):
            L.tf_eval(code, 64, x0.data_ptr(), x1.data_ptr(), z0.data_ptr(), z1.data_ptr(), 1,
                      s, 0)
        e0.record()
        for _ in range(1000):
            L.tf_eval(code, 64, x0.data_ptr(), x1.data_ptr(), z0.data_ptr(), z1.data_ptr(), 1,
                      s, 0)
        e1.record()
        torch.cuda.synchronize()
        out[f"kernel_back_to_back_{fn}"] = e0.elapsed_time(e1) / 1000 * 1e3
    t = torch.zeros(1, device=dev)

    def torch_op():
        t.add_(1.0)
        torch.cuda.synchronize()

    out["torch_add_sync"] = per_call_us(torch_op)
    out["python_noop_call"] = per_call_us(lambda: L.tf_version())
    print(json.dumps({k: round(v, 2) for k, v in out.items()}))


def launch_cost():
    """CPU cost of one tf_eval(n=1) launch (no synchronisation) and the tiny
    kernels' device time per launch (ncu: -k regex:k_tiny)."""
    dev = torch.device("cuda", 0)
    L = _lib.ensure_device(0)
    x0 = torch.full((1,), 1.25, dtype=torch.float64, device=dev)
    x1 = torch.full((1,), 1e-17, dtype=torch.float64, device=dev)
    z0, z1 = torch.empty_like(x0), torch.empty_like(x1)
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    for fn in ("texp", "tlog", "texpm1", "tlog1p"):
        code = _lib.FN_CODES[fn]
        args = (code, 64, x0.data_ptr(), x1.data_ptr(), z0.data_ptr(), z1.data_ptr(), 1, s, 0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(200):
            L.tf_eval(*args)
        res[f"launch_cpu_{fn}"] = (time.perf_counter() - t) / 200 * 1e6
        torch.cuda.synchronize()
    print(json.dumps({k: round(v, 2) for k, v in res.items()}))


if __name__ == "__main__":
    main()
    if os.environ.get("LAUNCH_COST"):
        launch_cost()
