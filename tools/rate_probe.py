"""Kernel rates outside bench.py, in bench.py's per-function order (diagnostics)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib, api
L = _lib.ensure_device(0)
sp = torch.cuda.current_stream().cuda_stream


def gen(dist, n, dt):
    x0 = torch.empty(n, dtype=dt, device="cuda"); x1 = torch.empty_like(x0)
    _lib.check(L.tf_generate(_lib.DIST_CODES[dist], 2024, 0, n, x0.data_ptr(), x1.data_ptr(), sp), "gen")
    return x0, x1


def rate(fn, w, dist, n, reps=10):
    a0, a1 = gen(dist, n, torch.float32 if w == 32 else torch.float64)
    z0, z1 = torch.empty_like(a0), torch.empty_like(a0)
    lib = api(w)
    for _ in range(3):
        lib._launch(fn, a0, a1, z0, z1, n, sp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib._launch(fn, a0, a1, z0, z1, n, sp)
    e1.record(); torch.cuda.synchronize()
    return round(n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)


order = [("texp", 64, "exp64s", 1 << 28), ("tlog", 64, "logu64s", 1 << 28),
         ("texp", 64, "exp64", 1 << 26), ("texpm1", 64, "pow10_64", 1 << 24), ("tlog", 64, "log64", 1 << 26),
         ("tlog1p", 64, "pow10c_64", 1 << 24), ("texp", 32, "exp32", 1 << 28), ("texpm1", 32, "exp32", 1 << 28),
         ("tlog", 32, "log32", 1 << 28), ("tlog1p", 32, "log32", 1 << 28)]
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    print({f"{fn}_f{w}_{d}": rate(fn, w, d, n) for fn, w, d, n in order}, flush=True)
