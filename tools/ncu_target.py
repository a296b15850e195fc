"""Small driver for ncu: generate one config on device and launch the kernel(s).
usage: python tools/ncu_target.py texpm1:64:pow10_64 tlog1p:64:pow10c_64 [--n 16777216] [--reps 3]"""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib, api

ap = argparse.ArgumentParser()
ap.add_argument("specs", nargs="+")
ap.add_argument("--n", type=int, default=1 << 24)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda", 0)
L = _lib.ensure_device(0)
for spec in a.specs:
    fn, w, dist = spec.split(":")
    w = int(w)
    dt = torch.float64 if w == 64 else torch.float32
    x0 = torch.empty(a.n, dtype=dt, device=dev); x1 = torch.empty_like(x0)
    _lib.check(L.tf_generate(_lib.DIST_CODES[dist], 2024, 0, a.n, x0.data_ptr(), x1.data_ptr(), None), "gen")
    z0 = torch.empty_like(x0); z1 = torch.empty_like(x0)
    lib = api(w)
    for _ in range(a.reps):
        lib._launch(fn, x0, x1, z0, z1, a.n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
print("ok")
