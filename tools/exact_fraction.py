"""Fraction of elements each kernel routes through the exact path, per config."""
import os, sys, ctypes
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib, api, workloads
L = _lib.ensure_device(0)
n = 1 << 22
for cfg, (fn, w, dist, _) in workloads.CONFIGS.items():
    dt = torch.float64 if w == 64 else torch.float32
    x0 = torch.empty(n, dtype=dt, device="cuda"); x1 = torch.empty_like(x0)
    _lib.check(L.tf_generate(_lib.DIST_CODES[dist], 2024, 0, n, x0.data_ptr(), x1.data_ptr(), None), "gen")
    z0 = torch.empty_like(x0); z1 = torch.empty_like(x0)
    c = ctypes.c_ulonglong(0)
    L.tf_exact_count(ctypes.byref(c), 1)
    api(w)._launch(fn, x0, x1, z0, z1, n, 0, _lib.FLAG_COUNT_EXACT)
    torch.cuda.synchronize()
    L.tf_exact_count(ctypes.byref(c), 1)
    print(f"{cfg:18s} exact-path fraction {c.value / n:.5f}")
