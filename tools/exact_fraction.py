"""Fraction of elements each kernel sends to the rare-element drain (admission
band rejects) and the fraction that reaches the exact path, per config."""
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
    fr = []
    for flags in (_lib.FLAG_COUNT_EXACT | _lib.FLAG_MARK_EXACT, _lib.FLAG_COUNT_EXACT):
        L.tf_exact_count(ctypes.byref(c), 1)
        api(w)._launch(fn, x0, x1, z0, z1, n, 0, flags)
        torch.cuda.synchronize()
        L.tf_exact_count(ctypes.byref(c), 1)
        fr.append(c.value / n)
    print(f"{cfg:18s} drained {fr[0]:.5f}  exact-path {fr[1]:.5f}")
