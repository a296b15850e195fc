"""Eager rate of back-to-back launches at small sizes (the per-launch fixed cost
and the partial last pass of the persistent grid), several functions.

    TWOFOLD_B200_LIB=... python tools/small_probe.py      (GPU box)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib, api  # noqa: E402

L = _lib.ensure_device(0)
s = torch.cuda.current_stream().cuda_stream
out = {}
for fn, w, dist in (("texp", 64, "exp64"), ("tlog", 64, "log64"), ("texp", 32, "exp32"),
                    ("tlog1p", 32, "log32")):
    dt = torch.float64 if w == 64 else torch.float32
    for k in (20, 22, 24, 26):
        n = 1 << k
        a0 = torch.empty(n, dtype=dt, device="cuda")
        a1 = torch.empty_like(a0)
        _lib.check(L.tf_generate(_lib.DIST_CODES[dist], 2024, 0, n, a0.data_ptr(), a1.data_ptr(),
                                 s), "gen")
        z0, z1 = torch.empty_like(a0), torch.empty_like(a0)
        lib = api(w)
        reps = max(5, (1 << 26) // n)
        for _ in range(3):
            lib._launch(fn, a0, a1, z0, z1, n, s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            lib._launch(fn, a0, a1, z0, z1, n, s)
        e1.record()
        torch.cuda.synchronize()
        out[f"{fn}{w}_2^{k}"] = round(n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
print(out, flush=True)
