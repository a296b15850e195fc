"""End-to-end rate of the host pipeline (bench.py's e2e leg at a smaller size):
api(64).texp / .tlog on pinned host tensors with out= pinned host tensors.

    TWOFOLD_B200_LIB=... python tools/e2e_probe.py [log2 n] [reps]     (GPU box)
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import Twofold, _lib, api  # noqa: E402

n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 28)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L = _lib.ensure_device(0)
f = api(64)
host = {}
for fn, dist in (("texp", "exp64s"), ("tlog", "logu64s")):
    d0 = torch.empty(n, dtype=torch.float64, device="cuda")
    d1 = torch.empty_like(d0)
    _lib.check(L.tf_generate(_lib.DIST_CODES[dist], 2024, 0, n, d0.data_ptr(), d1.data_ptr(), None),
               "gen")
    host[fn] = (d0.cpu().pin_memory(), d1.cpu().pin_memory())
    del d0, d1
out = (torch.empty(n, dtype=torch.float64, pin_memory=True),
       torch.empty(n, dtype=torch.float64, pin_memory=True))
for fn in host:
    f.function(fn)(Twofold(*host[fn]), out=out)
t = time.perf_counter()
for _ in range(reps):
    for fn in host:
        f.function(fn)(Twofold(*host[fn]), out=out)
dt = (time.perf_counter() - t) / reps
print(f"e2e {2 * n / dt / 1e9:.3f} G elem/s, {64 * n / dt / 1e9:.1f} GB/s both directions", flush=True)
