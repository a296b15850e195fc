"""Cost of config 3's 5% near-1 elements in tlog binary64 (and binary32 tlog on the
same idea): the kernel on log64 against the same inputs with the near-1 elements
(|y0 - 1| < 2^-20) replaced by 3.0.

    python tools/near1_cost.py      (GPU box)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib, api  # noqa: E402

L = _lib.ensure_device(0)
s = torch.cuda.current_stream().cuda_stream
n = 1 << 26
x0 = torch.empty(n, dtype=torch.float64, device="cuda")
x1 = torch.empty_like(x0)
_lib.check(L.tf_generate(_lib.DIST_CODES["log64"], 2024, 0, n, x0.data_ptr(), x1.data_ptr(), s), "gen")
near = (x0 - 1).abs() < 2.0 ** -20
c0 = torch.where(near, torch.full_like(x0, 3.0), x0)
c1 = torch.where(near, torch.zeros_like(x1), x1)
# the same, but each near-1 element replaced by an ordinary neighbour (same data mix)
d0, d1 = x0.clone(), x1.clone()
for sh in (1, 2, 3, 5, 7):
    m = (d0 - 1).abs() < 2.0 ** -20
    d0 = torch.where(m, torch.roll(x0, sh), d0)
    d1 = torch.where(m, torch.roll(x1, sh), d1)
z0, z1 = torch.empty_like(x0), torch.empty_like(x0)


def rate(a0, a1, reps=10):
    for _ in range(3):
        api(64)._launch("tlog", a0, a1, z0, z1, n, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        api(64)._launch("tlog", a0, a1, z0, z1, n, s)
    e1.record()
    torch.cuda.synchronize()
    return n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


print(f"near-1 fraction {near.float().mean().item():.4f}: log64 {rate(x0, x1):.1f}, "
      f"near-1 replaced by 3.0 {rate(c0, c1):.1f}, by neighbours "
      f"({((d0 - 1).abs() < 2.0 ** -20).float().mean().item():.5f} left) {rate(d0, d1):.1f} "
      f"G elem/s", flush=True)
