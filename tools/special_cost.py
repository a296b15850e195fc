"""Cost of config 5's 1% special values: texp / tlog binary64 on the cfg-5 inputs
and on the same inputs with every special replaced by an ordinary element of the
same distribution (texp: exp64 with the same seed, i.e. the value the position
would hold without the special; tlog: the neighbouring element).

    python tools/special_cost.py [log2 n]      (GPU box)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib, api  # noqa: E402

L = _lib.ensure_device(0)
sp = torch.cuda.current_stream().cuda_stream
n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 28)


def gen(dist):
    x0 = torch.empty(n, dtype=torch.float64, device="cuda")
    x1 = torch.empty_like(x0)
    _lib.check(L.tf_generate(_lib.DIST_CODES[dist], 2024, 0, n, x0.data_ptr(), x1.data_ptr(), sp),
               "gen")
    return x0, x1


def rate(fn, a0, a1, reps=8):
    z0, z1 = torch.empty_like(a0), torch.empty_like(a0)
    lib = api(64)
    for _ in range(3):
        lib._launch(fn, a0, a1, z0, z1, n, sp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib._launch(fn, a0, a1, z0, z1, n, sp)
    e1.record()
    torch.cuda.synchronize()
    return n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


for rnd in range(2):
    s0, s1 = gen("exp64s")
    c0, c1 = gen("exp64")
    r_s, r_c = rate("texp", s0, s1), rate("texp", c0, c1)
    print(f"texp f64: specials {(s0 != c0).float().mean().item():.4f}  cfg5 {r_s:.1f}  "
          f"without specials {r_c:.1f} G elem/s  ({100 * (1 - r_s / r_c):.1f}% cost)", flush=True)
    del s0, s1, c0, c1
    s0, s1 = gen("logu64s")
    sp_mask = s1 == 0
    c0, c1 = s0.clone(), s1.clone()
    c0[sp_mask] = torch.roll(s0, 1)[sp_mask]
    c1[sp_mask] = torch.roll(s1, 1)[sp_mask]
    c0[sp_mask & (c1 == 0)] = 3.0
    r_s, r_c = rate("tlog", s0, s1), rate("tlog", c0, c1)
    print(f"tlog f64: specials {sp_mask.float().mean().item():.4f}  cfg5 {r_s:.1f}  "
          f"without specials {r_c:.1f} G elem/s  ({100 * (1 - r_s / r_c):.1f}% cost)", flush=True)
    del s0, s1, c0, c1
