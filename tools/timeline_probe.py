"""Per-warp timeline of one k_eval launch (diagnostics build with TF_TIMELINE):
start, tables staged, main loop done, end (globaltimer ns) and drains per warp.

    make -C paper_1502_05216_b200/csrc timeline
    TWOFOLD_B200_LIB=paper_1502_05216_b200/lib/diag/libtwofold_b200_tl.so \\
        python tools/timeline_probe.py tlog1p 64 2 [n]
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1502_05216_b200 import _lib, api  # noqa: E402

fn, width, dist = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 24
L = _lib.ensure_device(0)
dev = torch.device("cuda", 0)
dt = torch.float64 if width == 64 else torch.float32
x0 = torch.empty(n, dtype=dt, device=dev)
x1 = torch.empty_like(x0)
_lib.check(L.tf_generate(dist, 2024, 0, n, x0.data_ptr(), x1.data_ptr(), None), "gen")
z0, z1 = torch.empty_like(x0), torch.empty_like(x0)
lib = api(width)
for _ in range(3):
    lib._launch(fn, x0, x1, z0, z1, n, None)
torch.cuda.synchronize()
NW = 1 << 16
t = np.zeros(4 * NW, np.uint64)
sm = np.zeros(NW, np.uint32)
L.tf_timeline.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
_lib.check(L.tf_timeline(t.ctypes.data, sm.ctypes.data, NW), "timeline")
t = t.reshape(-1, 4).astype(np.int64)
used = t[:, 0] > 0
t, sm = t[used], sm[used]
t0 = t[:, 0].min()
t = t - t0
drains = sm >> 16
smid = sm & 0xffff
print(f"{fn} f{width} n={n}: warps={len(t)} kernel span {t[:, 3].max()/1e3:.1f} us")
for name, col in (("start", 0), ("tables", 1), ("loop end", 2), ("end", 3)):
    c = t[:, col] / 1e3
    print(f"  {name:9s} min {c.min():7.1f}  p50 {np.median(c):7.1f}  p99 {np.percentile(c, 99):7.1f}  max {c.max():7.1f} us")
print(f"  table staging per warp: p50 {np.median(t[:,1]-t[:,0])/1e3:.2f} us")
print(f"  tail (end - loop end): p50 {np.median(t[:,3]-t[:,2])/1e3:.2f} us, max {(t[:,3]-t[:,2]).max()/1e3:.2f} us")
print(f"  drains per warp: mean {drains.mean():.2f}, max {drains.max()}")
# active warps over time
span = t[:, 3].max()
grid = np.linspace(0, span, 41)
act = [(np.sum((t[:, 0] <= g) & (t[:, 3] > g))) for g in grid]
print("  active warps over time (per 2.5% of span):", act)
per_sm = np.bincount(smid, minlength=smid.max() + 1)
print(f"  warps per SM: min {per_sm.min()} max {per_sm.max()} SMs used {np.count_nonzero(per_sm)}")
