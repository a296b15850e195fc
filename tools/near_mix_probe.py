import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1502_05216_b200 import _lib, api
L = _lib.ensure_device(0); s = torch.cuda.current_stream().cuda_stream
n = 1 << 26
x0 = torch.empty(n, dtype=torch.float64, device="cuda"); x1 = torch.empty_like(x0)
_lib.check(L.tf_generate(_lib.DIST_CODES["logu64s"], 2024, 0, n, x0.data_ptr(), x1.data_ptr(), s), "gen")
sp = x1 == 0
x0 = torch.where(sp, torch.full_like(x0, 3.0), x0); x1 = torch.where(sp, x0 * 2.0 ** -60, x1)
g = torch.Generator(device="cuda"); g.manual_seed(1)
d = (torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1) * 2.0 ** -40
n0 = 1.0 + d; n1 = n0 * (torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1) * 2.0 ** -53
z0, z1 = torch.empty_like(x0), torch.empty_like(x0)
def rate(a0, a1, reps=8):
    for _ in range(3): api(64)._launch("tlog", a0, a1, z0, z1, n, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): api(64)._launch("tlog", a0, a1, z0, z1, n, s)
    e1.record(); torch.cuda.synchronize()
    return round(n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
for frac in (0.0, 0.05, 0.5, 1.0):
    m = torch.rand(n, device="cuda", generator=g) < frac
    a0 = torch.where(m, n0, x0); a1 = torch.where(m, n1, x1)
    print(f"near-1 fraction {frac}: {rate(a0, a1)} G elem/s", flush=True)
