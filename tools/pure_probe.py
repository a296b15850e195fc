"""tlog1p binary32 on config 4's mix, on all-in-band and on all-out-of-band inputs
(the ceiling of class sorting).  Compare the default build with
    bash tools/build_variant.sh pure1 -DTF_T1P32_PURE=1   (in-band-only pipeline)
    bash tools/build_variant.sh pure2 -DTF_T1P32_PURE=2   (out-of-band-only pipeline)
    TWOFOLD_B200_LIB=paper_1502_05216_b200/lib/var/pure1.so python tools/pure_probe.py
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1502_05216_b200 import _lib, api
L = _lib.ensure_device(0)
s = torch.cuda.current_stream().cuda_stream
n = 1 << 28
x0 = torch.empty(n, dtype=torch.float32, device="cuda"); x1 = torch.empty_like(x0)
_lib.check(L.tf_generate(_lib.DIST_CODES["log32"], 2024, 0, n, x0.data_ptr(), x1.data_ptr(), s), "gen")
inb0 = torch.where(x0 > 1, 1.0 / x0, x0); inb1 = inb0 * 2.0 ** -30
out0 = torch.where(x0 <= 1, 1.0 / x0, x0); out0 = torch.where(out0 == 1.0, torch.full_like(out0, 3.0), out0); out1 = out0 * 2.0 ** -30
z0, z1 = torch.empty_like(x0), torch.empty_like(x0)
lib = api(32)
def rate(a0, a1, reps=8):
    for _ in range(3): lib._launch("tlog1p", a0, a1, z0, z1, n, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): lib._launch("tlog1p", a0, a1, z0, z1, n, s)
    e1.record(); torch.cuda.synchronize()
    return round(n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
print(os.environ.get("TWOFOLD_B200_LIB", "default"), {"mixed": rate(x0, x1), "all_in": rate(inb0, inb1), "all_out": rate(out0, out1)}, flush=True)
