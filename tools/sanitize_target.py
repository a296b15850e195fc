"""Small exhaustive-ish driver for compute-sanitizer: every kernel, ragged and
misaligned sizes, special inputs, the exact path forced."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_05216_b200 import _lib, api, workloads

dev = torch.device("cuda", 0)
for width in (64, 32):
    dt = torch.float64 if width == 64 else torch.float32
    for fn in ("texp", "texpm1", "tlog", "tlog1p"):
        g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"golden_{fn}_f{width}.npz"))
        x0 = torch.from_numpy(g["x0"]).to(dev); x1 = torch.from_numpy(g["x1"]).to(dev)
        lib = api(width)
        for n in (1, 3, 5, 1000, x0.numel()):
            for off in (0, 1):
                a0, a1 = x0[off:off + n], x1[off:off + n]
                if a0.numel() == 0:
                    continue
                z0 = torch.empty_like(a0); z1 = torch.empty_like(a0)
                for flags in (0, _lib.FLAG_FORCE_EXACT):
                    lib._launch(fn, a0, a1, z0, z1, a0.numel(), torch.cuda.current_stream().cuda_stream, flags)
        torch.cuda.synchronize()
print("sanitize target ok")

# every function, both widths, on raw random bit patterns (NaN, inf, subnormal
# and out-of-domain operands reach every rejected-lane path of the fast kernels)
from paper_1502_05216_b200 import FUNCTION_NAMES
rng = np.random.default_rng(5)
for width in (64, 32):
    it = np.uint64 if width == 64 else np.uint32
    ft = np.float64 if width == 64 else np.float32
    n = 4099
    b0 = rng.integers(0, np.iinfo(it).max, n, dtype=it, endpoint=True).view(ft)
    b1 = rng.integers(0, np.iinfo(it).max, n, dtype=it, endpoint=True).view(ft)
    x0 = torch.from_numpy(b0.copy()).to(dev); x1 = torch.from_numpy(b1.copy()).to(dev)
    lib = api(width)
    for fn in FUNCTION_NAMES:
        z0 = torch.empty_like(x0); z1 = torch.empty_like(x0)
        for flags in (0, _lib.FLAG_FORCE_EXACT):
            lib._launch(fn, x0, x1, z0, z1, n, torch.cuda.current_stream().cuda_stream, flags)
    torch.cuda.synchronize()
print("sanitize bit patterns ok")
