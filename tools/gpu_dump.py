"""Dump GPU outputs for golden vectors and config samples (for offline analysis
against the CPU oracle in the build container)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1502_05216_b200 import _lib, api, workloads  # noqa: E402

dev = torch.device("cuda", 0)
out = os.path.join(ROOT, "gpurun_out")
os.makedirs(out, exist_ok=True)
N = int(os.environ.get("DUMP_N", 1 << 18))


def run(fn, width, x0, x1, flags=0):
    lib = api(width)
    t0 = torch.from_numpy(np.ascontiguousarray(x0)).to(dev)
    t1 = torch.from_numpy(np.ascontiguousarray(x1)).to(dev)
    z = lib._device(fn, t0, t1, flags=flags)
    torch.cuda.synchronize()
    return z.value.cpu().numpy(), z.error.cpu().numpy()


res = {}
CFGS = os.environ.get("DUMP_CFGS")
GOLD = os.environ.get("DUMP_GOLDEN", "1") == "1"
for width in ((64, 32) if GOLD else ()):
    for fn in ("texp", "texpm1", "tlog", "tlog1p"):
        g = np.load(os.path.join(ROOT, "tests", "golden", f"golden_{fn}_f{width}.npz"))
        a0, a1 = run(fn, width, g["x0"], g["x1"])
        b0, b1 = run(fn, width, g["x0"], g["x1"], _lib.FLAG_FORCE_EXACT)
        res[f"g_{fn}_{width}"] = np.stack([a0, a1, b0, b1])
for cfg, (fn, width, dist, _) in workloads.CONFIGS.items():
    if CFGS and cfg not in CFGS.split(","):
        continue
    x0, x1 = workloads.generate(dist, 0, N, seed=1)
    a0, a1 = run(fn, width, x0, x1)
    b0, b1 = run(fn, width, x0, x1, _lib.FLAG_FORCE_EXACT)
    res[f"c_{cfg}"] = np.stack([a0, a1, b0, b1])
np.savez_compressed(os.path.join(out, "dump.npz"), **res)
print("dumped", len(res))
