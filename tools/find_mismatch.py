"""Find the elements where the GPU kernel's z0 differs from an oracle on a full
config input (2^24-element chunks, host comparison), and print them.

    python tools/find_mismatch.py fn width dist [log2 n] [oracle: ref|crsim]   (GPU box)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1502_05216_b200 import _lib, api  # noqa: E402

fn, width, dist = sys.argv[1], int(sys.argv[2]), sys.argv[3]
n = 1 << int(sys.argv[4] if len(sys.argv) > 4 else 28)
which = sys.argv[5] if len(sys.argv) > 5 else "crsim"
chunk = min(n, 1 << 24)
dt = torch.float64 if width == 64 else torch.float32
L = _lib.ensure_device(0)
x0 = torch.empty(n, dtype=dt, device="cuda")
x1 = torch.empty_like(x0)
_lib.check(L.tf_generate(_lib.DIST_CODES[dist], 2024, 0, n, x0.data_ptr(), x1.data_ptr(), None), "gen")
z = getattr(api(width), fn)((x0, x1))
torch.cuda.synchronize()
out = []
for lo in range(0, n, chunk):
    a0, a1 = x0[lo:lo + chunk].cpu().numpy(), x1[lo:lo + chunk].cpu().numpy()
    g0, g1 = z.value[lo:lo + chunk].cpu().numpy(), z.error[lo:lo + chunk].cpu().numpy()
    if which == "crsim":
        kw = {"backend": "fma", "libm32": "cr"} if width == 32 else {"backend": "fma", "libm64": "cr"}
    else:
        kw = {"backend": "dv"}
    r0, r1 = O.evaluate(fn, width, a0, a1, **kw)
    bad = np.nonzero((g0.view(np.uint32 if width == 32 else np.uint64) !=
                      r0.view(np.uint32 if width == 32 else np.uint64)) &
                     ~(np.isnan(g0) & np.isnan(r0)))[0]
    if os.environ.get("TOL"):       # tolerance violations / class mismatches instead
        from oracle.compare import compare
        bad = np.array(compare(g0, g1, r0, r1, width)["bad_idx"], dtype=np.int64)
    for i in bad[:20]:
        out.append({"index": int(lo + i), "x0": float(a0[i]).hex(), "x1": float(a1[i]).hex(),
                    "gpu": [float(g0[i]).hex(), float(g1[i]).hex()],
                    "oracle": [float(r0[i]).hex(), float(r1[i]).hex()]})
print(json.dumps(out, indent=1))
