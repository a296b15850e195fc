"""Parity counts of every element of a config input against an oracle, chunked
(host comparator, oracle/compare.py): z0 mismatches, beyond 1 ulp, tolerance
violations, violations with z0 equal, class mismatches, z0 ulp histogram.

    python tools/parity_full.py width [log2 n] [ref|crsim] [fn ...]     (GPU box)
"""
import json
import os
import sys
from collections import Counter

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from oracle.compare import compare  # noqa: E402
from paper_1502_05216_b200 import _lib, api  # noqa: E402

width = int(sys.argv[1])
n = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 28)
which = sys.argv[3] if len(sys.argv) > 3 else "ref"
DIST = {64: {"texp": "exp64", "texpm1": "pow10_64", "tlog": "log64", "tlog1p": "pow10c_64"},
        32: {"texp": "exp32", "texpm1": "exp32", "tlog": "log32", "tlog1p": "log32"}}[width]
fns = sys.argv[4:] or list(DIST)
chunk = min(n, 1 << 24)
dt = torch.float64 if width == 64 else torch.float32
L = _lib.ensure_device(0)
res = {}
for fn in fns:
    x0 = torch.empty(n, dtype=dt, device="cuda")
    x1 = torch.empty_like(x0)
    _lib.check(L.tf_generate(_lib.DIST_CODES[DIST[fn]], 2024, 0, n, x0.data_ptr(), x1.data_ptr(),
                             None), "gen")
    z = getattr(api(width), fn)((x0, x1))
    tot, hist = Counter(), Counter()
    for lo in range(0, n, chunk):
        a0, a1 = x0[lo:lo + chunk].cpu().numpy(), x1[lo:lo + chunk].cpu().numpy()
        g0, g1 = z.value[lo:lo + chunk].cpu().numpy(), z.error[lo:lo + chunk].cpu().numpy()
        if which == "crsim":
            kw = {"backend": "fma", ("libm32" if width == 32 else "libm64"): "cr"}
        else:
            kw = {"backend": "dv"}
        r = compare(g0, g1, *O.evaluate(fn, width, a0, a1, **kw), width)
        for k in ("n", "z0_mismatch", "z0_gt1ulp", "tol_violations",
                  "tol_violations_given_z0_match", "class_mismatch"):
            tot[k] += r[k]
        hist.update(r["z0_ulp_hist"])
    res[fn] = dict(tot) | {"z0_ulp_hist": {str(k): v for k, v in sorted(hist.items())}}
    print(fn, json.dumps(res[fn]), flush=True)
    del x0, x1, z
    torch.cuda.empty_cache()
