"""Every element of a 2^k config input against the oracle, for any of the
twenty functions, counted on the device (tf_compare; the oracle runs on the
host in 2^24-element chunks).  binary64 against the reference-equivalent oracle
("dv" residuals, glibc value parts); binary32 against CR-sim (fma residuals,
correctly rounded value parts).  Dotted functions get x1 = 0 (plain argument).

    python tools/parity_device.py width [log2 n] [fn[:dist] ...]      (GPU box)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1502_05216_b200 import DOTTED_ARG, FUNCTION_NAMES, _lib, api, family_of  # noqa: E402

width = int(sys.argv[1])
n = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 28)
fns = sys.argv[3:] or list(FUNCTION_NAMES)
DIST = {64: {"exp": "exp64", "expm1": "pow10_64", "log": "log64", "log1p": "pow10c_64"},
        32: {"exp": "exp32", "expm1": "exp32", "log": "log32", "log1p": "log32"}}[width]
chunk = min(n, 1 << 24)
dt = torch.float64 if width == 64 else torch.float32
rel, guard = (2.0 ** -95, 2 * 2.0 ** -1074) if width == 64 else (2.0 ** -42, 2 * 2.0 ** -149)
L = _lib.ensure_device(0)
for spec in fns:
    fn, _, dist = spec.partition(":")
    x0 = torch.empty(n, dtype=dt, device="cuda")
    x1 = torch.empty_like(x0)
    _lib.check(L.tf_generate(_lib.DIST_CODES[dist or DIST[family_of(fn)]], 2024, 0, n,
                             x0.data_ptr(), x1.data_ptr(), None), "gen")
    dotted = fn in DOTTED_ARG
    if dotted:
        x1.zero_()
    f = getattr(api(width), fn)
    z = f(x0) if dotted else f((x0, x1))
    st = torch.zeros(6, dtype=torch.int64, device="cuda")
    for lo in range(0, n, chunk):
        a0, a1 = x0[lo:lo + chunk].cpu().numpy(), x1[lo:lo + chunk].cpu().numpy()
        kw = {"backend": "dv"} if width == 64 else {"backend": "fma", "libm32": "cr"}
        r0, r1 = O.evaluate(fn, width, a0, a1, **kw)
        t0, t1 = torch.from_numpy(r0).cuda(), torch.from_numpy(r1).cuda()
        _lib.check(L.tf_compare(width, z.value[lo:].data_ptr(), z.error[lo:].data_ptr(),
                                t0.data_ptr(), t1.data_ptr(), chunk, rel, guard, st.data_ptr(),
                                None), "tf_compare")
    torch.cuda.synchronize()
    c = st.tolist()
    print(json.dumps({"fn": fn, "dist": dist or DIST[family_of(fn)], "width": width, "n": c[0], "z0_mismatch": c[1], "z0_gt1ulp": c[2],
                      "tol_violations": c[3], "class_mismatch": c[4], "z1_bit_mismatch": c[5]}),
          flush=True)
    del x0, x1, z
    torch.cuda.empty_cache()
