"""Diagnostics: GPU texp / tlog on a cfg-5 prefix of n elements against the
reference-equivalent oracle ("dv", glibc); every tolerance violation is
re-checked against the CR-sim oracle (correctly rounded libm, fma residuals)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from oracle.compare import bad_mask, compare  # noqa: E402
from paper_1502_05216_b200 import api, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
for fn, dist in (("texp", "exp64s"), ("tlog", "logu64s")):
    x0, x1 = workloads.generate(dist, 0, n, seed=2024)
    z = getattr(api(64), fn)((torch.from_numpy(x0).cuda(), torch.from_numpy(x1).cuda()))
    z0, z1 = z.value.cpu().numpy(), z.error.cpu().numpy()
    ref = O.evaluate(fn, 64, x0, x1, backend="dv")
    bad = np.nonzero(bad_mask(z0, z1, *ref, 64))[0]
    print(fn, "violations vs ref:", bad.size, flush=True)
    for i in bad[:20]:
        a, b = x0[i:i + 1], x1[i:i + 1]
        cr = O.evaluate(fn, 64, a, b, backend="fma", libm64="cr")
        fm = O.evaluate(fn, 64, a, b, backend="fma")
        print("  i", i, "x", a[0].hex(), b[0].hex(), "| gpu", z0[i].hex(), z1[i].hex(),
              "| ref", ref[0][i].hex(), ref[1][i].hex(), "| crsim", cr[0][0].hex(), cr[1][0].hex(),
              "| fma+glibc", fm[0][0].hex(), fm[1][0].hex(), flush=True)
