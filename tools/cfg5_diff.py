"""Diagnostics: GPU texp / tlog on a cfg-5 prefix against the CR-sim and the
reference-equivalent ("dv", glibc) oracles; prints every violating element."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from oracle.compare import bad_mask, compare  # noqa: E402
from paper_1502_05216_b200 import api, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
for fn, dist in (("texp", "exp64s"), ("tlog", "logu64s")):
    x0, x1 = workloads.generate(dist, 0, n, seed=2024)
    z = getattr(api(64), fn)((torch.from_numpy(x0).cuda(), torch.from_numpy(x1).cuda()))
    z0, z1 = z.value.cpu().numpy(), z.error.cpu().numpy()
    cr = O.evaluate(fn, 64, x0, x1, backend="fma", libm64="cr")
    ref = O.evaluate(fn, 64, x0, x1, backend="dv")
    for name, r in (("crsim", cr), ("ref", ref)):
        c = compare(z0, z1, *r, 64)
        print(fn, name, {k: v for k, v in c.items() if k != "bad_idx"})
        for i in np.nonzero(bad_mask(z0, z1, *r, 64))[0][:10]:
            print("   ", i, x0[i].hex(), x1[i].hex(), "gpu", z0[i].hex(), z1[i].hex(),
                  "oracle", r[0][i].hex(), r[1][i].hex())
