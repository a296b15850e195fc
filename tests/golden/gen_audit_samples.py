"""Golden audit sample streams made by RUNNING the reference's own
gen_samples (pkg/src/twofold/audit.py:130-158) in this build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_audit_samples.py

audit.py imports the gmpy2-backed oracle module at import time although
gen_samples never touches it; gmpy2 is absent here, so an empty stand-in
module is registered first (nothing of it is called).  Writes
tests/golden/audit_samples.npz: for every (function, width), the first N
samples of seed 42 (the CLI default) and of the bench pool seed 0xB0B.
"""

from __future__ import annotations

import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
N = 256


def main():
    stub = types.ModuleType("gmpy2")
    stub.mpfr = object
    stub.ieee = lambda *a, **k: None
    stub.context = lambda *a, **k: None
    sys.modules.setdefault("gmpy2", stub)
    from twofold import audit, explog

    out = {}
    for width in (64, 32):
        for fn in explog.FUNCTION_NAMES:
            for seed in (42, 0xB0B):
                spec = audit.SampleSpec(fn=fn, width=width, count=N, seed=seed)
                ts = list(audit.gen_samples(spec))
                dt = np.float64 if width == 64 else np.float32
                out[f"{fn}_{width}_{seed}_x0"] = np.array([t[0] for t in ts], dtype=dt)
                out[f"{fn}_{width}_{seed}_x1"] = np.array([t[1] for t in ts], dtype=dt)
    np.savez_compressed(os.path.join(HERE, "audit_samples.npz"), **out)
    print(f"wrote {len(out)} arrays", file=sys.stderr)


if __name__ == "__main__":
    main()
