"""Golden vectors for the element-wise EFT / twofold arithmetic ops, made by
RUNNING the reference's own eft.py / eft32.py (pkg/src/twofold) here:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_eft_golden.py

For each op, lane and residual backend: seeded random operands over many
binades (both signs, near-cancelling pairs, subnormals, values beyond the
split threshold) plus a special-value grid.  Inputs where the reference
raises (fma_sim's debug precondition assert) are dropped.  Output:
tests/golden/eft_golden.npz, keys "<op>_<width>_<backend>_{a0,a1,b0,b1,z0,z1}".
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OPS = ("fast_two_sum", "two_sum", "two_diff", "two_prod", "split", "renorm_fast", "renorm",
       "t_add", "t_add_d", "t_mul", "t_mul_d", "t_div", "t_sqrt")
N_RAND = 1000


def operands(width: int, rng: np.random.Generator, n: int):
    dt = np.float32 if width == 32 else np.float64
    p, emax, emin = (24, 127, -149) if width == 32 else (53, 1023, -1074)
    e = rng.integers(emin + p, emax, n)
    m = rng.uniform(1.0, 2.0, n) * rng.choice([-1.0, 1.0], n)
    a = np.ldexp(m, e).astype(dt)
    # b: independent, near-cancelling, or a small coupled-like partner
    kind = rng.integers(0, 3, n)
    e2 = np.where(kind == 0, rng.integers(emin + p, emax, n), e - rng.integers(0, p + 8, n))
    b = np.ldexp(rng.uniform(1.0, 2.0, n) * rng.choice([-1.0, 1.0], n), e2)
    b = np.where(kind == 1, -a.astype(np.float64) * (1 + rng.uniform(-1, 1, n) * 2.0 ** -20), b)
    b = b.astype(dt)
    # tails: |a1| ~ ulp(a0) scale
    a1 = (a.astype(np.float64) * rng.uniform(-1, 1, n) * 2.0 ** -p).astype(dt)
    b1 = (b.astype(np.float64) * rng.uniform(-1, 1, n) * 2.0 ** -p).astype(dt)
    return a, a1, b, b1


def specials(width: int):
    if width == 64:
        big, tiny, mx = 2.0 ** 1000, 5e-324, 1.7976931348623157e308
    else:
        big, tiny, mx = 2.0 ** 120, 2.0 ** -149, float(np.finfo(np.float32).max)
    return [0.0, -0.0, 1.0, -1.0, 3.0, 0.1, tiny, -tiny, big, -big, mx, -mx, math.inf,
            -math.inf, math.nan, 1e-30, 2.0 ** -60]


def exact_fma64(x: float, y: float, z: float) -> float:
    """fl(x*y + z), one rounding: exact rational arithmetic, then Python's
    correctly rounded int/int -> float conversion.  Stands in for math.fma
    (Python >= 3.13) / gmpy2, both absent here, which the reference's binary64
    "fma" backend calls (_fp.py:95-109)."""
    from fractions import Fraction

    if not (math.isfinite(x) and math.isfinite(y) and math.isfinite(z)):
        return x * y + z
    r = Fraction(x) * Fraction(y) + Fraction(z)
    if r == 0:
        return x * y + z          # exact zero: IEEE sign rules of the unfused form
    return r.numerator / r.denominator


def main():
    from twofold import eft, eft32
    from twofold.eft import Twofold

    eft.fma64 = exact_fma64

    out = {}
    rng = np.random.default_rng(20241020)
    for width in (64, 32):
        mod = eft if width == 64 else eft32
        dt = np.float32 if width == 32 else np.float64
        a, a1, b, b1 = operands(width, rng, N_RAND)
        sp = specials(width)
        g = np.array([(x, y) for x in sp for y in sp], dtype=np.float64)
        a = np.concatenate([a, g[:, 0].astype(dt)])
        b = np.concatenate([b, g[:, 1].astype(dt)])
        a1 = np.concatenate([a1, np.zeros(len(g), dt)])
        b1 = np.concatenate([b1, (g[:, 1] * 2.0 ** -40).astype(dt)])
        for backend in ("fma", "dv"):
            ar = mod.arith(backend)
            fns = {
                "fast_two_sum": lambda x0, x1, y0, y1: mod.fast_two_sum(x0, y0),
                "two_sum": lambda x0, x1, y0, y1: mod.two_sum(x0, y0),
                "two_diff": lambda x0, x1, y0, y1: mod.two_diff(x0, y0),
                "two_prod": lambda x0, x1, y0, y1: (mod.two_prod_fma if backend == "fma"
                                                    else mod.two_prod_dv)(x0, y0),
                "split": lambda x0, x1, y0, y1: mod.split(x0),
                "renorm_fast": lambda x0, x1, y0, y1: mod.renorm_fast(Twofold(x0, x1)),
                "renorm": lambda x0, x1, y0, y1: mod.renorm(Twofold(x0, x1)),
                "t_add": lambda x0, x1, y0, y1: ar.t_add(Twofold(x0, x1), Twofold(y0, y1)),
                "t_add_d": lambda x0, x1, y0, y1: ar.t_add_d(Twofold(x0, x1), y0),
                "t_mul": lambda x0, x1, y0, y1: ar.t_mul(Twofold(x0, x1), Twofold(y0, y1)),
                "t_mul_d": lambda x0, x1, y0, y1: ar.t_mul_d(Twofold(x0, x1), y0),
                "t_div": lambda x0, x1, y0, y1: ar.t_div(Twofold(x0, x1), Twofold(y0, y1)),
                "t_sqrt": lambda x0, x1, y0, y1: ar.t_sqrt(Twofold(abs(x0), x1)),
            }
            for op in OPS:
                keep, z0, z1 = [], [], []
                for i in range(a.size):
                    x0, x1, y0, y1 = float(a[i]), float(a1[i]), float(b[i]), float(b1[i])
                    try:
                        r = fns[op](x0, x1, y0, y1)
                    except (AssertionError, OverflowError, ValueError):
                        continue
                    keep.append(i)
                    z0.append(r[0])
                    z1.append(r[1])
                k = np.array(keep, dtype=np.int64)
                key = f"{op}_{width}_{backend}"
                sa0 = np.abs(a[k]) if op == "t_sqrt" else a[k]
                out[key + "_a0"], out[key + "_a1"] = sa0, a1[k]
                out[key + "_b0"], out[key + "_b1"] = b[k], b1[k]
                out[key + "_z0"] = np.array(z0, dtype=dt)
                out[key + "_z1"] = np.array(z1, dtype=dt)
                print(key, len(keep), file=sys.stderr)
    np.savez_compressed(os.path.join(HERE, "eft_golden.npz"), **out)


if __name__ == "__main__":
    main()
