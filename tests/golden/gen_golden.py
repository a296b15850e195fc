"""Generate golden vectors by RUNNING the reference package (this container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

For each (function, width) it evaluates the reference's own public API
(``twofold.api(width).<fn>((x0, x1))``, explog.py:115-317) element by element on

  * a seeded sample of the BASELINE.json config distribution
    (paper_1502_05216_b200.workloads.generate, global indices [0, N_CFG)),
  * a special-class grid x0 x x1,
  * seeded edge samples (under/overflow bands, ln2 / 0.5 / 2 / -1 band edges,
    subnormals, near-one cancellation),

and stores x0, x1, z0, z1 plus provenance in tests/golden/golden_<fn>_f<w>.npz.
The reference backend in this image is "dv" (no gmpy2, no math.fma).
These fixtures pin the CPU oracle (tests/test_oracle_golden.py) and the CUDA
kernels (tests/test_gpu_parity.py); /root/reference is never read at test time.
"""

from __future__ import annotations

import json
import math
import os
import platform
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.normpath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from paper_1502_05216_b200.workloads import generate  # noqa: E402

N_CFG = 3000
N_EDGE = 1500
SEED = 20241017

DIST = {
    ("texp", 64): "exp64", ("texpm1", 64): "pow10_64", ("tlog", 64): "log64",
    ("tlog1p", 64): "pow10c_64",
    ("texp", 32): "exp32", ("texpm1", 32): "exp32", ("tlog", 32): "log32",
    ("tlog1p", 32): "log32",
}

INF, NAN = math.inf, math.nan


def special_x0(fn: str, width: int) -> list[float]:
    if width == 64:
        lo = float.fromhex("-0x1.74385446d71c4p+9")
        hi = float.fromhex("0x1.62e42fefa39f0p+9")
        tiny, dmax, mn = 5e-324, 1.7976931348623157e308, 2.2250738585072014e-308
        ln2 = float.fromhex("0x1.62e42fefa39efp-1")
    else:
        lo = float.fromhex("-0x1.9d1da0p+6")
        hi = float.fromhex("0x1.62e430p+6")
        tiny, dmax, mn = 2.0 ** -149, float(np.finfo(np.float32).max), 2.0 ** -126
        ln2 = float.fromhex("0x1.62e430p-1")
    nx = (lambda a, b: float(np.nextafter(np.float32(a), np.float32(b)))) if width == 32 \
        else math.nextafter
    base = [0.0, -0.0, tiny, -tiny, mn, -mn, mn * 0.75, 1.0, -1.0, 0.5, 2.0, 3.0, -3.0,
            INF, -INF, NAN, dmax, -dmax, 1e-30, -1e-30, 0.25, 1e-5, -1e-5]
    if fn in ("texp", "texpm1"):
        base += [lo, nx(lo, -INF), nx(lo, INF), hi, nx(hi, INF), nx(hi, -INF),
                 ln2, -ln2, nx(ln2, INF), nx(-ln2, -INF), 50.0, -50.0, 700.0 if width == 64 else 80.0,
                 -700.0 if width == 64 else -80.0]
        if width == 64:
            base += [709.782712893384, -745.13, -708.40, -720.0, 1e-300]
        else:
            base += [88.7, -103.0, -87.5, -95.0]
    else:
        base += [nx(1.0, 0.0), nx(1.0, 2.0), nx(0.5, 0.0), nx(2.0, 3.0), -0.5, nx(-0.5, -1.0),
                 nx(-1.0, 0.0), nx(-1.0, -2.0), 1e-300 if width == 64 else 1e-38, 10.0, 1e30]
    return base


def special_x1(x0: float, width: int) -> list[float]:
    tiny = 5e-324 if width == 64 else 2.0 ** -149
    p = 53 if width == 64 else 24
    small = x0 * 2.0 ** -(p + 7) if math.isfinite(x0) else 0.0
    return [0.0, -0.0, small, -small, tiny, INF, -INF, NAN, 1e-20 if width == 64 else 1e-12, -1.0]


def edge_x0(fn: str, width: int, rng: np.random.Generator, n: int) -> np.ndarray:
    if width == 64:
        if fn == "texp":
            bands = [(-745.2, -697.0), (700.0, 709.79), (-1e-3, 1e-3), (-30.0, 30.0)]
        elif fn == "texpm1":
            bands = [(-0.7, 0.7), (0.69, 0.697), (-0.697, -0.69), (-745.2, -30.0), (1.0, 709.79)]
        elif fn == "tlog":
            bands = [(0.45, 0.55), (1.9, 2.1), (1 - 1e-6, 1 + 1e-6), (1e-320, 1e-300), (1e300, 1.7e308)]
        else:
            bands = [(-1.0 + 1e-15, -0.99), (-0.51, -0.49), (0.99, 1.01), (-1e-9, 1e-9), (1.0, 1e6)]
    else:
        if fn == "texp":
            bands = [(-103.3, -87.0), (80.0, 88.72), (-1e-3, 1e-3), (-10.0, 10.0)]
        elif fn == "texpm1":
            bands = [(-0.7, 0.7), (0.69, 0.697), (-0.697, -0.69), (-103.3, -10.0), (1.0, 88.72)]
        elif fn == "tlog":
            bands = [(0.45, 0.55), (1.9, 2.1), (1 - 1e-3, 1 + 1e-3), (1e-45, 1e-38), (1e30, 3e38)]
        else:
            bands = [(-1.0 + 1e-7, -0.99), (-0.51, -0.49), (0.99, 1.01), (-1e-5, 1e-5), (1.0, 1e6)]
    k = rng.integers(0, len(bands), n)
    lo = np.array([bands[i][0] for i in k])
    hi = np.array([bands[i][1] for i in k])
    x0 = lo + (hi - lo) * rng.random(n)
    return x0.astype(np.float32 if width == 32 else np.float64)


# the sixteen sibling functions (explog.py:101-325), keyed to their family's
# hot-path function for inputs; smaller samples
FAMILY_OF = {
    "pexp0": "texp", "texp0": "texp", "texpp": "texp", "pexp": "texp",
    "pexpm10": "texpm1", "texpm10": "texpm1", "texpm1p": "texpm1", "pexpm1": "texpm1",
    "plog0": "tlog", "tlog0": "tlog", "tlogp": "tlog", "plog": "tlog",
    "plog1p0": "tlog1p", "tlog1p0": "tlog1p", "tlog1pp": "tlog1p", "plog1p": "tlog1p",
}
N_SIB = 1000


def build_inputs(fn: str, width: int, n_cfg: int = N_CFG, n_edge: int = N_EDGE):
    dt = np.float32 if width == 32 else np.float64
    p = 53 if width == 64 else 24
    x0c, x1c = generate(DIST[(fn, width)], 0, n_cfg, seed=SEED)
    sx0, sx1 = [], []
    for a in special_x0(fn, width):
        a = float(dt(a))
        for b in special_x1(a, width):
            sx0.append(a)
            sx1.append(b)
    rng = np.random.default_rng(SEED + width + len(fn))
    ex0 = edge_x0(fn, width, rng, n_edge)
    u = rng.uniform(-1.0, 1.0, n_edge)
    ex1 = (ex0.astype(np.float64) * u * 2.0 ** -p).astype(dt)
    x0 = np.concatenate([x0c.astype(dt), np.array(sx0, dt), ex0])
    x1 = np.concatenate([x1c.astype(dt), np.array(sx1, dt), ex1])
    return x0, x1


def main():
    import twofold
    from twofold import _fp, api, eft

    out_dir = HERE
    prov = {
        "generator": "tests/golden/gen_golden.py",
        "reference": "twofold " + twofold.__version__ + " (/root/reference/pkg/src)",
        "backend": eft.get_default_backend(),
        "python": platform.python_version(),
        "numpy": np.__version__,
        "libc": " ".join(platform.libc_ver()),
        "have_native_fma": _fp.HAVE_NATIVE_FMA,
        "seed": SEED,
        "n_cfg": N_CFG,
        "npy_disable_cpu_features": os.environ.get("NPY_DISABLE_CPU_FEATURES", ""),
    }
    for width in (64, 32):
        lib = api(width)
        dt = np.float32 if width == 32 else np.float64
        for fn in ("texp", "texpm1", "tlog", "tlog1p"):
            x0, x1 = build_inputs(fn, width)
            f = getattr(lib, fn)
            z0 = np.empty_like(x0)
            z1 = np.empty_like(x1)
            for i in range(x0.size):
                r = f((float(x0[i]), float(x1[i])))
                z0[i] = dt(r.value)
                z1[i] = dt(r.error)
            path = os.path.join(out_dir, f"golden_{fn}_f{width}.npz")
            np.savez_compressed(path, x0=x0, x1=x1, z0=z0, z1=z1, n_cfg=N_CFG,
                                provenance=json.dumps(prov))
            print(f"{path}: {x0.size} vectors", file=sys.stderr)
        for fn, fam in FAMILY_OF.items():
            x0, x1 = build_inputs(fam, width, N_SIB, N_EDGE // 3)
            f = getattr(lib, fn)
            dotted = fn.endswith("0")
            if dotted:
                x1 = np.zeros_like(x1)       # dotted argument: x0 only
            z0 = np.empty_like(x0)
            z1 = np.empty_like(x1)
            keep = np.ones(x0.size, bool)
            for i in range(x0.size):
                try:
                    r = f(float(x0[i])) if dotted else f((float(x0[i]), float(x1[i])))
                except OverflowError:
                    # coupled-argument functions (tlogp, plog, ...) given a
                    # non-coupled special-grid input: math.ldexp raises in the
                    # reference (explog.py:192); no golden value exists
                    keep[i] = False
                    continue
                z0[i] = dt(r.value)
                z1[i] = dt(r.error)
            x0, x1, z0, z1 = x0[keep], x1[keep], z0[keep], z1[keep]
            path = os.path.join(out_dir, f"golden_{fn}_f{width}.npz")
            np.savez_compressed(path, x0=x0, x1=x1, z0=z0, z1=z1, n_cfg=N_SIB,
                                provenance=json.dumps(prov))
            print(f"{path}: {x0.size} vectors", file=sys.stderr)


if __name__ == "__main__":
    main()
