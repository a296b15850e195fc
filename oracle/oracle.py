"""Python driver for the CPU oracle (oracle/twofold_oracle.c).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product
package.  It evaluates the reference algorithm (pkg/src/twofold/explog.py:115-317)
op for op on the CPU:

  binary64: one C pass, libm = glibc (the library CPython's math calls);
  binary32: replay passes, libm = numpy float32 ufuncs (the reference's
            _Libm32, _fp.py:221-245), evaluated vectorised between passes.

Parity pinning: tests/test_oracle_golden.py checks this oracle bit-for-bit
against outputs of the reference package itself (tests/golden/*.npz, produced
by tests/golden/gen_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libtforacle.so")

FNS = {"texp": 0, "texpm1": 1, "tlog": 2, "tlog1p": 3,
       "pexp0": 4, "texp0": 5, "texpp": 6, "pexp": 7, "pexpm10": 8, "texpm10": 9,
       "texpm1p": 10, "pexpm1": 11, "plog0": 12, "tlog0": 13, "tlogp": 14, "plog": 15,
       "plog1p0": 16, "tlog1p0": 17, "tlog1pp": 18, "plog1p": 19}
_LIBM32 = {0: np.exp, 1: np.expm1, 2: np.log, 3: np.log1p}


def _cr32(ufunc):
    """binary32 libm stand-in that is correctly rounded up to double-rounding
    (p ~ 2^-28): evaluate in binary64, round once to binary32."""
    def f(x):
        return ufunc(x.astype(np.float64)).astype(np.float32)
    return f


_LIBM32_CR = {k: _cr32(v) for k, v in _LIBM32.items()}


def _rn64(x) -> float:
    """Round an mpmath number to the nearest binary64 (ties-to-even), with
    gradual underflow and overflow to +-inf."""
    import mpmath

    if x == 0:
        return 0.0
    sign, man, exp, bc = x._mpf_
    lead = exp + bc - 1
    if lead > 1023:
        return -math.inf if sign else math.inf
    q = max(lead - 52, -1074)
    shift = q - exp
    if shift <= 0:
        r = man << (-shift)
    else:
        r = man >> shift
        rem = man - (r << shift)
        half = 1 << (shift - 1)
        if rem > half or (rem == half and (r & 1)):
            r += 1
    v = math.ldexp(float(r), q) if r < (1 << 60) else math.inf
    del mpmath
    return -v if sign else v


def _cr64_scalar(f: int, x: float) -> float:
    """Correctly rounded binary64 exp/expm1/log/log1p (mpmath, 160 bits) with
    the reference's IEEE special results (_fp.py:191-218)."""
    import mpmath

    if math.isnan(x):
        return x
    if f == 0:
        if math.isinf(x):
            return x if x > 0 else 0.0
        if x > 710.0:
            return math.inf
        if x < -746.0:
            return 0.0
    elif f == 1:
        if math.isinf(x):
            return x if x > 0 else -1.0
        if x == 0.0:
            return x
        if x > 710.0:
            return math.inf
        if x < -50.0:
            return -1.0
    elif f == 2:
        if x < 0.0:
            return math.nan
        if x == 0.0:
            return -math.inf
        if math.isinf(x):
            return x
    else:
        if x < -1.0:
            return math.nan
        if x == -1.0:
            return -math.inf
        if math.isinf(x) or x == 0.0:
            return x
    with mpmath.workprec(160):
        v = (mpmath.exp, mpmath.expm1, mpmath.log, mpmath.log1p)[f](mpmath.mpf(x))
        return _rn64(v)


def _cr64(f: int):
    def g(x):
        return np.array([_cr64_scalar(f, float(v)) for v in x], dtype=np.float64)
    return g


_LIBM64_CR = {k: _cr64(k) for k in range(4)}

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off).  Several
    processes may call this at once (bench.py's ranks): the build runs under a
    file lock into a temporary name that is renamed into place, so no process
    ever loads a half-written library."""
    import fcntl

    src = os.path.join(HERE, "twofold_oracle.c")

    def stale():
        return force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(src)

    if not stale():
        return LIB_PATH
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    with open(os.path.join(os.path.dirname(LIB_PATH), ".build.lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if stale():
            tmp = f"{LIB_PATH}.{os.getpid()}.tmp"
            subprocess.run(["make", "-s", "-B", "-C", HERE, f"OUT={tmp}"], check=True)
            os.replace(tmp, LIB_PATH)
            force = False
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.tfo_eval_f64.argtypes = [i32, i32, vp, vp, vp, vp, i64, i32]
        L.tfo_eval_f64.restype = i32
        L.tfo_eval_f32_pass.argtypes = [i32, i32, vp, vp, vp, vp, i64, vp, i32, vp, vp, i32]
        L.tfo_eval_f32_pass.restype = i64
        L.tfo_eval_f64_pass.argtypes = [i32, i32, vp, vp, vp, vp, i64, vp, i32, vp, vp, i32]
        L.tfo_eval_f64_pass.restype = i64
        L.tfo_maxcalls.restype = i32
        for name in ("tfo_pexp0_raw64", "tfo_pexpm10_raw64", "tfo_taylor_exp64",
                     "tfo_taylor_expm1_64"):
            getattr(L, name).argtypes = [i32, ctypes.c_double, vp]
        for name in ("tfo_pexp0_raw32", "tfo_pexpm10_raw32"):
            getattr(L, name).argtypes = [i32, ctypes.c_float, vp]
        L.tfo_decompose_exp64.argtypes = [ctypes.c_double, vp, vp]
        L.tfo_decompose_expm1_64.argtypes = [ctypes.c_double, vp, vp]
        L.tfo_decompose_exp32.argtypes = [ctypes.c_float, vp, vp]
        L.tfo_decompose_expm1_32.argtypes = [ctypes.c_float, vp, vp]
        L.tfo_eft64.argtypes = [i32, i32, vp, vp]
        L.tfo_eft.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, vp, ctypes.c_int64]
        L.tfo_eft.restype = i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1)


def evaluate(fn: str, width: int, x0, x1, backend: str = "dv", nthreads: int | None = None,
             libm32: str = "numpy", libm64: str = "glibc"):
    """Reference result (z0, z1) for arrays x0, x1 of the lane's dtype.

    libm32="numpy" is the reference's binary32 libm (_fp.py:221-245);
    libm32="cr" swaps in correctly rounded values (the "CR-sim" oracle of
    SURVEY.md B.6), which isolates the algorithm from numpy's libm error.
    libm64="cr" does the same for binary64 (mpmath; slow, small samples only).
    """
    L = lib()
    code = FNS[fn]
    dv = 1 if backend == "dv" else 0
    if backend not in ("dv", "fma"):
        raise ValueError(f"unknown backend {backend!r}")
    nt = nthreads or default_threads()
    if width == 64 and libm64 == "glibc":
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        x1 = np.ascontiguousarray(x1, dtype=np.float64)
        n = x0.size
        z0 = np.empty(n, np.float64)
        z1 = np.empty(n, np.float64)
        rc = L.tfo_eval_f64(code, dv, _ptr(x0), _ptr(x1), _ptr(z0), _ptr(z1), n, nt)
        if rc != 0:
            raise RuntimeError("oracle rejected arguments")
        return z0, z1
    if width not in (32, 64):
        raise ValueError(f"unsupported width {width!r}")
    dt = np.float64 if width == 64 else np.float32
    run_pass = L.tfo_eval_f64_pass if width == 64 else L.tfo_eval_f32_pass
    x0 = np.ascontiguousarray(x0, dtype=dt)
    x1 = np.ascontiguousarray(x1, dtype=dt)
    n = x0.size
    mc = L.tfo_maxcalls()
    z0 = np.full(n, np.nan, dt)
    z1 = np.full(n, np.nan, dt)
    ans = np.zeros((n, mc), dt)
    req_arg = np.zeros(n, dt)
    req_fn = np.full(n, -1, np.int8)
    if width == 64:
        table = _LIBM64_CR
    else:
        table = _LIBM32 if libm32 == "numpy" else _LIBM32_CR
    for k in range(mc + 1):
        pending = run_pass(code, dv, _ptr(x0), _ptr(x1), _ptr(z0), _ptr(z1), n,
                           _ptr(ans), k, _ptr(req_arg), _ptr(req_fn), nt)
        if pending < 0:
            raise RuntimeError("oracle rejected arguments")
        if pending == 0:
            return z0, z1
        if k == mc:
            break
        with np.errstate(all="ignore"):
            for f, ufunc in table.items():
                sel = req_fn == f
                if sel.any():
                    ans[sel, k] = ufunc(req_arg[sel])
    raise RuntimeError("replay oracle did not converge (more libm calls than expected)")


# ---- building blocks (known-answer tests) -----------------------------------

def pexp0_raw(x: float, width: int = 64, backend: str = "fma"):
    out = np.zeros(2, np.float64 if width == 64 else np.float32)
    f = lib().tfo_pexp0_raw64 if width == 64 else lib().tfo_pexp0_raw32
    f(1 if backend == "dv" else 0, x, _ptr(out))
    return float(out[0]), float(out[1])


def pexpm10_raw(x: float, width: int = 64, backend: str = "fma"):
    out = np.zeros(2, np.float64 if width == 64 else np.float32)
    f = lib().tfo_pexpm10_raw64 if width == 64 else lib().tfo_pexpm10_raw32
    f(1 if backend == "dv" else 0, x, _ptr(out))
    return float(out[0]), float(out[1])


def taylor_exp(y: float, backend: str = "fma"):
    out = np.zeros(2, np.float64)
    lib().tfo_taylor_exp64(1 if backend == "dv" else 0, y, _ptr(out))
    return float(out[0]), float(out[1])


def taylor_expm1(y: float, backend: str = "fma"):
    out = np.zeros(2, np.float64)
    lib().tfo_taylor_expm1_64(1 if backend == "dv" else 0, y, _ptr(out))
    return float(out[0]), float(out[1])


def decompose_exp(x: float, width: int = 64):
    mn = np.zeros(2, np.int64)
    y = np.zeros(1, np.float64 if width == 64 else np.float32)
    f = lib().tfo_decompose_exp64 if width == 64 else lib().tfo_decompose_exp32
    f(x, _ptr(mn), _ptr(y))
    return int(mn[0]), int(mn[1]), float(y[0])


def decompose_expm1(x: float, width: int = 64):
    n = np.zeros(1, np.int64)
    y = np.zeros(1, np.float64 if width == 64 else np.float32)
    f = lib().tfo_decompose_expm1_64 if width == 64 else lib().tfo_decompose_expm1_32
    f(x, _ptr(n), _ptr(y))
    return 0, int(n[0]), float(y[0])


_EFT_OPS = {"two_sum": 0, "fast_two_sum": 1, "renorm": 2, "t_add": 3, "t_add_d": 4,
            "t_mul": 5, "t_mul_d": 6, "two_prod": 7}


def eft64(op: str, *args: float, backend: str = "fma"):
    a = np.zeros(4, np.float64)
    a[: len(args)] = args
    out = np.zeros(2, np.float64)
    lib().tfo_eft64(_EFT_OPS[op], 1 if backend == "dv" else 0, _ptr(a), _ptr(out))
    return float(out[0]), float(out[1])


EFT_OPS = ("fast_two_sum", "two_sum", "two_diff", "two_prod", "split", "renorm_fast", "renorm",
           "t_add", "t_add_d", "t_mul", "t_mul_d", "t_div", "t_sqrt")


def eft_arrays(op: str, width: int, a0, a1=None, b0=None, b1=None, backend: str = "fma"):
    """Element-wise EFT / twofold op over arrays (op codes = TF_OP_*), the C
    restatement of eft.py:77-237 / eft32.py:36-214."""
    dt = np.float64 if width == 64 else np.float32
    a0 = np.ascontiguousarray(a0, dtype=dt)
    arrs = [a0] + [None if v is None else np.ascontiguousarray(v, dtype=dt) for v in (a1, b0, b1)]
    z0 = np.empty_like(a0)
    z1 = np.empty_like(a0)
    rc = lib().tfo_eft(EFT_OPS.index(op), width, 1 if backend == "dv" else 0,
                       *[None if v is None else _ptr(v) for v in arrs], _ptr(z0), _ptr(z1), a0.size)
    if rc:
        raise ValueError(f"tfo_eft({op}) failed")
    return z0, z1
