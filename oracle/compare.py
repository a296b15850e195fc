"""Parity comparator (TEST INFRASTRUCTURE ONLY; used by tests/, smoke() and bench).

Implements the north-star acceptance rule (BASELINE.json north_star; SURVEY.md
section 8(d) "Parity tolerances"):
  * z0 bitwise vs the reference, mismatches counted with an ulp histogram;
  * |(z0+z1) - (r0+r1)| <= max(rel * |r0+r1|, guard, 2 ulp(r1)) with
      binary64: rel = 2^-95, guard = 2 * 2^-1074
      binary32: rel = 2^-42, guard = 2 * 2^-149
    (the absolute guard and 2 ulp(r1) are the stated edge tolerance: at exp's
    underflow edge the error part itself nears the subnormal range -- for
    binary64 |z| < 2^-969, where ulp(z1) > 2^-95 |z| -- and two
    implementations whose value parts differ by one ulp (glibc vs the
    correctly rounded value) each round their own error part, so they may
    differ by two ulps of z1; e.g. texp(-0x1.51f5145c64954p+9, ...) in cfg 5.
    Elsewhere 2 ulp(z1) ~ 2^-104 |z| and the relative bound decides.  For
    non-coupled inputs z1 is O(z) and its last bits are the limit of any
    implementation whose core splits the value differently);
  * non-finite results: same class (NaN <-> NaN, +-inf same sign).
"""

from __future__ import annotations

import numpy as np

TOL = {64: (2.0 ** -95, 2.0 * 2.0 ** -1074), 32: (2.0 ** -42, 2.0 * 2.0 ** -149)}


def _ulp(r1: np.ndarray) -> np.ndarray:
    """Two ulps of the reference error part: the rounding of z1 on each side.
    For coupled inputs |z1| ~ 2^-53 |z| and this is ~2^-104 |z| (no effect)
    except at exp's underflow edge; for non-coupled inputs (|x1| ~ |x0|) z1 is
    O(z) and its last bits are the limit of any implementation whose core
    splits the value differently."""
    return 2.0 * np.abs(np.spacing(np.abs(r1).astype(r1.dtype))).astype(np.float64)


def _ordered(a: np.ndarray) -> np.ndarray:
    """Map floats to integers whose difference is the ulp distance."""
    if a.dtype == np.float64:
        b = a.view(np.int64).astype(np.int64)
        mag = b & np.int64(0x7FFFFFFFFFFFFFFF)
    else:
        b = a.view(np.int32).astype(np.int64)
        mag = b & np.int64(0x7FFFFFFF)
    return np.where(b < 0, -mag, mag)


def ulp_distance(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    d = np.abs(_ordered(a) - _ordered(b))
    return np.where(np.isnan(a) | np.isnan(b), np.where(np.isnan(a) & np.isnan(b), 0, -1), d)


def same_bits(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    return (a.view(u) == b.view(u)) | (np.isnan(a) & np.isnan(b))


def compare(z0, z1, r0, r1, width: int) -> dict:
    with np.errstate(all="ignore"):
        return _compare(z0, z1, r0, r1, width)


# COUPLED_ARG functions (reference explog.py:52) assume |x1| <= ulp(x0)/2; their
# cores drop the x1*s1 product term (t_mul, eft.py:207-212), so on a
# non-coupled argument the reference itself is only ~2^-54 (2^-25) accurate and
# a 1-ulp different Newton seed moves the result by that much.  Such inputs are
# held to this looser relative bound (plus the class rule) instead of TOL.
LOOSE_REL = {64: 2.0 ** -48, 32: 2.0 ** -19}


def coupled_mask(x0, x1) -> np.ndarray:
    """x0 + x1 rounds to x0 in the lane's own precision (non-finite x0 counts)."""
    x0, x1 = np.asarray(x0), np.asarray(x1)
    with np.errstate(all="ignore"):
        return ((x0 + x1) == x0) | (np.isinf(x0) & np.isfinite(x1))


def bad_mask(z0, z1, r0, r1, width: int, rel: float | None = None, scale=0.0) -> np.ndarray:
    """Elements violating the tolerance or the non-finite class rule.  `scale`
    (an array or scalar) is added to |r0 + r1| in the relative bound: for a
    non-coupled argument it is |x0| + |x1|, the size of the cancellation the
    core performs."""
    z0, z1, r0, r1 = (np.asarray(v) for v in (z0, z1, r0, r1))
    rel0, guard = TOL[width]
    rel = rel0 if rel is None else rel
    with np.errstate(all="ignore"):
        finite = np.isfinite(z0) & np.isfinite(z1) & np.isfinite(r0) & np.isfinite(r1)
        a0, a1, b0, b1 = (v.astype(np.float64) for v in (z0, z1, r0, r1))
        d = (a0 - b0) + (a1 - b1)
        mag = np.abs(b0 + b1) + np.where(np.isfinite(scale), scale, 0.0)
        tol = np.maximum(np.maximum(rel * mag, guard), _ulp(r1))
        viol = finite & ~(np.abs(d) <= tol)

        def cls(a, b):
            return (np.isnan(a) & np.isnan(b)) | (np.isinf(a) & (a == b)) | \
                (np.isfinite(a) & np.isfinite(b))

        return viol | ~(cls(z0, r0) & cls(z1, r1))


def _compare(z0, z1, r0, r1, width: int) -> dict:
    z0, z1, r0, r1 = (np.asarray(v) for v in (z0, z1, r0, r1))
    rel, guard = TOL[width]
    n = z0.size
    s0 = same_bits(z0, r0)
    s1 = same_bits(z1, r1)
    ud = ulp_distance(z0, r0)
    finite = np.isfinite(z0) & np.isfinite(z1) & np.isfinite(r0) & np.isfinite(r1)
    with np.errstate(all="ignore"):
        a0, a1, b0, b1 = (v.astype(np.float64) for v in (z0, z1, r0, r1))
        d = (a0 - b0) + (a1 - b1)
        tol = np.maximum(np.maximum(rel * np.abs(b0 + b1), guard), _ulp(r1))
        viol = finite & ~(np.abs(d) <= tol)
    def cls(a, b):  # same class per field: NaN <-> NaN, +-inf same sign, finite <-> finite
        return (np.isnan(a) & np.isnan(b)) | (np.isinf(a) & (a == b)) | \
            (np.isfinite(a) & np.isfinite(b))

    cls_bad = ~(cls(z0, r0) & cls(z1, r1))
    mism = ~s0
    hist = {}
    if mism.any():
        vals, cnts = np.unique(ud[mism], return_counts=True)
        hist = {int(v): int(c) for v, c in zip(vals, cnts)}
    return {
        "n": int(n),
        "z0_mismatch": int(mism.sum()),
        "z0_ulp_hist": hist,
        "z0_gt1ulp": int((mism & ((ud > 1) | (ud < 0))).sum()),
        "tol_violations": int(viol.sum()),
        "tol_violations_given_z0_match": int((viol & s0).sum()),
        "class_mismatch": int(cls_bad.sum()),
        "z1_bit_mismatch": int((~s1).sum()),
        "z1_bit_mismatch_given_z0_match": int((~s1 & s0).sum()),
        "worst_rel_log2": float(np.log2(np.max(np.where(finite & (np.abs(b0 + b1) > 0),
                                                        np.abs(d) / np.abs(b0 + b1), 0.0))
                                        + 1e-300)),
        "bad_idx": np.nonzero(viol | cls_bad)[0][:20].tolist(),
    }
