"""The binary32 rounding guard (paper_1502_05216_b200/csrc/tf_fast.cuh:
kguard / rn_guard / rn_guard_p) restated in exact rational arithmetic.

The kernels round a twofold core h + l to z = RN32(h + l) and flag the element
when RN32(z + rho k) != z, rho = RN32(RN32(h - z) + l), k = 1 + eps + 2 eps^2
(eps = 2^(TOL+25); one ulp of k when 2 eps^2 is below it).  Claim: whenever the
exact value X lies within 2^TOL |z| of h + l and RN32(X) != z, the element is
flagged.  Checked here on the boundary of that error ball (RN is monotone, so
the ball's end points decide) for random cores placed near rounding midpoints,
including powers of two and their half-size midpoints below.  CPU only.
"""
from fractions import Fraction as Fr
import random

import numpy as np
import pytest


def rn32(x):
    """Round a rational to the nearest binary32 (ties to even), normal range."""
    c = np.float32(float(x))
    best = None
    for cand in (np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))):
        d = abs(Fr(float(cand)) - x)
        if best is None or d < best[0] or (d == best[0] and
                                           int(np.float32(cand).view(np.int32)) % 2 == 0):
            best = (d, cand)
    return np.float32(best[1])


def kguard(tol):
    sq = 23 + 2 * (tol + 25) + 1
    bits = 0x3F800000 + (1 << (23 + tol + 25)) + ((1 << sq) if sq > 0 else 1)
    return np.array([bits], dtype=np.uint32).view(np.float32)[0]


def guard(h, l, tol):
    z = rn32(Fr(float(h)) + Fr(float(l)))
    rho = rn32(Fr(float(rn32(Fr(float(h)) - Fr(float(z))))) + Fr(float(l)))
    k = kguard(tol)
    hard = rn32(Fr(float(rho)) * Fr(float(k)) + Fr(float(z))) != z
    return z, bool(hard)


def ulp(z):
    return Fr(float(np.nextafter(np.float32(abs(z)), np.float32(np.inf)))) - Fr(float(abs(z)))


@pytest.mark.parametrize("tol", (-36, -32))
def test_guard_flags_every_element_that_could_misround(tol):
    rng = random.Random(1234 + tol)
    flagged = checked = 0
    for i in range(4000):
        e = rng.randint(-60, 60)
        if i % 4 == 0:
            z0 = np.float32(2.0 ** e)                          # power of two
        else:
            z0 = np.float32(rng.uniform(1, 2) * 2.0 ** e)
        u = ulp(z0)
        below = Fr(float(z0)) - Fr(float(np.float32(z0) - np.nextafter(
            np.float32(z0), np.float32(-np.inf)))) / 2   # midpoint below (half-size at 2^e)
        mid = Fr(float(z0)) + u / 2 if rng.random() < 0.5 else below
        # core value h + l within a few tolerances of the midpoint
        off = Fr(rng.uniform(-8, 8)) * Fr(2) ** tol * Fr(float(abs(z0)))
        s = mid + off
        h = rn32(s)
        l = rn32(s - Fr(float(h)))
        z, hard = guard(h, l, tol)
        core = Fr(float(h)) + Fr(float(l))
        r = Fr(2) ** tol * Fr(float(abs(z)))
        misround = rn32(core - r) != z or rn32(core + r) != z
        checked += 1
        flagged += hard
        assert hard or not misround, (float(h), float(l), tol)
    assert 0 < flagged < checked


def test_guard_rarely_flags_generic_values():
    rng = random.Random(7)
    n, hard_n = 3000, 0
    for _ in range(n):
        h = np.float32(rng.uniform(1, 2) * 2.0 ** rng.randint(-30, 30))
        l = np.float32(float(h) * rng.uniform(-1, 1) * 2.0 ** -25)
        hard_n += guard(h, l, -36)[1]
    assert hard_n <= 10                                        # ~2^-11 expected
