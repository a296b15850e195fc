"""The reference's exponential-core tests (pkg/tests/test_expcore.py:150-230,
TestPexp0 / TestPexpm10: exact points, saturation, NaN, accuracy sweeps at
2^-95 / 2^-38 against a high-precision reference, the coupled invariant),
restated against the B200 kernels of pexp0 / pexpm10 (explog.py:101-103,
135-137 -- the renormalised cores) over whole arrays.  mpmath at 200 bits
stands in for the reference's MPFR oracle."""

import math
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LO64 = float.fromhex("-0x1.74385446d71c4p+9")
HI64 = float.fromhex("0x1.62e42fefa39f0p+9")
FLOOR = {64: 2.0 ** (-1022 + 53), 32: 2.0 ** (-126 + 24)}


@pytest.fixture()
def rng():
    return random.Random(20240917)


def _rel_errors(z, xs, f, width):
    import mpmath

    out = []
    with mpmath.workprec(200):
        for v, e, x in zip(np.atleast_1d(z.value).tolist(), np.atleast_1d(z.error).tolist(), xs):
            if abs(v) < FLOOR[width]:
                continue
            ref = f(mpmath.mpf(x))
            out.append(float(abs((mpmath.mpf(v) + mpmath.mpf(e) - ref) / ref)))
    return np.array(out)


def _coupled(z, width):
    from fractions import Fraction

    dt = np.float64 if width == 64 else np.float32
    v, e = np.asarray(z.value), np.asarray(z.error)
    keep = np.abs(v) >= FLOOR[width]
    rn = np.array([float(Fraction(a) + Fraction(b)) for a, b in
                   zip(v[keep].tolist(), e[keep].tolist())]).astype(dt)
    return np.array_equal(rn, v[keep])


def test_pexp0_points_and_saturation(cuda):
    from paper_1502_05216_b200 import api

    f = api(64)
    assert tuple(f.pexp0(0.0)) == (1.0, 0.0)
    assert tuple(f.pexp0(710.0)) == (math.inf, math.inf)
    assert tuple(f.pexp0(-745.0)) == (0.0, 0.0)
    assert tuple(f.pexp0(math.nextafter(HI64, math.inf))) == (math.inf, math.inf)
    assert tuple(f.pexp0(math.nextafter(LO64, -math.inf))) == (0.0, 0.0)
    assert f.pexp0(HI64).value == math.inf
    assert 0.0 <= f.pexp0(LO64).value <= 2.0 ** -1070
    z = f.pexp0(math.nan)
    assert math.isnan(z.value) and math.isnan(z.error)
    g = api(32)
    assert g.pexp0(0.0).value == 1.0
    assert tuple(g.pexp0(89.0)) == (math.inf, math.inf)
    assert tuple(g.pexp0(-104.0)) == (0.0, 0.0)


def test_pexp0_sweep_accuracy_and_coupled(rng, cuda):
    import mpmath

    from paper_1502_05216_b200 import api

    xs = [min(max(rng.uniform(-1.0, 1.0) * 2.0 ** rng.uniform(-10, 9), -700.0), 700.0)
          for _ in range(2000)] + [1.0]
    z = api(64).pexp0(np.array(xs))
    assert _rel_errors(z, xs, mpmath.exp, 64).max() <= 2.0 ** -95
    assert _coupled(z, 64)


def test_pexp0_binary32_accuracy(rng, cuda):
    import mpmath

    from paper_1502_05216_b200 import api

    xs = np.array([rng.uniform(-87.0, 87.0) for _ in range(2000)], dtype=np.float32)
    z = api(32).pexp0(xs)
    assert _rel_errors(z, xs.astype(np.float64).tolist(), mpmath.exp, 32).max() <= 2.0 ** -38
    assert _coupled(z, 32)


def test_pexpm10_points(cuda):
    import mpmath

    from paper_1502_05216_b200 import api

    f = api(64)
    assert tuple(f.pexpm10(0.0)) == (0.0, 0.0)
    z = f.pexpm10(-50.0)                       # fallback branch: pexp0(x) - 1
    assert abs(z.value + 1.0) < 1e-15
    for x in (-50.0, 3.0, 2.0 ** -30):
        z = f.pexpm10(x)
        assert _rel_errors(z, [x], mpmath.expm1, 64).max() <= 2.0 ** -95
    assert tuple(f.pexpm10(-800.0)) == (-1.0, 0.0)
    assert tuple(f.pexpm10(800.0)) == (math.inf, math.inf)


def test_pexpm10_sweep(rng, cuda):
    import mpmath

    from paper_1502_05216_b200 import api

    xs = [rng.uniform(-1.0, 1.0) * 2.0 ** rng.uniform(-20, 5.3) for _ in range(2000)]
    z = api(64).pexpm10(np.array(xs))
    assert _rel_errors(z, xs, mpmath.expm1, 64).max() <= 2.0 ** -95
    assert _coupled(z, 64)
