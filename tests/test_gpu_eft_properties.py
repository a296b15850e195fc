"""The reference's own EFT / twofold-arithmetic test suite (pkg/tests/test_eft.py:
examples, exactness in rational arithmetic, backend equivalence, the coupled
invariant, the 8*2^-2p residual bound, the non-finite policy), restated
against the B200 element-wise kernels: each property is checked on whole
arrays evaluated in one launch.  Exactness is verified with Python rationals
(fractions.Fraction) and the residual bound with mpmath at 200 bits, never
against another float path."""

import math
import random
from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NAN, INF = math.nan, math.inf


@pytest.fixture()
def rng():
    return random.Random(20240917)            # the reference conftest's seed


def rand_double(rng, emin=-300, emax=300):
    return rng.uniform(-1.0, 1.0) * 2.0 ** rng.randint(emin, emax)


def rand_single(rng, emin=-60, emax=60):
    return float(np.float32(rng.uniform(-1.0, 1.0) * 2.0 ** rng.randint(emin, emax)))


def _arr(xs, width=64):
    return np.array(xs, dtype=np.float64 if width == 64 else np.float32)


def _exact(op, a, b, v, e):
    """a (op) b == v + e in exact rational arithmetic, element-wise."""
    ok = []
    for ai, bi, vi, ei in zip(a.tolist(), b.tolist(), v.tolist(), e.tolist()):
        if not all(math.isfinite(t) for t in (ai, bi, vi, ei)):
            ok.append(False)
            continue
        lhs = {"+": Fraction(ai) + Fraction(bi), "-": Fraction(ai) - Fraction(bi),
               "*": Fraction(ai) * Fraction(bi)}[op]
        ok.append(lhs == Fraction(vi) + Fraction(ei))
    return np.array(ok)


def _sig_bits(x):
    if x == 0.0:
        return 0
    n = Fraction(abs(x)).numerator
    while n % 2 == 0:
        n //= 2
    return n.bit_length()


def test_examples(cuda):
    from paper_1502_05216_b200 import Twofold, eft

    assert eft.fast_two_sum(1.0, 2.0 ** -60) == (1.0, 2.0 ** -60)
    assert eft.fast_two_sum(3.0, 0.0) == (3.0, 0.0)
    assert eft.two_sum(2.0 ** -60, 1.0) == (1.0, 2.0 ** -60)
    assert eft.two_sum(1.0, -1.0) == (0.0, 0.0)
    assert eft.two_diff(1.0, 2.0 ** -60) == (1.0, -(2.0 ** -60))
    assert eft.two_diff(0.7, 0.7) == (0.0, 0.0)
    assert eft.split(3.0) == (3.0, 0.0)
    assert eft.split(1.0 + 2.0 ** -30) == (1.0, 2.0 ** -30)
    big = 2.0 ** 27 + 1.0
    assert eft.two_prod_fma(big, big) == (2.0 ** 54 + 2.0 ** 28, 1.0)
    assert eft.two_prod_fma(123.25, 0.0) == (0.0, 0.0)
    assert eft.two_prod_dv(big, big) == eft.two_prod_fma(big, big)
    assert eft.fma_sim(1.5, 2.0, -3.0) == 0.0
    x = 1.0 + 2.0 ** -30
    assert eft.fma_sim(x, x, -(1.0 + 2.0 ** -29)) == 2.0 ** -60
    assert eft.renorm_fast(Twofold(1.0, 2.0 ** -60)) == (1.0, 2.0 ** -60)
    assert eft.renorm_fast(Twofold(1.0, 1.0)) == (2.0, 0.0)
    assert eft.renorm(Twofold(2.0 ** -60, 1.0)) == (1.0, 2.0 ** -60)
    assert eft.renorm(Twofold(1.0, -1.0)) == (0.0, 0.0)
    assert eft.t_add(Twofold(1.0, 0.0), Twofold(-1.0, 0.0)) == (0.0, 0.0)
    assert eft.t_mul_d(Twofold(1.0, 2.0 ** -60), 2.0) == (2.0, 2.0 ** -59)


def test_corrected_subtraction_regression(cuda):
    from paper_1502_05216_b200 import eft, eft32

    a = float.fromhex("0x1.5f5cacb16e2d4p-27")
    b = float.fromhex("-0x1.9b37401de3f40p-9")
    g = eft.two_diff(a, b)
    assert g.value == float.fromhex("0x1.9b3797f50f206p-9")
    assert g.error == float.fromhex("-0x1.1d2c000000000p-63")
    a = float.fromhex("0x1.324b4cp-6")
    b = float.fromhex("-0x1.35f33cp-10")
    g = eft32.two_diff(a, b)
    assert g.value == float.fromhex("0x1.45aa80p-6")
    assert g.error == float.fromhex("-0x1p-32")


@pytest.mark.parametrize("width", (64, 32))
def test_sums_and_differences_exact(width, rng, cuda):
    from paper_1502_05216_b200 import eft, eft32

    mod = eft if width == 64 else eft32
    draw = rand_double if width == 64 else rand_single
    a = _arr([draw(rng) for _ in range(20000)], width)
    b = _arr([draw(rng) for _ in range(20000)], width)
    assert _exact("+", a, b, *mod.two_sum(a, b)).all()
    assert _exact("-", a, b, *mod.two_diff(a, b)).all()
    big = np.where(np.abs(a) >= np.abs(b), a, b)
    small = np.where(np.abs(a) >= np.abs(b), b, a)
    assert _exact("+", big, small, *mod.fast_two_sum(big, small)).all()


def test_split_bits_and_exactness(rng, cuda):
    from paper_1502_05216_b200 import eft, eft32

    xs = [rand_double(rng) for _ in range(20000)]
    xs += [2.0 ** 1000, -(2.0 ** 1023), 1.7e308, math.nextafter(INF, 0.0),
           float.fromhex("0x1.fffffffp+1023"), float.fromhex("-0x1.fffffffp+1023")]
    xs += [rng.uniform(1.0, 2.0) * 2.0 ** 1020 for _ in range(2000)]
    x = _arr(xs)
    h, lo = eft.split(x)
    assert np.isfinite(h).all() and np.isfinite(lo).all()
    assert _exact("+", h, lo, x, np.zeros_like(x)).all()
    assert max(_sig_bits(v) for v in h.tolist()) <= 27
    assert max(_sig_bits(v) for v in lo.tolist()) <= 27
    x32 = _arr([rand_single(rng) for _ in range(20000)] + [3e38, -3.4e38, 2.0 ** 120], 32)
    h, lo = eft32.split(x32)
    assert np.isfinite(h).all() and _exact("+", h, lo, x32, np.zeros_like(x32)).all()


@pytest.mark.parametrize("width", (64, 32))
def test_two_prod_exact_and_backend_equivalence(width, rng, cuda):
    from paper_1502_05216_b200 import eft, eft32

    mod = eft if width == 64 else eft32
    if width == 64:
        a = _arr([rand_double(rng) for _ in range(20000)])
        b = _arr([rand_double(rng) for _ in range(20000)])
    else:   # exponents within +-25: the exact residual never underflows
        a = _arr([rand_single(rng, -25, 25) for _ in range(20000)], 32)
        b = _arr([rand_single(rng, -25, 25) for _ in range(20000)], 32)
    v, e = mod.two_prod_fma(a, b)
    assert _exact("*", a, b, v, e).all()
    v2, e2 = mod.two_prod_dv(a, b)
    assert np.array_equal(v, v2) and np.array_equal(e, e2)


def test_fma_sim_matches_fused_op_on_remainder_domain(rng, cuda):
    from paper_1502_05216_b200 import eft

    a = _arr([rand_double(rng, -200, 200) for _ in range(20000)])
    b = _arr([rand_double(rng, -200, 200) for _ in range(20000)])
    with np.errstate(all="ignore"):
        q = a / b
    keep = np.isfinite(q) & (q != 0) & (b != 0)
    a, b, q = a[keep], b[keep], q[keep]
    got = eft.fma_sim(-q, b, a)
    # fused reference: exact a - q*b rounded once (rational arithmetic)
    want = np.array([float(Fraction(x) - Fraction(y) * Fraction(z))
                     for x, y, z in zip(a.tolist(), q.tolist(), b.tolist())])
    assert np.array_equal(got, want)
    assert np.array_equal(eft.arith("fma").rem(q, b, a), want)


@pytest.mark.parametrize("width", (64, 32))
def test_renorm_coupled_invariant(width, rng, cuda):
    from paper_1502_05216_b200 import Twofold, eft, eft32

    mod = eft if width == 64 else eft32
    if width == 64:
        v = _arr([rand_double(rng, -100, 100) for _ in range(5000)])
        e = _arr([rand_double(rng, -100, 100) for _ in range(5000)])
    else:
        v = _arr([rand_single(rng) for _ in range(5000)], 32)
        e = _arr([rand_single(rng) for _ in range(5000)], 32)
    t = mod.renorm(Twofold(v, e))
    assert _exact("+", v, e, t.value, t.error).all()
    dt = np.float64 if width == 64 else np.float32
    # coupled: value + error rounds to value (exact sum rounded once)
    rn = np.array([float(Fraction(a) + Fraction(b)) for a, b in
                   zip(t.value.tolist(), t.error.tolist())]).astype(dt)
    assert np.array_equal(rn, t.value)
    if width == 64:
        d = v * np.array([rng.uniform(-1.0, 1.0) for _ in range(5000)])
        f = eft.renorm_fast(Twofold(v, d))
        assert _exact("+", v, d, f.value, f.error).all()


@pytest.mark.parametrize("backend", ("fma", "dv"))
@pytest.mark.parametrize("width", (64, 32))
def test_residual_bound(width, backend, rng, cuda):
    import mpmath

    from paper_1502_05216_b200 import Twofold, eft, eft32

    ar = (eft if width == 64 else eft32).arith(backend)
    p = 53 if width == 64 else 24
    bound = 8.0 * 2.0 ** (-2 * p)
    dt = np.float64 if width == 64 else np.float32
    x0 = np.array([2.0 ** rng.uniform(-8, 8) for _ in range(4000)]).astype(dt)
    y0 = np.array([2.0 ** rng.uniform(-8, 8) for _ in range(4000)]).astype(dt)
    x1 = (x0.astype(np.float64) * np.array([rng.uniform(-1, 1) for _ in range(4000)])
          * 2.0 ** -p).astype(dt)
    y1 = (y0.astype(np.float64) * np.array([rng.uniform(-1, 1) for _ in range(4000)])
          * 2.0 ** -p).astype(dt)
    x, y = Twofold(x0, x1), Twofold(y0, y1)
    res = {"add": ar.t_add(x, y), "mul": ar.t_mul(x, y), "div": ar.t_div(x, y),
           "sqrt": ar.t_sqrt(x)}
    with mpmath.workprec(200):
        for i in range(0, 4000, 7):
            xs = mpmath.mpf(float(x0[i])) + mpmath.mpf(float(x1[i]))
            ys = mpmath.mpf(float(y0[i])) + mpmath.mpf(float(y1[i]))
            ref = {"add": xs + ys, "mul": xs * ys, "div": xs / ys, "sqrt": mpmath.sqrt(xs)}
            for k, r in res.items():
                got = mpmath.mpf(float(r.value[i])) + mpmath.mpf(float(r.error[i]))
                assert abs((got - ref[k]) / ref[k]) <= bound, (k, i)
    with np.errstate(all="ignore"):
        assert np.array_equal(res["add"].value, x0 + y0)
        assert np.array_equal(res["mul"].value, x0 * y0)
        assert np.array_equal(res["div"].value, x0 / y0)


def test_division_sqrt_and_special_policy(cuda):
    from paper_1502_05216_b200 import Twofold, eft

    assert eft.t_div(Twofold(1.0, 0.0), Twofold(0.0, 0.0)) == (INF, INF)
    z = eft.t_div(Twofold(0.0, 0.0), Twofold(0.0, 0.0))
    assert math.isnan(z.value) and math.isnan(z.error)
    assert eft.t_div(Twofold(-1.0, 0.0), Twofold(0.0, 0.0)) == (-INF, -INF)
    assert eft.t_sqrt(Twofold(0.0, 0.0)) == (0.0, 0.0)
    z = eft.t_sqrt(Twofold(-1.0, 0.0))
    assert math.isnan(z.value) and math.isnan(z.error)
    assert eft.two_sum(INF, -1.0) == (INF, INF)
    assert eft.fast_two_sum(-INF, 1.0) == (-INF, -INF)
    assert eft.t_add_d(Twofold(INF, INF), -1.0) == (INF, INF)
    z = eft.t_add(Twofold(INF, NAN), Twofold(0.0, 0.0))
    assert z.value == INF and math.isnan(z.error)
    z = eft.two_sum(INF, -INF)
    assert math.isnan(z.value) and math.isnan(z.error)
    z = eft.renorm(Twofold(INF, NAN))
    assert math.isnan(z.value) and math.isnan(z.error)


def test_backend_selection_routes_the_kernels(cuda):
    from paper_1502_05216_b200 import eft

    old = eft.get_default_backend()
    try:
        eft.set_default_backend("dv")
        assert eft.get_default_backend() == "dv" and eft.arith().backend == "dv"
    finally:
        eft.set_default_backend(old)
    with pytest.raises(ValueError):
        eft.set_default_backend("avx")
    with pytest.raises(ValueError):
        eft.arith("nope")
