"""Known-answer tests of the CPU oracle's building blocks, restating the
reference's own pinned vectors (pkg/tests/test_expcore.py, test_eft.py,
audit.py:run_demo), plus accuracy spot checks against mpmath (the reference
checks against a 192-bit MPFR oracle, absent here)."""

import math

import mpmath
import numpy as np
import pytest

from oracle import oracle as O

F12 = float(math.factorial(12))
LO64 = float.fromhex("-0x1.74385446d71c4p+9")
HI64 = float.fromhex("0x1.62e42fefa39f0p+9")
LN2 = float.fromhex("0x1.62e42fefa39efp-1")
INF, NAN = math.inf, math.nan


# ---- decomposition (test_expcore.py:37-106)
def test_decompose_exp_examples():
    assert O.decompose_exp(1.0) == (0, 32, 0.0)
    assert O.decompose_exp(0.0) == (0, 0, 0.0)
    m, n, y = O.decompose_exp(0.3)
    assert (m, n) == (0, 10) and y == 0.3 - 0.3125
    m, n, y = O.decompose_exp(-0.3)
    assert (m, n) == (0, -10) and y == -(0.3 - 0.3125)


def test_decompose_exp_table_edges():
    assert O.decompose_exp(HI64)[0] == 177
    assert O.decompose_exp(LO64)[0] == -186
    assert O.decompose_exp(float.fromhex("0x1.62e430p+6"), 32)[0] == 44
    assert O.decompose_exp(float.fromhex("-0x1.9d1da0p+6"), 32)[0] == -51


def test_decompose_expm1_examples():
    assert O.decompose_expm1(0.0) == (0, 0, 0.0)
    _, n, y = O.decompose_expm1(0.1)
    assert n == 13 and y == 0.1 - 13.0 / 128.0
    assert O.decompose_expm1(LN2)[1] == 89 and O.decompose_expm1(-LN2)[1] == -89


def test_decompose_exact_random():
    rng = np.random.default_rng(20240917)
    for x in rng.uniform(LO64, HI64, 2000):
        m, n, y = O.decompose_exp(float(x))
        assert mpmath.mpf(4 * m) + mpmath.mpf(n) / 32 + mpmath.mpf(y) == mpmath.mpf(float(x))
        assert abs(y) <= 2.0 ** -6


# ---- Taylor cores (test_expcore.py:108-149)
def test_taylor_at_zero():
    assert O.taylor_exp(0.0) == (F12, 0.0)
    assert O.taylor_expm1(0.0) == (0.0, 0.0)


@pytest.mark.parametrize("y", [2.0 ** -6, -(2.0 ** -6), 1e-3, -7e-4])
def test_taylor_exp_accuracy(y):
    v, e = O.taylor_exp(y)
    with mpmath.workprec(200):
        ref = mpmath.exp(mpmath.mpf(y)) * F12
        rel = abs((mpmath.mpf(v) + mpmath.mpf(e)) - ref) / ref
    assert rel <= 2.0 ** -100


# ---- pexp0 / pexpm10 (test_expcore.py:151-230)
def test_pexp0_saturation_and_one():
    assert O.pexp0_raw(0.0) == (1.0, 0.0)
    assert O.pexp0_raw(-745.0) == (0.0, 0.0)
    assert O.pexp0_raw(710.0) == (INF, INF)
    assert O.pexp0_raw(math.nextafter(HI64, INF)) == (INF, INF)
    assert O.pexp0_raw(math.nextafter(LO64, -INF)) == (0.0, 0.0)
    assert O.pexp0_raw(HI64)[0] == INF
    assert 0.0 <= O.pexp0_raw(LO64)[0] <= 2.0 ** -1070
    v, e = O.pexp0_raw(NAN)
    assert math.isnan(v) and math.isnan(e)


def test_pexp0_f32():
    assert O.pexp0_raw(0.0, 32)[0] == 1.0
    assert O.pexp0_raw(89.0, 32) == (INF, INF)
    assert O.pexp0_raw(-104.0, 32) == (0.0, 0.0)


def test_pexpm10_cases():
    assert O.pexpm10_raw(0.0) == (0.0, 0.0)
    assert O.pexpm10_raw(-800.0) == (-1.0, 0.0)
    assert O.pexpm10_raw(800.0) == (INF, INF)
    for x in (-50.0, 3.0, 2.0 ** -30, 0.5):
        v, e = O.pexpm10_raw(x)
        with mpmath.workprec(200):
            ref = mpmath.expm1(mpmath.mpf(x))
            assert abs(mpmath.mpf(v) + mpmath.mpf(e) - ref) / abs(ref) <= 2.0 ** -95


def test_pexp0_sweep_accuracy():
    rng = np.random.default_rng(7)
    for x in rng.uniform(-670.0, 700.0, 300):   # |e^x| above ERROR_FLOOR64 = 2^-969
        v, e = O.pexp0_raw(float(x))
        with mpmath.workprec(200):
            ref = mpmath.exp(mpmath.mpf(float(x)))
            assert abs(mpmath.mpf(v) + mpmath.mpf(e) - ref) / ref <= 2.0 ** -95


# ---- EFT examples and the special-value policy (test_eft.py)
def test_eft_examples():
    assert O.eft64("fast_two_sum", 1.0, 2.0 ** -60) == (1.0, 2.0 ** -60)
    assert O.eft64("two_sum", 2.0 ** -60, 1.0) == (1.0, 2.0 ** -60)
    assert O.eft64("two_sum", 1.0, -1.0) == (0.0, 0.0)
    big = 2.0 ** 27 + 1.0
    for be in ("fma", "dv"):
        assert O.eft64("two_prod", big, big, backend=be) == (2.0 ** 54 + 2.0 ** 28, 1.0)
    assert O.eft64("renorm", 2.0 ** -60, 1.0) == (1.0, 2.0 ** -60)
    assert O.eft64("renorm", 1.0, -1.0) == (0.0, 0.0)
    assert O.eft64("t_add", 1.0, 0.0, -1.0, 0.0) == (0.0, 0.0)
    assert O.eft64("t_mul_d", 1.0, 2.0 ** -60, 2.0) == (2.0, 2.0 ** -59)


def test_special_policy():
    assert O.eft64("two_sum", INF, -1.0) == (INF, INF)
    assert O.eft64("fast_two_sum", -INF, 1.0) == (-INF, -INF)
    assert O.eft64("t_add_d", INF, INF, -1.0) == (INF, INF)
    v, e = O.eft64("t_add", INF, NAN, 0.0, 0.0)
    assert v == INF and math.isnan(e)
    v, e = O.eft64("two_sum", INF, -INF)
    assert math.isnan(v) and math.isnan(e)


# ---- the reference demo's corner cases (audit.py:409-459)
def _ev(fn, width, x0, x1=0.0):
    dt = np.float64 if width == 64 else np.float32
    z0, z1 = O.evaluate(fn, width, np.array([x0], dt), np.array([x1], dt))
    return float(z0[0]), float(z1[0])


@pytest.mark.parametrize("width", (64, 32))
def test_demo_corner_cases(width):
    z = _ev("texp", width, NAN)
    assert math.isnan(z[0]) and math.isnan(z[1])
    assert _ev("texp", width, INF) == (INF, INF)
    assert _ev("texp", width, -INF) == (0.0, 0.0)
    assert _ev("tlog", width, INF) == (INF, INF)
    z = _ev("tlog", width, 1.0, -1.0)
    assert z[0] == 0.0 and math.isnan(z[1])
    assert _ev("texp", width, 0.0)[0] == 1.0


def test_demo_values_f64():
    assert _ev("texp", 64, 1.0)[0] == math.exp(1.0)
    assert _ev("texpm1", 64, 1.0)[0] == math.expm1(1.0)
    assert _ev("tlog", 64, 2.0)[0] == math.log(2.0)
    assert _ev("tlog1p", 64, 1.0)[0] == math.log1p(1.0)
    z = _ev("tlog1p", 64, -1.0)
    assert z == (-INF, -INF)
