"""Generation and bit-exact serialization of the coupled constant tables
(reference pkg/src/twofold/tables.py:93-155 semantics, regenerated with mpmath
instead of the gmpy2/MPFR oracle).

  E[m]    = exp(2**L * m),            m in [m_min, m_max]
  C[n]    = exp(n * 2**-K) / N!,      n in [n_min, n_max]
  CM1[n]  = expm1(n * 2**-K_m1),      n in [-n_m1, n_m1]
  LN2     = ln 2
  INVFACT = 1 / N_m1!
each stored "coupled": value = RN_w(ref), error = RN_w(ref - value) (RN_w =
round-to-nearest-even onto binary64/binary32 including subnormals; a zero error
keeps the sign of the remainder).  ``dump_tables`` writes the reference's text
format (tables.py:141-155) -- the CUDA kernels compile the same entries in
through csrc/tf_tables.h (tools/gen_tables.py), and tests/test_tables.py checks
both against the reference's packaged dumps bit for bit.
"""

from __future__ import annotations

import math

import mpmath

__all__ = ["gen", "dump_tables", "round_nearest", "coupled", "WIDTHS", "PREC"]

FORMAT_TAG = "twofold-tables"
FORMAT_VERSION = 1

PREC = 192

# (width, p, emin, L, K, N, Km1, Nm1, m_min, m_max, n_min, n_max, n_m1)
WIDTHS = {
    64: dict(p=53, emin=-1022, L=2, K=5, N=12, Km1=7, Nm1=10,
             m_min=-186, m_max=177, n_min=-128, n_max=128, n_m1=89),
    32: dict(p=24, emin=-126, L=1, K=5, N=6, Km1=7, Nm1=5,
             m_min=-51, m_max=44, n_min=-64, n_max=64, n_m1=89),
}


def round_nearest(x: mpmath.mpf, p: int, emin: int) -> float:
    """RN-even of an mpf onto the binary format (p, emin) incl. subnormals.

    Returns a Python float (exact for both formats); signed zero follows x.
    """
    if x == 0:
        return math.copysign(0.0, float(mpmath.sign(x)) or 1.0)
    sign, man, exp, bc = x._mpf_
    # |x| = man * 2**exp, man odd or normalised; leading bit weight 2**(exp+bc-1)
    lead = exp + bc - 1
    q = max(lead - (p - 1), emin - (p - 1))  # quantum exponent
    shift = q - exp
    if shift <= 0:
        r = man << (-shift)
    else:
        r = man >> shift
        rem = man - (r << shift)
        half = 1 << (shift - 1)
        if rem > half or (rem == half and (r & 1)):
            r += 1
    v = math.ldexp(float(r), q) if r < (1 << 60) else math.ldexp(float(r >> 8), q + 8)
    assert math.ldexp(v, -q) == r, "exact representation expected"
    return -v if sign else v


def coupled(ref: mpmath.mpf, p: int, emin: int) -> tuple[float, float]:
    v = round_nearest(ref, p, emin)
    rem = ref - mpmath.mpf(v)
    e = round_nearest(rem, p, emin)
    if e == 0.0:
        e = -0.0 if rem < 0 else 0.0
    return v, e


def gen(width: int, precision: int = PREC) -> dict:
    """All tables of one width at `precision` bits (>= 2p + 60, tables.py:95-99)."""
    P = WIDTHS[width]
    p, emin = P["p"], P["emin"]
    if precision < 2 * p + 60:
        raise ValueError(f"oracle precision {precision} too low for width {width}")
    with mpmath.workprec(precision):
        stride = mpmath.mpf(2) ** P["L"]
        fact = mpmath.mpf(math.factorial(P["N"]))
        E = [coupled(mpmath.exp(stride * m), p, emin)
             for m in range(P["m_min"], P["m_max"] + 1)]
        sc = mpmath.mpf(2) ** -P["K"]
        C = [coupled(mpmath.exp(n * sc) / fact, p, emin)
             for n in range(P["n_min"], P["n_max"] + 1)]
        sm = mpmath.mpf(2) ** -P["Km1"]
        CM1 = [coupled(mpmath.expm1(n * sm), p, emin)
               for n in range(-P["n_m1"], P["n_m1"] + 1)]
        LN2 = coupled(mpmath.log(2), p, emin)
        INV = coupled(1 / mpmath.mpf(math.factorial(P["Nm1"])), p, emin)
    return dict(E=E, C=C, CM1=CM1, LN2=LN2, INVFACT=INV, **P)



def dump_tables(width: int, precision: int = PREC) -> str:
    """The reference's line format (tables.py:141-155): a header line, then
    ``NAME INDEX VALUE ERROR`` with hex float literals."""
    t = gen(width, precision)
    lines = [f"{FORMAT_TAG} {FORMAT_VERSION} width={width} L={t['L']} K={t['K']} "
             f"N={t['N']} Km1={t['Km1']} Nm1={t['Nm1']} prec={precision}"]
    for name, lo in (("E", t["m_min"]), ("C", t["n_min"]), ("CM1", -t["n_m1"])):
        for j, (v, e) in enumerate(t[name]):
            lines.append(f"{name} {lo + j} {v.hex()} {e.hex()}")
    lines.append(f"LN2 0 {t['LN2'][0].hex()} {t['LN2'][1].hex()}")
    lines.append(f"INVFACT 0 {t['INVFACT'][0].hex()} {t['INVFACT'][1].hex()}")
    return "\n".join(lines) + "\n"
