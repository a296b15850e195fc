// tf_etalon.cuh -- triple-double etalon for the GPU accuracy audit.
//
// The reference audits every function against an MPFR etalon of >= 192 bits
// (pkg/src/twofold/oracle.py:37-123, audit.py:207-286).  gmpy2/MPFR is absent
// here, and the audit is a throughput job, so the etalon is evaluated on the
// GPU in triple-double arithmetic (three non-overlapping binary64 words,
// ~2^-150 relative).  The audited errors live at 2^-93 .. 2^-110 (binary64)
// and 2^-36 .. 2^-50 (binary32), so a 2^-140 etalon measures them to better
// than 2^-30 of themselves; tests/test_gpu_audit.py pins the etalon against
// mpmath at 240 bits.
//
// Values come back as (m, k) = m * 2^k with m a triple-double near [0.5, 2]
// for the exponential families, so results near the binary64 underflow
// threshold (the audit keeps |z| >= 2^-969) keep full relative precision.
//   exp(x):   x = k ln2 + r, |r| <= ln2/2; expm1(r 2^-12) by a degree-11
//             Taylor series, 12 doublings em <- em (em + 2), m = 1 + em;
//   expm1(x): the same without the +1 for |x| <= 0.34, else exp(x) - 1;
//   log1p(d), |d| <= 0.42: Newton on expm1 from the binary64 seed,
//             r <- r - (expm1(r) - d) exp(-r), twice (quadratic: 2^-53 ->
//             2^-106 -> below the triple-double floor);
//   log(y):   y = f 2^e, f in [1/sqrt2, sqrt2], log1p(f - 1) + e ln2;
//   log1p(y): log1p directly for y in [-0.29, 0.41], else log(1 + y).
#pragma once
#include "tf_common.cuh"

namespace tf {
namespace et {

struct TD {
  double a, b, c;
};

__constant__ double c_ln2[3] = {TFE_LN2_INIT};
__constant__ double c_invf[3 * TFE_INVFACT_COUNT] = {TFE_INVFACT_INIT};

TF_DEV TD td(double a, double b = 0.0, double c = 0.0) { return TD{a, b, c}; }
TF_DEV TD ln2() { return td(c_ln2[0], c_ln2[1], c_ln2[2]); }
TF_DEV TD invf(int n) { return td(c_invf[3 * n], c_invf[3 * n + 1], c_invf[3 * n + 2]); }

TF_DEV void two_sum(double a, double b, double& s, double& e) {
  s = add(a, b);
  double bb = sub(s, a);
  e = add(sub(a, sub(s, bb)), sub(b, bb));
}
TF_DEV void two_prod(double a, double b, double& p, double& e) {
  p = mul(a, b);
  e = fmaop(a, b, -p);
}

// Four components (any order of magnitude) -> three non-overlapping words.
// The bottom-up two_sum cascade is exact; only the last addition of the two
// smallest errors rounds (~2^-159 of the total).
TF_DEV TD renorm4(double c0, double c1, double c2, double c3) {
  double s, e1, e2, e3;
  two_sum(c2, c3, s, e3);
  two_sum(c1, s, s, e2);
  two_sum(c0, s, c0, e1);
  double t, u;
  two_sum(e1, e2, t, u);
  u = add(u, e3);
  two_sum(t, u, t, u);
  return td(c0, t, u);
}

TF_DEV TD neg(TD x) { return td(-x.a, -x.b, -x.c); }

TF_DEV TD add3(TD x, TD y) {
  double s0, e0, s1, e1, t1, f1;
  two_sum(x.a, y.a, s0, e0);
  two_sum(x.b, y.b, s1, e1);
  two_sum(s1, e0, t1, f1);
  double s2 = add(add(x.c, y.c), e1);
  return renorm4(s0, t1, s2, f1);
}
TF_DEV TD sub3(TD x, TD y) { return add3(x, neg(y)); }
TF_DEV TD add_d(TD x, double d) { return add3(x, td(d)); }

TF_DEV TD mul3(TD x, TD y) {
  double p0, q0, p1, q1, p2, q2, s1, r1, r2;
  two_prod(x.a, y.a, p0, q0);
  two_prod(x.a, y.b, p1, q1);
  two_prod(x.b, y.a, p2, q2);
  two_sum(p1, p2, s1, r1);
  two_sum(s1, q0, s1, r2);
  double t = fmaop(x.a, y.c, fmaop(x.b, y.b, mul(x.c, y.a)));
  t = add(t, add(add(q1, q2), add(r1, r2)));
  return renorm4(p0, s1, t, 0.0);
}
TF_DEV TD mul_d(TD x, double d) {
  double p0, q0, p1, q1, s1, r;
  two_prod(x.a, d, p0, q0);
  two_prod(x.b, d, p1, q1);
  two_sum(p1, q0, s1, r);
  double t = fmaop(x.c, d, add(q1, r));
  return renorm4(p0, s1, t, 0.0);
}
TF_DEV TD scale(TD x, int k) { return td(ldexp(x.a, k), ldexp(x.b, k), ldexp(x.c, k)); }

// expm1 of a small argument (|r| <= 0.36)
TF_DEV TD expm1_small(TD r) {
  int s = fabs(r.a) > 0x1p-13 ? 12 : 0;
  TD x = scale(r, -s);
  TD p = invf(11);
#pragma unroll 1
  for (int n = 10; n >= 1; --n) p = add3(mul3(p, x), invf(n));
  TD em = mul3(p, x);
#pragma unroll 1
  for (int i = 0; i < s; ++i) em = mul3(em, add_d(em, 2.0));
  return em;
}

// exp(x) = m * 2^k
TF_DEV TD exp3(TD x, int& k) {
  double kd = fmin(fmax(rint(mul(x.a, 0x1.71547652b82fep+0)), -4000.0), 4000.0);
  k = (int)kd;
  TD r = sub3(x, mul_d(ln2(), kd));
  return add_d(expm1_small(r), 1.0);
}

// expm1(x) = m * 2^k
TF_DEV TD expm1_3(TD x, int& k) {
  if (fabs(x.a) <= 0.34) {
    k = 0;
    return expm1_small(x);
  }
  TD m = exp3(x, k);
  if (k >= 1) return add_d(m, -ldexp(1.0, -k));
  TD v = add_d(scale(m, k), -1.0);
  k = 0;
  return v;
}

// log1p(d) for |d| <= ~0.42
TF_DEV TD log1p_core3(TD d) {
  TD r = td(log1p(d.a));
#pragma unroll 1
  for (int it = 0; it < 2; ++it) {
    int k1, k2;
    TD em = expm1_3(r, k1);
    TD e = exp3(neg(r), k2);
    TD f = sub3(scale(em, k1), d);
    r = sub3(r, mul3(f, scale(e, k2)));
  }
  return r;
}

// log(y), y > 0 finite
TF_DEV TD log3(TD y) {
  int e = ilogb(y.a);
  TD f = scale(y, -e);
  if (f.a > 1.4142135623730951) {
    f = scale(f, -1);
    e += 1;
  }
  TD l = log1p_core3(add_d(f, -1.0));
  return e == 0 ? l : add3(mul_d(ln2(), (double)e), l);
}

// log1p(y), y > -1 finite
TF_DEV TD log1p3(TD y) {
  if (y.a >= -0.29 && y.a <= 0.41) return log1p_core3(y);
  return log3(add_d(y, 1.0));
}

enum Family { EXP = 0, EXPM1 = 1, LOG = 2, LOG1P = 3 };

// Etalon of the family at x0 + x1 (exact), as m * 2^k.  Returns false for an
// argument outside the mathematical domain (the reference OracleDomainError,
// oracle.py:93-116): non-finite, log of <= 0, log1p of <= -1.
TF_DEV bool etalon(int fam, double x0, double x1, TD& m, int& k) {
  k = 0;
  if (!(fabs(x0) <= 1.79769313486231570e308) || !(fabs(x1) <= 1.79769313486231570e308))
    return false;
  double s, e;
  two_sum(x0, x1, s, e);
  if (!(fabs(s) <= 1.79769313486231570e308)) return false;
  TD x = td(s, e);
  if (fam == EXP) {
    m = exp3(x, k);
  } else if (fam == EXPM1) {
    m = expm1_3(x, k);
  } else if (fam == LOG) {
    if (!(s > 0.0)) return false;
    m = log3(x);
  } else {
    if (!(s > -1.0) && !(s == -1.0 && e > 0.0)) return false;
    m = log1p3(x);
  }
  return true;
}

}  // namespace et
}  // namespace tf
