// tf_general.cuh -- the exact ("rare") path: a complete device restatement of
// the reference texp/texpm1/tlog/tlog1p (pkg/src/twofold/explog.py:115-317,
// expcore.py:35-147) with every _special check, for ANY input: NaN/inf,
// out-of-domain, subnormal, under/overflowing intermediates, non-coupled
// twofolds, second Newton iterations.  The fast kernels divert every element
// outside their admission band to this path (per-warp queue, tf_kernels.cu).
//
// The platform-libm values of the reference (glibc for binary64, numpy float32
// for binary32; _fp.py:191-245) are replaced by correctly rounded values
// computed from the method's own twofold cores:
//   exp/expm1(x)   = RN(v0 + v1) of pexp0/pexpm10 (scaled table near underflow)
//   log/log1p(y)   = RN(r0 + r1) of the reference log core of (y, 0)
// Newton seeds use CUDA log/log1p (<= 1 ulp; the Newton step absorbs it).
#pragma once
#include "tf_common.cuh"

namespace tf {

// ------------------------------------------------------------- tables (gmem)
__device__ const double g_E64[] = {TF64_E_INIT};
__device__ const double g_C64[] = {TF64_C_INIT};
__device__ const double g_CM164[] = {TF64_CM1_INIT};
__device__ const double g_ESC64[] = {TF64_ESC_INIT};
__device__ const float g_E32[] = {TF32_E_INIT};
__device__ const float g_C32[] = {TF32_C_INIT};
__device__ const float g_CM132[] = {TF32_CM1_INIT};
__device__ const float g_ESC32[] = {TF32_ESC_INIT};
__device__ const double2 g_SEED64[] = {TF64_SEED_INIT};
__device__ const float2 g_SEED32[] = {TF32_SEED_INIT};

template <class T> struct GT;
template <> struct GT<double> {
  TF_DEV static TF<double> E(int m) { const double* p = g_E64 + 2 * (m - TF64_E_LO); return mk(__ldg(p), __ldg(p + 1)); }
  TF_DEV static TF<double> C(int n) { const double* p = g_C64 + 2 * (n - TF64_C_LO); return mk(__ldg(p), __ldg(p + 1)); }
  TF_DEV static TF<double> CM1(int n) { const double* p = g_CM164 + 2 * (n - TF64_CM1_LO); return mk(__ldg(p), __ldg(p + 1)); }
};
template <> struct GT<float> {
  TF_DEV static TF<float> E(int m) { const float* p = g_E32 + 2 * (m - TF32_E_LO); return mk(__ldg(p), __ldg(p + 1)); }
  TF_DEV static TF<float> C(int n) { const float* p = g_C32 + 2 * (n - TF32_C_LO); return mk(__ldg(p), __ldg(p + 1)); }
  TF_DEV static TF<float> CM1(int n) { const float* p = g_CM132 + 2 * (n - TF32_CM1_LO); return mk(__ldg(p), __ldg(p + 1)); }
};

// 2^k as an exact double for k in [-1074, 1023]
TF_DEV double p2d(int k) {
  if (k >= -1022) return __longlong_as_double((long long)(k + 1023) << 52);
  return __longlong_as_double(1ll << (k + 1074));
}
TF_DEV float p2f(int k) {  // k in [-149, 127]
  if (k >= -126) return __int_as_float((k + 127) << 23);
  return __int_as_float(1 << (k + 149));
}

// Python math.frexp for finite nonzero x: x = f * 2^n, 0.5 <= |f| < 1.
TF_DEV double frexp_d(double x, int* n) { return frexp(x, n); }
// Python math.ldexp(x, k) = RN(x * 2^k); single rounding via one exact power
TF_DEV double ldexp_d(double x, int k) {
  if (k > 1023) return mul(mul(x, p2d(1023)), p2d(k - 1023));  // exact scaling up
  if (k < -1074) return mul(mul(x, p2d(-1074)), p2d(k + 1074));
  return mul(x, p2d(k));
}

// biased exponent continuing through the subnormals (2^(e - 1023) <= |x|)
TF_DEV int eexp_g(double x) {
  int b = bexp(x);
  return b ? b : 12 - __clzll((long long)(ubits(x) & 0x000fffffffffffffull));
}

// reciprocal of x in [0.5, 2]: MUFU approximation + one Newton step (~2^-44)
TF_DEV double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fmaop(-x, r, 1.0);
  return fmaop(r, e, r);
}
// bare MUFU reciprocal (~2^-22): for corrections that only need a few bits
TF_DEV double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
TF_DEV float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
TF_DEV float rcp_nr(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  float e = fmaop(-x, r, 1.0f);
  return fmaop(r, e, r);
}

// ------------------------------------------------------------ exp cores
// decompose_exp (expcore.py:35-50).  Python round() is ties-to-even == rint.
template <class T> TF_DEV void decompose_exp(T x, int* m, int* n, T* y) {
  double xd = (double)x;
  double M = rint(mul(xd, 32.0));
  *y = (T)sub(xd, mul(M, 0.03125));     // exact
  int Mi = (int)M;
  int a = Mi < 0 ? -Mi : Mi;
  int hi = a >> P<T>::SPAN_SHIFT, lo = a & ((1 << P<T>::SPAN_SHIFT) - 1);
  *m = Mi < 0 ? -hi : hi;
  *n = Mi < 0 ? -lo : lo;
}
// decompose_expm1 (expcore.py:53-58)
template <class T> TF_DEV void decompose_expm1(T x, int* n, T* y) {
  double xd = (double)x;
  double M = rint(mul(xd, 128.0));
  *y = (T)sub(xd, mul(M, 0.0078125));
  *n = (int)M;
}

// Taylor coefficients N!/k! (params.py:48-59), constant memory, warp-uniform index
__constant__ double c_texp64[9] = {11880.0, 95040.0, 665280.0, 3991680.0, 19958400.0,
                                   79833600.0, 239500800.0, 479001600.0, 479001600.0};
__constant__ double c_texpm1_64[6] = {5040.0, 30240.0, 151200.0, 604800.0, 1814400.0,
                                      3628800.0};
__constant__ float c_texp32[4] = {120.f, 360.f, 720.f, 720.f};
__constant__ float c_texpm1_32[2] = {60.f, 120.f};

// _seed + taylor_exp / taylor_expm1 (expcore.py:82-116)
TF_DEV TF<double> taylor_exp_c(double y) {
  double s = add(y, 12.0);
  s = add(mul(s, y), 132.0);
  s = add(mul(s, y), 1320.0);
  TF<double> t = mk(s, 0.0);
#pragma unroll 1
  for (int k = 0; k < 9; ++k) t = t_add_d_c(t_mul_d_c(t, y), c_texp64[k]);
  return t;
}
TF_DEV TF<float> taylor_exp_c(float y) {
  float s = add(y, 6.0f);
  s = add(mul(s, y), 30.0f);
  TF<float> t = mk(s, 0.0f);
#pragma unroll 1
  for (int k = 0; k < 4; ++k) t = t_add_d_c(t_mul_d_c(t, y), c_texp32[k]);
  return t;
}
TF_DEV TF<double> taylor_expm1_c(double y) {
  double s = add(y, 10.0);
  s = add(mul(s, y), 90.0);
  s = add(mul(s, y), 720.0);
  TF<double> t = mk(s, 0.0);
#pragma unroll 1
  for (int k = 0; k < 6; ++k) t = t_add_d_c(t_mul_d_c(t, y), c_texpm1_64[k]);
  t = t_mul_d_c(t, y);
  return t_mul_c(t, mk(P<double>::INVF_V, P<double>::INVF_E));
}
TF_DEV TF<float> taylor_expm1_c(float y) {
  float s = add(y, 5.0f);
  s = add(mul(s, y), 20.0f);
  TF<float> t = mk(s, 0.0f);
#pragma unroll 1
  for (int k = 0; k < 2; ++k) t = t_add_d_c(t_mul_d_c(t, y), c_texpm1_32[k]);
  t = t_mul_d_c(t, y);
  return t_mul_c(t, mk(P<float>::INVF_V, P<float>::INVF_E));
}

// pexp0_raw (expcore.py:120-133)
template <class T> TF_DEV TF<T> pexp0_raw_c(T x) {
  if (is_nan(x)) return mk(Lim<T>::qnan(), Lim<T>::qnan());
  if (x < P<T>::LO) return mk(T(0), T(0));
  if (x > P<T>::HI) return mk(Lim<T>::inf(), Lim<T>::inf());
  int m, n;
  T y;
  decompose_exp(x, &m, &n, &y);
  TF<T> t = taylor_exp_c(y);
  return t_mul_c(GT<T>::E(m), t_mul_c(GT<T>::C(n), t));
}

// pexpm10_raw (expcore.py:138-147)
template <class T> TF_DEV TF<T> pexpm10_raw_c(T x) {
  if (is_nan(x)) return mk(Lim<T>::qnan(), Lim<T>::qnan());
  if (abits(x) <= abits(P<T>::LN2_V)) {
    int n;
    T y;
    decompose_expm1(x, &n, &y);
    TF<T> c = GT<T>::CM1(n);
    TF<T> t = taylor_expm1_c(y);
    return t_add_c(t_mul_c(c, t), t_add_c(c, t));
  }
  return t_add_d_c(pexp0_raw_c(x), T(-1));
}

// ------------------------------------------- correctly rounded libm stand-ins
// exp(x) < 2^-1075 (rounds to 0) iff x <= EXP_UNF; exp(x) rounds to inf iff
// x >= EXP_OVF (thresholds computed with mpmath, see tests/test_tables.py).
constexpr double EXP_UNF = -0x1.74910d52d3052p+9;   // < ln(2^-1075)
constexpr double EXP_OVF = 0x1.62e42fefa39fp+9;     // > ln(DBL_MAX + ulp/2)

// RN(h + l) onto the binary64 grid, where (h, l) is a twofold scaled by 2^128
// whose true value may lie in the subnormal range after unscaling.
TF_DEV double round_unscale128(double h, double l) {
  double s = add(h, l);
  if (fabs(s) >= 0x1p-894) return mul(s, 0x1p-128);  // normal after scaling: exact
  const double q = 0x1p-946;                           // 2^-1074 * 2^128
  const double C = 0x1.8p-894;                         // 1.5 * 2^52 * q
  double t = sub(add(h, C), C);                        // h rounded to multiples of q
  double r = add(sub(h, t), l);                        // h - t exact
  if (r > 0.5 * q) t = add(t, q);
  else if (r < -0.5 * q) t = sub(t, q);
  else if (fabs(r) == 0.5 * q) {                       // tie: to even multiple
    long long k = (long long)(t * 0x1p946);
    if (k & 1) t = r > 0 ? add(t, q) : sub(t, q);
  }
  return mul(t, 0x1p-128);                             // exact
}

TF_DEV double exp_cr(double x) {
  if (is_nan(x)) return x;
  if (x >= EXP_OVF) return Lim<double>::inf();
  if (x <= EXP_UNF) return 0.0;
  int m, n;
  double y;
  decompose_exp(x, &m, &n, &y);
  TF<double> ct = t_mul_u(GT<double>::C(n), taylor_exp_c(y));
  if (m <= TF64_ESC_LO + TF64_ESC_COUNT - 1) {
    const double* p = g_ESC64 + 2 * (m - TF64_ESC_LO);
    TF<double> v = t_mul_u(mk(__ldg(p), __ldg(p + 1)), ct);
    return round_unscale128(v.v, v.e);
  }
  TF<double> e = GT<double>::E(m);
  if (m > 170) {  // keep the product finite; rescaling is exact or overflows
    TF<double> v = t_mul_u(mk(mul(e.v, 0x1p-64), mul(e.e, 0x1p-64)), ct);
    return mul(add(v.v, v.e), 0x1p64);
  }
  TF<double> v = t_mul_u(e, ct);
  return add(v.v, v.e);
}

// expm1(x1) for a tiny twofold tail: x + x^2/2 + x^3/6, correctly rounded
// (|x| < 2^-27 for binary64, < 2^-16 for binary32 via binary64); also the t1
// of the fast kernels, so both paths produce the same bits.
TF_DEV double t1_tiny(double x) {
  double r = fmaop(mul(x, x), fmaop(x, 0x1.5555555555555p-3, 0.5), x);
  return zbits(x) ? x : r;
}
TF_DEV float t1_tiny(float x) {
  double d = (double)x;
  double r = fmaop(mul(d, d), fmaop(d, 0x1.5555555555555p-3, 0.5), d);
  return x == 0.0f ? x : __double2float_rn(r);
}

TF_DEV double expm1_cr(double x) {
  if (is_nan(x) || x == 0.0) return x;
  if (abits(x) < 0x3c90000000000000ull) return x;   // |x| < 2^-54
  if (x >= EXP_OVF) return Lim<double>::inf();
  if (x <= -38.0) return -1.0;
  if (x > 709.0) return exp_cr(x);                  // 1 << ulp(e^x)
  TF<double> w = pexpm10_raw_c(x);
  return add(w.v, w.e);
}

// RN to binary32 of a binary64 twofold (h + l), immune to double rounding.
TF_DEV float rn32_twofold(double h, double l) {
  float f = __double2float_rn(h);
  if (!is_finite(f) || l == 0.0) return f;
  double fd = (double)f;
  double r = add(sub(h, fd), l);                     // h - fd exact
  if (r == 0.0) return f;
  float nb = nextafterf(f, r > 0 ? Lim<float>::inf() : -Lim<float>::inf());
  if (!is_finite(nb)) return f;
  double half = 0.5 * sub((double)nb, fd);           // exact
  if (fabs(r) > fabs(half)) return nb;
  if (fabs(r) == fabs(half) && (ubits(f) & 1u)) return nb;
  return f;
}

TF_DEV float exp_cr(float x) {
  if (is_nan(x)) return x;
  if (x > 89.0f) return Lim<float>::inf();
  if (x < -104.0f) return 0.0f;
  TF<double> v = pexp0_raw_c((double)x);             // normal doubles throughout
  return rn32_twofold(v.v, v.e);
}

TF_DEV float expm1_cr(float x) {
  if (is_nan(x) || x == 0.0f) return x;
  if (x > 89.0f) return Lim<float>::inf();
  if (x < -18.0f) return -1.0f;
  TF<double> w = pexpm10_raw_c((double)x);
  return rn32_twofold(w.v, w.e);
}

// t1 = expm1(x1) (explog.py:123, 157): the tail of a coupled input is tiny
TF_DEV double expm1_t1(double x) {
  return ((uint32_t)hi32(x) & 0x7fffffffu) < 0x3e400000u ? t1_tiny(x) : expm1_cr(x);
}
TF_DEV float expm1_t1(float x) {
  return (ubits(x) & 0x7fffffffu) < 0x37800000u ? t1_tiny(x) : expm1_cr(x);
}

// ------------------------------------------------------------ log cores
// Newton seeds: the reference calls libm log / log1p (explog.py:197-199,277);
// CUDA's are within 1 ulp and the Newton step absorbs the difference.
//
// The seed is a compact table-driven log1p (relative error ~2^-52 / 2^-23,
// 10 FP64 ops, no branches) over a in [-1/2, 1], where every caller's argument
// lies: f = 1 + a split exactly as f + clo, bucket (invc, logc) from the
// exponent and 10 (binary32: 7) leading mantissa bits of f, r = f * invc - 1
// (|r| <= 2^-11, resp. 2^-8), log1p(a) = logc + log1p(r) + clo/f; |a| below
// that uses r = a directly.  The
// fast kernels read the table from shared memory, the exact path through the
// read-only cache, so both produce the same seed bits.
TF_DEV double seed_poly(double r) {  // log1p(r), |r| <= 2^-11 (+slack), degree 5
  double q = mul(r, r);
  double p = fmaop(r, 0x1.999999999999ap-3, -0.25);
  p = fmaop(r, p, 0x1.5555555555555p-2);
  p = fmaop(r, p, -0.5);
  return fmaop(q, p, r);
}
TF_DEV float seed_poly(float r) {   // degree 4
  float q = mul(r, r);
  float p = fmaop(r, -0.25f, 0x1.555556p-2f);
  p = fmaop(r, p, -0.5f);
  return fmaop(q, p, r);
}
// The table entry also carries invc - 1 (exact: invc is in [1/2, 2]),
// so the reduced argument r = (1 + a) invc - 1 is one FMA on a itself,
// fma(a, invc, invc - 1), rounded once -- no split of 1 + a into f + clo and
// no clo / f correction term (8 FP ops instead of 11).  Entry 2 NB + 1 is the
// identity (invc 1, log 0) used for |a| < 2^-11 (binary32: 2^-8), where r = a.
struct SeedE64 { double invc, invcm1, logc; };
template <class Get> TF_DEV double seed_log1p_t(double a, Get get) {
  constexpr int B = TF64_SEED_BITS, NB = 1 << B;
  double f = add(1.0, a);
  // (exponent, leading B mantissa bits) of f in [1/2, 2] as one field,
  // ((e - 1022) << B) | m, in [0, 2 NB]; the unsigned clamp keeps any other
  // argument's index in range
  const uint32_t u = ((uint32_t)hi32(f) >> (20 - B)) - (1022u << B);
  bool small = ahi(a) < 0x3f400000u;                  // |a| < 2^-11
  const int idx = small ? 2 * NB + 1 : (int)min(u, 2u * NB);
  const SeedE64 t = get(idx);
  double r = fmaop(a, t.invc, t.invcm1);
  double p = seed_poly(r);
  return add(t.logc, p);
}
struct SeedE32 { float invc, invcm1, logc; };
template <class Get> TF_DEV float seed_log1p_t(float a, Get get) {   // as binary64
  constexpr int B = TF32_SEED_BITS, NB = 1 << B;
  float f = add(1.0f, a);
  const uint32_t u = (ubits(f) >> (23 - B)) - (126u << B);
  bool small = fabsf(a) < 0x1p-8f;                    // |a| < 2^-8
  const int idx = small ? 2 * NB + 1 : (int)min(u, 2u * NB);
  const SeedE32 t = get(idx);
  float r = fmaop(a, t.invc, t.invcm1);
  float p = seed_poly(r);
  return add(t.logc, p);
}
// exact path: table seed on [-1/2, 1] (bit-identical to the fast kernels),
// CUDA log1p elsewhere (non-finite / out-of-domain arguments only)
TF_DEV double seed_log1p(double x) {
  if (x >= -0.5 && x <= 1.0)
    return seed_log1p_t(x, [](int i) {
      if (i == TF64_SEED_COUNT) return SeedE64{1.0, 0.0, 0.0};
      const double2 t = __ldg(&g_SEED64[i]);
      return SeedE64{t.x, sub(t.x, 1.0), t.y};
    });
  return log1p(x);
}
TF_DEV float seed_log1p(float x) {
  if (x >= -0.5f && x <= 1.0f)
    return seed_log1p_t(x, [](int i) {
      if (i == TF32_SEED_COUNT) return SeedE32{1.0f, 0.0f, 0.0f};
      const float2 t = __ldg(&g_SEED32[i]);
      return SeedE32{t.x, sub(t.x, 1.0f), t.y};
    });
  return log1pf(x);
}

// The Newton tolerance test is plain binary64 Python arithmetic in both lanes
// (explog.py:201, 279).
template <class T> TF_DEV bool newton_again(T r1, T r0) {
  return fabs((double)r1) > 0x1p-20 * fabs((double)r0) + 0x1p-20;
}

// _newton_log_z (explog.py:170-186)
template <class T> TF_DEV T newton_log_z_c(T z0, T z1, T r0) {
  TF<T> s = pexpm10_raw_c(T(-r0));
  T zm1 = sub(z0, T(1));
  TF<T> u;
  if (z1 == T(0)) {
    u = t_add_d_c(t_mul_d_c(s, z0), zm1);
  } else {
    TF<T> w = fast_two_sum_c(zm1, z1);
    u = t_add_c(t_mul_c(mk(z0, z1), s), w);
  }
  return add(u.v, u.e);
}

// _log_core (explog.py:188-208)
template <class T> TF_DEV TF<T> log_core_c(T y0, T y1) {
  T z0, z1;
  int n = 0;
  if (y0 < T(0.5) || y0 > T(2)) {
    if (is_finite(y0) && y0 != T(0)) z0 = (T)frexp_d((double)y0, &n);
    else z0 = y0;
    z1 = (y1 != T(0)) ? (T)ldexp_d((double)y1, -n) : T(0);
  } else {
    z0 = y0;
    z1 = y1;
  }
  // explog.py:196-199 seeds with log(z0) when y1 == z1 == 0, else with
  // log1p((z0 - 1) + z1); z0 - 1 is exact, so one log1p covers both (the seed
  // only needs to be within an ulp: the Newton step absorbs it).
  T r0 = seed_log1p(add(sub(z0, T(1)), z1));
  T r1 = newton_log_z_c(z0, z1, r0);
  if (newton_again(r1, r0)) {
    r0 = add(r0, r1);
    r1 = newton_log_z_c(z0, z1, r0);
  }
  if (n == 0) return mk(r0, r1);
  TF<T> nl = t_mul_d_c(mk(P<T>::LN2_V, P<T>::LN2_E), (T)n);
  return t_add_c(mk(r0, r1), nl);
}

// _newton_log1p_in_band (explog.py:260-274)
template <class T> TF_DEV T newton_log1p_c(T y0, T y1, T x0) {
  TF<T> s = pexpm10_raw_c(T(-x0));
  TF<T> u;
  if (y1 == T(0)) {
    TF<T> w = fast_two_sum_c(T(1), y0);
    u = t_add_d_c(t_mul_c(w, s), y0);
  } else {
    TF<T> ys = t_mul_c(mk(y0, y1), s);
    u = t_add_c(t_add_c(ys, mk(y0, y1)), s);
  }
  return add(u.v, u.e);
}

// _log1p_core (explog.py:276-282)
template <class T> TF_DEV TF<T> log1p_core_c(T y0, T y1) {
  T x0 = seed_log1p(y0);
  T x1 = newton_log1p_c(y0, y1, x0);
  if (newton_again(x1, x0)) {
    x0 = add(x0, x1);
    x1 = newton_log1p_c(y0, y1, x0);
  }
  return mk(x0, x1);
}

// log(1 + d) for an exact |d| <= 2^-20 (binary32: log_near1_g, tf_fast.cuh), correctly
// rounded up to ~2^-40 ulp: d - d^2/2 with d^2 split exactly by an FMA, then
// d^3/3 - d^4/4 + d^5/5.  Near y = 1 the log core's absolute accuracy is not
// enough to round log(y) when d has few significant bits (y = 1 + k*2^-52),
// where the exact value sits within d^3/3 of a rounding midpoint.
TF_DEV double log_near1(double d) {
  double q = mul(d, d);
  double qe = fmaop(d, d, -q);
  double c = mul(mul(q, d), fmaop(d, fmaop(d, 0.2, -0.25), 0x1.5555555555555p-2));
  double lo = fmaop(-0.5, qe, c);
  TF<double> s = fast_two_sum_u(d, mul(-0.5, q));
  return add(s.v, add(s.e, lo));
}
constexpr uint64_t NEAR1_64 = 0x3eb0000000000000ull;  // 2^-20
constexpr uint32_t NEAR1_32 = 0x3c000000u;            // 2^-7

TF_DEV double log_cr(double y) {
  if (is_nan(y) || y < 0.0) return Lim<double>::qnan();
  if (y == 0.0) return -Lim<double>::inf();
  if (is_inf(y)) return y;
  double d = sub(y, 1.0);
  if (abits(d) <= NEAR1_64) return log_near1(d);   // y in [1 - 2^-20, 1 + 2^-20]: d exact
  TF<double> c = log_core_c(y, 0.0);
  return add(c.v, c.e);
}

TF_DEV double log1p_cr(double y) {
  if (is_nan(y) || y < -1.0) return Lim<double>::qnan();
  if (y == -1.0) return -Lim<double>::inf();
  if (is_inf(y)) return y;
  if (abits(y) < 0x3c90000000000000ull) return y;   // |y| < 2^-54 (incl. +-0)
  TF<double> c;
  if (y < -0.5 || y > 1.0) {
    TF<double> w = renorm_c(t_add_d_c(mk(y, 0.0), 1.0));
    c = log_core_c(w.v, w.e);
  } else {
    c = log1p_core_c(y, 0.0);
  }
  return add(c.v, c.e);
}

TF_DEV float log_cr(float y) {
  if (is_nan(y) || y < 0.0f) return Lim<float>::qnan();
  if (y == 0.0f) return -Lim<float>::inf();
  if (is_inf(y)) return y;
  TF<double> c = log_core_c((double)y, 0.0);
  return rn32_twofold(c.v, c.e);
}

TF_DEV float log1p_cr(float y) {
  if (is_nan(y) || y < -1.0f) return Lim<float>::qnan();
  if (y == -1.0f) return -Lim<float>::inf();
  if (is_inf(y)) return y;
  if (y == 0.0f) return y;
  double yd = (double)y;
  TF<double> c;
  if (yd < -0.5 || yd > 1.0) {
    TF<double> w = renorm_c(t_add_d_c(mk(yd, 0.0), 1.0));   // exact: 1 + y
    c = log_core_c(w.v, w.e);
  } else {
    c = log1p_core_c(yd, 0.0);
  }
  return rn32_twofold(c.v, c.e);
}

// ------------------------------------------------------ public functions
// ExpLog.texp (explog.py:115-125)
template <class T> TF_DEV TF<T> texp_gen(T x0, T x1) {
  TF<T> v = pexp0_raw_c(x0);
  T z0;
  if constexpr (sizeof(T) == 8) {
    // inside [-687, 709.76] the raw core is normal and accurate: RN(v0 + v1) is
    // exp_cr(x0) without a second evaluation
    uint32_t h = (uint32_t)hi32(x0);
    bool band = (h & 0x7fffffffu) <= ((int)h < 0 ? 0x40857800u : 0x40862e14u);
    z0 = band ? add(v.v, v.e) : exp_cr(x0);
  } else {
    z0 = exp_cr(x0);
  }
  if (z0 == v.v && is_inf(z0)) return mk(z0, z0);
  T t1 = expm1_t1(x1);
  return mk(z0, add(mul(z0, t1), add(v.e, sub(v.v, z0))));
}

// ExpLog.texpm1 (explog.py:149-160)
template <class T> TF_DEV TF<T> texpm1_gen(T x0, T x1) {
  TF<T> w = pexpm10_raw_c(x0);
  T z0;
  if constexpr (sizeof(T) == 8) {
    // the same RN(w0 + w1) expm1_cr computes for these x, without re-evaluating
    bool reuse = x0 >= -38.0 && x0 <= 709.0 && abits(x0) >= 0x3c90000000000000ull;
    z0 = reuse ? add(w.v, w.e) : expm1_cr(x0);
  } else {
    z0 = expm1_cr(x0);
  }
  if (z0 == w.v && is_inf(z0)) return mk(z0, z0);
  T t1 = expm1_t1(x1);
  T tail = add(w.e, sub(w.v, z0));
  return mk(z0, add(mul(add(z0, T(1)), t1), tail));
}

// _correct (explog.py:216-223)
template <class T> TF_DEV TF<T> correct_c(TF<T> core, T lib0) {
  if (is_inf(lib0) && core.v == lib0) return mk(lib0, lib0);
  return mk(lib0, add(core.e, sub(core.v, lib0)));
}

// ExpLog.tlog (explog.py:244-249)
template <class T> TF_DEV TF<T> tlog_gen(T y0, T y1) {
  TF<T> v = renorm_c(mk(y0, y1));
  TF<T> core = log_core_c(v.v, v.e);
  T lib0;
  if constexpr (sizeof(T) == 8) {
    // y1 == 0: the core IS log_core(y0, 0), the core log_cr would recompute
    bool reuse = y1 == 0.0 && y0 > 0.0 && is_finite(y0) && abits(sub(y0, 1.0)) > NEAR1_64;
    lib0 = reuse ? add(core.v, core.e) : log_cr(y0);
  } else {
    lib0 = log_cr(y0);
  }
  return correct_c(core, lib0);
}

// ExpLog.tlog1p (explog.py:290-317) incl. tlogp for the out-of-band branch
template <class T> TF_DEV TF<T> tlog1p_gen(T y0, T y1) {
  TF<T> v = renorm_c(mk(y0, y1));
  TF<T> core, raw;
  bool oob = v.v < T(-0.5) || v.v > T(1);
  if (oob) {
    TF<T> w = renorm_c(t_add_d_c(v, T(1)));
    raw = log_core_c(w.v, w.e);
    T lw0;
    if constexpr (sizeof(T) == 8) {
      // log(w0) = log(w) - log1p(w1/w0): w is renormalized (|w1/w0| <= 2^-53)
      // and out of band (|log w0| > 0.4), so one correction term is exact enough
      bool fine = is_finite(raw.v) && is_finite(w.v) && w.v > 0.0 && !zbits(w.v);
      lw0 = fine ? add(raw.v, sub(raw.e, __ddiv_rn(w.e, w.v))) : log_cr(w.v);
    } else {
      lw0 = log_cr(w.v);
    }
    core = correct_c(raw, lw0);                                  // tlogp (239-242)
  } else {
    core = log1p_core_c(v.v, v.e);
    raw = core;
  }
  T lib0;
  if constexpr (sizeof(T) == 8) {
    // log1p(y0) = log1p(v) - log1p(y1 / (1 + y0)) (renorm is error-free); when
    // |y1| <= 2^-50 (1 + y0) the quotient is negligible beyond its first term
    // (near y0 = -1, e.g. the cfg-2 clamp, 1 + y0 is tiny and this falls back)
    double a1 = add(1.0, y0);
    bool coupled = is_finite(y0) && is_finite(raw.v) && is_finite(raw.e) && a1 > 0.0 &&
                   abits(y0) >= 0x3c90000000000000ull &&
                   (zbits(y1) || (is_finite(y1) && eexp_g(y1) + 50 <= eexp_g(a1)));
    lib0 = coupled ? add(raw.v, sub(raw.e, __ddiv_rn(y1, a1))) : log1p_cr(y0);
  } else {
    lib0 = log1p_cr(y0);
  }
  return correct_c(core, lib0);
}

// ------------------------------------------------ the sixteen siblings
// explog.py:101-325: the same cores with other arguments and finishing steps.
// renorm_fast = fast_two_sum (eft.py:163-165).
template <class T> TF_DEV TF<T> renorm_fast_c(TF<T> x) { return fast_two_sum_c(x.v, x.e); }

// texp0 / texpm10 (explog.py:105-113, 139-147): value = libm(x0), error =
// (core0 - z0) + core1
template <class T> TF_DEV TF<T> texp0_gen(T x0) {
  TF<T> v = pexp0_raw_c(x0);
  T z0;
  if constexpr (sizeof(T) == 8) {
    uint32_t h = (uint32_t)hi32(x0);
    bool band = (h & 0x7fffffffu) <= ((int)h < 0 ? 0x40857800u : 0x40862e14u);
    z0 = band ? add(v.v, v.e) : exp_cr(x0);
  } else {
    z0 = exp_cr(x0);
  }
  if (z0 == v.v && is_inf(z0)) return mk(z0, z0);
  return mk(z0, add(sub(v.v, z0), v.e));
}
template <class T> TF_DEV TF<T> texpm10_gen(T x0) {
  TF<T> w = pexpm10_raw_c(x0);
  T z0 = expm1_cr(x0);
  if (z0 == w.v && is_inf(z0)) return mk(z0, z0);
  return mk(z0, add(sub(w.v, z0), w.e));
}

// _plog1p0_raw (explog.py:284-288)
template <class T> TF_DEV TF<T> plog1p0_raw_c(T y0) {
  if (y0 < T(-0.5) || y0 > T(1)) {
    TF<T> v = renorm_c(mk(T(1), y0));
    return log_core_c(v.v, v.e);
  }
  return log1p_core_c(y0, T(0));
}

// _plog1p_raw (explog.py:290-294) incl. tlogp for the out-of-band branch
template <class T> TF_DEV TF<T> plog1p_raw_c(TF<T> y) {
  if (y.v < T(-0.5) || y.v > T(1)) {
    TF<T> w = renorm_c(t_add_d_c(y, T(1)));
    return correct_c(log_core_c(w.v, w.e), log_cr(w.v));
  }
  return log1p_core_c(y.v, y.e);
}

enum Fn {
  FN_TEXP = 0, FN_TEXPM1 = 1, FN_TLOG = 2, FN_TLOG1P = 3,
  FN_PEXP0 = 4, FN_TEXP0 = 5, FN_TEXPP = 6, FN_PEXP = 7,
  FN_PEXPM10 = 8, FN_TEXPM10 = 9, FN_TEXPM1P = 10, FN_PEXPM1 = 11,
  FN_PLOG0 = 12, FN_TLOG0 = 13, FN_TLOGP = 14, FN_PLOG = 15,
  FN_PLOG1P0 = 16, FN_TLOG1P0 = 17, FN_TLOG1PP = 18, FN_PLOG1P = 19,
  FN_COUNT = 20
};

// functions of a plain ("dotted") argument: x1 is not read
__host__ __device__ constexpr bool dotted_fn(int fn) {
  return fn == FN_PEXP0 || fn == FN_TEXP0 || fn == FN_PEXPM10 || fn == FN_TEXPM10 ||
         fn == FN_PLOG0 || fn == FN_TLOG0 || fn == FN_PLOG1P0 || fn == FN_TLOG1P0;
}

template <class T, int FN> __device__ __noinline__ TF<T> eval_gen(T x0, T x1) {
  const T INF = Lim<T>::inf();
  if constexpr (FN == FN_TEXP || FN == FN_TEXPP) return texp_gen(x0, x1);
  else if constexpr (FN == FN_TEXPM1 || FN == FN_TEXPM1P) return texpm1_gen(x0, x1);
  else if constexpr (FN == FN_TLOG) return tlog_gen(x0, x1);
  else if constexpr (FN == FN_TLOG1P) return tlog1p_gen(x0, x1);
  else if constexpr (FN == FN_PEXP0) return renorm_fast_c(pexp0_raw_c(x0));
  else if constexpr (FN == FN_TEXP0) return texp0_gen(x0);
  else if constexpr (FN == FN_PEXP) return renorm_fast_c(texp_gen(x0, x1));
  else if constexpr (FN == FN_PEXPM10) return renorm_fast_c(pexpm10_raw_c(x0));
  else if constexpr (FN == FN_TEXPM10) return texpm10_gen(x0);
  else if constexpr (FN == FN_PEXPM1) return renorm_fast_c(texpm1_gen(x0, x1));
  else if constexpr (FN == FN_PLOG0) {                       // explog.py:225-232
    if (x0 == T(0)) return mk(-INF, -INF);
    if (x0 == INF) return mk(INF, INF);
    return renorm_fast_c(log_core_c(x0, T(0)));
  } else if constexpr (FN == FN_TLOG0) {                     // explog.py:234-237
    return correct_c(log_core_c(x0, T(0)), log_cr(x0));
  } else if constexpr (FN == FN_TLOGP) {                     // explog.py:239-242
    return correct_c(log_core_c(x0, x1), log_cr(x0));
  } else if constexpr (FN == FN_PLOG) {                      // explog.py:251-258
    if (x0 == T(0)) return mk(-INF, -INF);
    if (x0 == INF) return mk(INF, INF);
    return renorm_fast_c(log_core_c(x0, x1));
  } else if constexpr (FN == FN_PLOG1P0) {                   // explog.py:296-303
    if (x0 == T(-1)) return mk(-INF, -INF);
    if (x0 == INF) return mk(INF, INF);
    return renorm_fast_c(plog1p0_raw_c(x0));
  } else if constexpr (FN == FN_TLOG1P0) {                   // explog.py:305-308
    return correct_c(plog1p0_raw_c(x0), log1p_cr(x0));
  } else if constexpr (FN == FN_TLOG1PP) {                   // explog.py:310-312
    return correct_c(plog1p_raw_c(mk(x0, x1)), log1p_cr(x0));
  } else {                                                   // plog1p, explog.py:319-325
    if (x0 == T(-1) && x1 == T(0)) return mk(-INF, -INF);
    if (x0 == INF) return mk(INF, INF);
    return renorm_fast_c(plog1p_raw_c(mk(x0, x1)));
  }
}

}  // namespace tf
