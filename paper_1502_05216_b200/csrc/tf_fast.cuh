// tf_fast.cuh -- the admission-band ("fast") paths of the four functions.
//
// Each fast path executes exactly the reference operation sequence (same
// IEEE ops, same order, fused residual = the reference "fma" backend) but
// WITHOUT the per-op _special checks: its admission band proves that every
// intermediate is finite, that the table indices are in range, that the
// Newton step does not need a second iteration, and that the correctly
// rounded value part can be obtained from the twofold core.  Elements outside
// the band return ok=false and are re-evaluated by the exact path
// (tf_general.cuh) through the per-warp rare queue, so divergence never
// costs more than one full-warp pass of the exact path per 32 rare elements.
//
// Integer-pipe work (band tests, index arithmetic, frexp/ldexp via exponent
// fields) is kept off the FP64/FP32 pipe, whose cycles are the roofline.
#pragma once
#include "tf_general.cuh"

namespace tf {

// -------------------------------------------------------- shared tables
template <class T> struct V2;
template <> struct V2<double> { typedef double2 t; };
template <> struct V2<float> { typedef float2 t; };

template <class T> struct STab {
  typename V2<T>::t E[P<T>::E_N];
  typename V2<T>::t C[P<T>::C_N];
  typename V2<T>::t CM1[P<T>::CM1_N];
  typename V2<T>::t ESC[sizeof(T) == 8 ? TF64_ESC_COUNT : TF32_ESC_COUNT];
};

template <class T> __device__ void load_tables(STab<T>& s) {
  const T* srcE = sizeof(T) == 8 ? (const T*)g_E64 : (const T*)g_E32;
  const T* srcC = sizeof(T) == 8 ? (const T*)g_C64 : (const T*)g_C32;
  const T* srcM = sizeof(T) == 8 ? (const T*)g_CM164 : (const T*)g_CM132;
  const T* srcS = sizeof(T) == 8 ? (const T*)g_ESC64 : (const T*)g_ESC32;
  constexpr int NS = sizeof(T) == 8 ? TF64_ESC_COUNT : TF32_ESC_COUNT;
  for (int i = threadIdx.x; i < P<T>::E_N; i += blockDim.x) { s.E[i].x = srcE[2 * i]; s.E[i].y = srcE[2 * i + 1]; }
  for (int i = threadIdx.x; i < P<T>::C_N; i += blockDim.x) { s.C[i].x = srcC[2 * i]; s.C[i].y = srcC[2 * i + 1]; }
  for (int i = threadIdx.x; i < P<T>::CM1_N; i += blockDim.x) { s.CM1[i].x = srcM[2 * i]; s.CM1[i].y = srcM[2 * i + 1]; }
  for (int i = threadIdx.x; i < NS; i += blockDim.x) { s.ESC[i].x = srcS[2 * i]; s.ESC[i].y = srcS[2 * i + 1]; }
}

template <class T, class V> TF_DEV TF<T> tv(V a) { return mk(a.x, a.y); }

// --------------------------------------------------- band constants
// |x| bit patterns used by the integer band tests
constexpr uint64_t B64_TEXP_POS = 0x40862e147ae147aeull;  // 709.76 -> exp < DBL_MAX
constexpr uint64_t B64_TEXP_NEG = 0x4085780000000000ull;  // 687.0 -> exp > 2^-991
constexpr uint64_t B64_X1_TINY = 0x3e40000000000000ull;   // 2^-27: t1 polynomial is CR
constexpr uint64_t B64_TINY54 = 0x3c90000000000000ull;    // 2^-54
constexpr uint64_t B64_LN2 = 0x3fe62e42fefa39efull;       // LN2 value part
constexpr uint64_t B64_HALF = 0x3fe0000000000000ull;
constexpr uint64_t B64_ONE = 0x3ff0000000000000ull;
constexpr uint64_t B64_TWO = 0x4000000000000000ull;
constexpr uint32_t B32_TEXP_POS = 0x42b170a4u;  // 88.72 (< ln FLT_MAX)
constexpr uint32_t B32_TEXP_NEG = 0x42ae999au;  // 87.3  (exp > 2^-126)
constexpr uint32_t B32_LO = 0x42ce8ed0u;        // |lo_bound| 103.27893
constexpr uint32_t B32_X1_TINY = 0x37800000u;   // 2^-16
constexpr uint32_t B32_TINY25 = 0x33000000u;    // 2^-25
constexpr uint32_t B32_LN2 = 0x3f317218u;
constexpr uint32_t B32_HALF = 0x3f000000u;
constexpr uint32_t B32_ONE = 0x3f800000u;
constexpr uint32_t B32_TWO = 0x40000000u;

TF_DEV bool sgn(double x) { return hi32(x) < 0; }
TF_DEV bool sgn(float x) { return (int)ubits(x) < 0; }

// ---------------------------------------------------- unchecked cores
TF_DEV TF<double> taylor_exp_u(double y) {  // expcore.py:82-105, N=12
  double s = add(y, 12.0);
  s = add(mul(s, y), 132.0);
  s = add(mul(s, y), 1320.0);
  TF<double> t = mk(s, 0.0);
  const double c[9] = {11880.0, 95040.0, 665280.0, 3991680.0, 19958400.0,
                       79833600.0, 239500800.0, 479001600.0, 479001600.0};
#pragma unroll
  for (int k = 0; k < 9; ++k) t = t_add_d_u(t_mul_d_u(t, y), c[k]);
  return t;
}
TF_DEV TF<float> taylor_exp_u(float y) {    // N=6, 2 dotted steps
  float s = add(y, 6.0f);
  s = add(mul(s, y), 30.0f);
  TF<float> t = mk(s, 0.0f);
  const float c[4] = {120.f, 360.f, 720.f, 720.f};
#pragma unroll
  for (int k = 0; k < 4; ++k) t = t_add_d_u(t_mul_d_u(t, y), c[k]);
  return t;
}
TF_DEV TF<double> taylor_expm1_u(double y) {  // expcore.py:107-116, N_m1=10
  double s = add(y, 10.0);
  s = add(mul(s, y), 90.0);
  s = add(mul(s, y), 720.0);
  TF<double> t = mk(s, 0.0);
  const double c[6] = {5040.0, 30240.0, 151200.0, 604800.0, 1814400.0, 3628800.0};
#pragma unroll
  for (int k = 0; k < 6; ++k) t = t_add_d_u(t_mul_d_u(t, y), c[k]);
  t = t_mul_d_u(t, y);
  return t_mul_u(t, mk(P<double>::INVF_V, P<double>::INVF_E));
}
TF_DEV TF<float> taylor_expm1_u(float y) {    // N_m1=5
  float s = add(y, 5.0f);
  s = add(mul(s, y), 20.0f);
  TF<float> t = mk(s, 0.0f);
  const float c[2] = {60.f, 120.f};
#pragma unroll
  for (int k = 0; k < 2; ++k) t = t_add_d_u(t_mul_d_u(t, y), c[k]);
  t = t_mul_d_u(t, y);
  return t_mul_u(t, mk(P<float>::INVF_V, P<float>::INVF_E));
}

// decompose_exp via the magic constant: M = round-half-even(x * 32) in the
// low word, y = x - M/32 exact (the reference's two ops give the same value).
TF_DEV void decomp_exp_u(double x, int& m, int& n, double& y) {
  double t = fmaop(x, 32.0, MAGIC);
  int M = __double2loint(t);
  y = fmaop(sub(t, MAGIC), -0.03125, x);
  int a = abs(M);
  m = M < 0 ? -(a >> 7) : (a >> 7);
  n = M < 0 ? -(a & 127) : (a & 127);
}
TF_DEV void decomp_exp_u(float x, int& m, int& n, float& y) {
  const float MG = 12582912.0f;  // 1.5 * 2^23
  float t = fmaop(x, 32.0f, MG);
  int M = (int)ubits(t) - 0x4b400000;
  y = fmaop(sub(t, MG), -0.03125f, x);
  int a = abs(M);
  m = M < 0 ? -(a >> 6) : (a >> 6);
  n = M < 0 ? -(a & 63) : (a & 63);
}
TF_DEV void decomp_expm1_u(double x, int& n, double& y) {
  double t = fmaop(x, 128.0, MAGIC);
  n = __double2loint(t);
  y = fmaop(sub(t, MAGIC), -0.0078125, x);
}
TF_DEV void decomp_expm1_u(float x, int& n, float& y) {
  const float MG = 12582912.0f;
  float t = fmaop(x, 128.0f, MG);
  n = (int)ubits(t) - 0x4b400000;
  y = fmaop(sub(t, MG), -0.0078125f, x);
}

// pexpm10_raw, in-band branch only (expcore.py:142-146)
template <class T> TF_DEV TF<T> pexpm10_inband_u(const STab<T>& tb, T x) {
  int n;
  T y;
  decomp_expm1_u(x, n, y);
  TF<T> c = tv<T>(tb.CM1[n - P<T>::CM1_LO]);
  TF<T> t = taylor_expm1_u(y);
  return t_add_u(t_mul_u(c, t), t_add_u(c, t));
}

// expm1(x1) for a tiny twofold tail: x + x^2/2 + x^3/6, correctly rounded
// (|x| < 2^-27 for binary64, < 2^-16 for binary32 via binary64).
TF_DEV double t1_tiny(double x) {
  double r = fmaop(mul(x, x), fmaop(x, 0x1.5555555555555p-3, 0.5), x);
  return abits(x) == 0 ? x : r;
}
TF_DEV float t1_tiny(float x) {
  double d = (double)x;
  double r = fmaop(mul(d, d), fmaop(d, 0x1.5555555555555p-3, 0.5), d);
  return abits(x) == 0 ? x : __double2float_rn(r);
}

// 2^k for k in [-1074, 1023], branch-free
TF_DEV double p2d_bf(int k) {
  long long nb = (long long)(k + 1023) << 52;
  long long sb = 1ll << ((k + 1074) & 63);
  return __longlong_as_double(k >= -1022 ? nb : sb);
}
TF_DEV float p2f_bf(int k) {  // k in [-149, 127]
  int nb = (k + 127) << 23;
  int sb = 1 << ((k + 149) & 31);
  return __int_as_float(k >= -126 ? nb : sb);
}

// "second Newton iteration cannot fire": |r1| < 2^-21 * max(|r0|, 1), a
// conservative integer form of explog.py:351/429 (binary64 arithmetic there).
TF_DEV bool newton_quiet(double r1, double r0) {
  int e1 = bexp(r1), e0 = bexp(r0);
  return e1 + 22 <= max(e0, 1023);
}
TF_DEV bool newton_quiet(float r1, float r0) {
  int e1 = bexp(r1), e0 = bexp(r0);
  return e1 + 22 <= max(e0, 127);
}

// ================================================================ texp
TF_DEV bool fast_texp(const STab<double>& tb, double x0, double x1, double& z0, double& z1) {
  bool ok = abits(x0) <= (sgn(x0) ? B64_TEXP_NEG : B64_TEXP_POS);
  ok &= abits(x1) < B64_X1_TINY;
  x0 = ok ? x0 : 0.0;
  int m, n;
  double y;
  decomp_exp_u(x0, m, n, y);
  TF<double> t = taylor_exp_u(y);
  TF<double> ct = t_mul_u(tv<double>(tb.C[n - P<double>::C_LO]), t);
  TF<double> v = t_mul_u(tv<double>(tb.E[m - P<double>::E_LO]), ct);
  z0 = add(v.v, v.e);                                   // CR exp(x0)
  double t1 = t1_tiny(x1);
  z1 = add(mul(z0, t1), add(v.e, sub(v.v, z0)));       // explog.py:275
  return ok;
}

TF_DEV bool fast_texp(const STab<float>& tb, float x0, float x1, float& z0, float& z1) {
  bool ok = abits(x0) <= (sgn(x0) ? B32_TEXP_NEG : B32_TEXP_POS);
  ok &= abits(x1) < B32_X1_TINY;
  x0 = ok ? x0 : 0.0f;
  int m, n;
  float y;
  decomp_exp_u(x0, m, n, y);
  TF<float> t = taylor_exp_u(y);
  TF<float> ct = t_mul_u(tv<float>(tb.C[n - P<float>::C_LO]), t);
  TF<float> v = t_mul_u(tv<float>(tb.E[m - P<float>::E_LO]), ct);
  // value part: near the subnormal range use the 2^64-scaled coarse table so
  // the twofold keeps full precision (result is normal: exact unscaling)
  bool scaled = m <= -35;  // e^(2m) < 2^-100: residuals would underflow
  int is = scaled ? m - TF32_ESC_LO : 0;
  TF<float> es = tv<float>(tb.ESC[is]);
  TF<float> vs = t_mul_u(scaled ? es : tv<float>(tb.E[m - P<float>::E_LO]), ct);
  z0 = mul(add(vs.v, vs.e), scaled ? 0x1p-64f : 1.0f);
  float t1 = t1_tiny(x1);
  z1 = add(mul(z0, t1), add(v.e, sub(v.v, z0)));
  return ok;
}

// ============================================================== texpm1
// binary64: the in-band core is the bulk (cfg 2: 99.5%)
TF_DEV bool fast_texpm1(const STab<double>& tb, double x0, double x1, double& z0, double& z1) {
  bool ok = abits(x0) <= B64_LN2;
  ok &= abits(x1) < B64_X1_TINY;
  x0 = ok ? x0 : 0.0;
  TF<double> w = pexpm10_inband_u(tb, x0);
  z0 = abits(x0) < B64_TINY54 ? x0 : add(w.v, w.e);    // CR expm1(x0)
  double t1 = t1_tiny(x1);
  double tail = add(w.e, sub(w.v, z0));
  z1 = add(mul(add(z0, 1.0), t1), tail);               // explog.py:309-310
  return ok;
}

// binary32: the pexp0 - 1 fallback is the bulk (cfg 4: 99.2%)
TF_DEV bool fast_texpm1(const STab<float>& tb, float x0, float x1, float& z0, float& z1) {
  uint32_t ax = abits(x0);
  bool ok = ax > B32_LN2 && ax <= (sgn(x0) ? B32_LO : B32_TEXP_POS);
  ok &= abits(x1) < B32_X1_TINY;
  x0 = ok ? x0 : 1.0f;
  int m, n;
  float y;
  decomp_exp_u(x0, m, n, y);
  TF<float> t = taylor_exp_u(y);
  TF<float> v = t_mul_u(tv<float>(tb.E[m - P<float>::E_LO]), t_mul_u(tv<float>(tb.C[n - P<float>::C_LO]), t));
  TF<float> w = t_add_d_u(v, -1.0f);                    // expcore.py:147
  z0 = add(w.v, w.e);
  float t1 = t1_tiny(x1);
  float tail = add(w.e, sub(w.v, z0));
  z1 = add(mul(add(z0, 1.0f), t1), tail);
  return ok;
}

// ================================================================= tlog
// explog.py:394-399 -> _log_core (338-358) -> _newton_log_z (320-336),
// with the value part replaced by a correctly rounded log(y0):
//   log(y0) = log(v) - log1p(d),  d = (v - y0)/y0,  v = renorm(y0 + y1).
TF_DEV bool fast_tlog(const STab<double>& tb, double y0, double y1, double& z0, double& z1) {
  uint32_t eb0 = (uint32_t)hi32(y0) >> 20;          // sign|exponent
  bool ok = eb0 - 1u < 2046u;                        // positive normal
  ok &= abits(y1) == 0 || bexp(y1) + 50 <= (int)eb0;
  y0 = ok ? y0 : 1.0;
  y1 = ok ? y1 : 0.0;
  TF<double> v = renorm_u(mk(y0, y1));
  uint64_t vb = ubits(v.v);
  bool band = vb >= B64_HALF && vb <= B64_TWO;
  int n = band ? 0 : (int)(vb >> 52) - 1022;
  double zc0 = band ? v.v : __longlong_as_double((vb & 0x800fffffffffffffull) | (1022ull << 52));
  double zc1 = band ? v.e : (abits(v.e) == 0 ? 0.0 : mul(v.e, p2d_bf(-n)));
  double r0 = seed_log1p(add(sub(zc0, 1.0), zc1));
  ok &= abits(r0) <= B64_LN2;
  TF<double> s = pexpm10_inband_u(tb, -r0);
  TF<double> w = fast_two_sum_u(sub(zc0, 1.0), zc1);
  TF<double> u = t_add_u(t_mul_u(mk(zc0, zc1), s), w);
  double r1 = add(u.v, u.e);
  ok &= newton_quiet(r1, r0);
  TF<double> nl = t_mul_d_u(mk(P<double>::LN2_V, P<double>::LN2_E), (double)n);
  TF<double> core = t_add_u(mk(r0, r1), nl);
  // renorm is error-free, so v - y0 == y1 exactly: log(y0) = log(v) - log1p(d),
  // d = y1 / y0 = ys1 / ys0 (both scaled by 2^-n, ys0 in [0.5, 2]) to ~2^-100.
  double sc = p2d_bf(-n);
  double ys0 = mul(y0, sc), ys1 = mul(y1, sc);
  double rc = rcp_nr(ys0);
  double d0 = mul(ys1, rc);
  double d1 = mul(fmaop(-d0, ys0, ys1), rc);
  TF<double> a = two_sum_u(core.v, -d0);
  double tail = add(add(a.e, core.e), sub(mul(mul(0.5, d0), d0), d1));
  z0 = add(a.v, tail);
  double dl = sub(y0, 1.0);                          // exact near 1
  if (abits(dl) <= NEAR1_64) z0 = log_near1(dl);
  z1 = add(core.e, sub(core.v, z0));                 // _correct (372-373)
  return ok;
}

TF_DEV bool fast_tlog(const STab<float>& tb, float y0, float y1, float& z0, float& z1) {
  uint32_t eb0 = ubits(y0) >> 23;
  bool ok = eb0 - 1u < 254u;
  ok &= abits(y1) == 0 || bexp(y1) + 21 <= (int)eb0;
  y0 = ok ? y0 : 1.0f;
  y1 = ok ? y1 : 0.0f;
  TF<float> v = renorm_u(mk(y0, y1));
  uint32_t vb = ubits(v.v);
  bool band = vb >= B32_HALF && vb <= B32_TWO;
  int n = band ? 0 : (int)(vb >> 23) - 126;
  float zc0 = band ? v.v : __int_as_float((vb & 0x807fffffu) | (126u << 23));
  float zc1 = band ? v.e : (abits(v.e) == 0 ? 0.0f : mul(v.e, p2f_bf(-n)));
  float r0 = seed_log1p(add(sub(zc0, 1.0f), zc1));
  ok &= abits(r0) <= B32_LN2;
  TF<float> s = pexpm10_inband_u(tb, -r0);
  TF<float> w = fast_two_sum_u(sub(zc0, 1.0f), zc1);
  TF<float> u = t_add_u(t_mul_u(mk(zc0, zc1), s), w);
  float r1 = add(u.v, u.e);
  ok &= newton_quiet(r1, r0);
  TF<float> nl = t_mul_d_u(mk(P<float>::LN2_V, P<float>::LN2_E), (float)n);
  TF<float> core = t_add_u(mk(r0, r1), nl);
  float sc = p2f_bf(-n);
  float ys0 = mul(y0, sc), ys1 = mul(y1, sc);
  float rc = rcp_nr(ys0);
  float d0 = mul(ys1, rc);
  float d1 = mul(fmaop(-d0, ys0, ys1), rc);
  TF<float> a = two_sum_u(core.v, -d0);
  float tail = add(add(a.e, core.e), sub(mul(mul(0.5f, d0), d0), d1));
  z0 = add(a.v, tail);
  float dl = sub(y0, 1.0f);
  if (abits(dl) <= NEAR1_32) z0 = log_near1(dl);
  z1 = add(core.e, sub(core.v, z0));
  return ok;
}

// =============================================================== tlog1p
// In-band branch of _plog1p_raw (explog.py:440-444, 410-432); the
// out-of-band branch (y0 < -1/2 or y0 > 1) goes to the exact path.
// log1p(y0) = log1p(v) - log1p(d), d = (v - y0)/(1 + y0), |d| ~ 2^-53 |log1p(y0)|.
template <class T> TF_DEV bool fast_tlog1p(const STab<T>& tb, T y0, T y1, T& z0, T& z1) {
  constexpr bool D = sizeof(T) == 8;
  const int SMALL = D ? 50 : 21;
  bool ok = is_finite(y0) && (abits(y1) == 0 || bexp(y1) + SMALL <= bexp(y0));
  y0 = ok ? y0 : T(0);
  y1 = ok ? y1 : T(0);
  TF<T> v = renorm_u(mk(y0, y1));
  if (D) ok &= abits(v.v) <= (sgn(v.v) ? (uint64_t)B64_HALF : (uint64_t)B64_ONE);
  else ok &= abits(v.v) <= (sgn(v.v) ? B32_HALF : B32_ONE);
  v.v = ok ? v.v : T(0);
  v.e = ok ? v.e : T(0);
  T x0 = seed_log1p(v.v);
  TF<T> s = pexpm10_inband_u(tb, T(-x0));
  TF<T> u;
  if (v.e == T(0)) {                                  // explog.py:418-420
    TF<T> w = fast_two_sum_u(T(1), v.v);
    u = t_add_d_u(t_mul_u(w, s), v.v);
  } else {                                            // explog.py:421-423
    TF<T> ys = t_mul_u(v, s);
    u = t_add_u(t_add_u(ys, v), s);
  }
  T x1 = add(u.v, u.e);
  ok &= newton_quiet(x1, x0);
  bool tiny = D ? abits(y0) < B64_TINY54 : abits(y0) < (uint64_t)B32_TINY25;
  T d = mul(y1, rcp_nr(add(T(1), y0)));              // v - y0 == y1 exactly
  z0 = tiny ? y0 : add(x0, sub(x1, d));
  z1 = add(x1, sub(x0, z0));                          // _correct (372-373)
  return ok;
}

template <class T, int FN> TF_DEV bool fast_eval(const STab<T>& tb, T x0, T x1, T& z0, T& z1) {
  if (FN == FN_TEXP) return fast_texp(tb, x0, x1, z0, z1);
  if (FN == FN_TEXPM1) return fast_texpm1(tb, x0, x1, z0, z1);
  if (FN == FN_TLOG) return fast_tlog(tb, x0, x1, z0, z1);
  return fast_tlog1p(tb, x0, x1, z0, z1);
}

}  // namespace tf
