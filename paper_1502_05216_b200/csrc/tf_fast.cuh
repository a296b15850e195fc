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
  typename V2<T>::t SEED[(sizeof(T) == 8 ? TF64_SEED_COUNT : TF32_SEED_COUNT) + 1];
  T SEEDM1[(sizeof(T) == 8 ? TF64_SEED_COUNT : TF32_SEED_COUNT) + 1];   // invc - 1
};

// SEED (the log seed table, 32 KB in binary64) is staged only by the
// logarithm kernels
template <class T> __device__ void load_tables(STab<T>& s, bool seed) {
  const T* srcE = sizeof(T) == 8 ? (const T*)g_E64 : (const T*)g_E32;
  const T* srcC = sizeof(T) == 8 ? (const T*)g_C64 : (const T*)g_C32;
  const T* srcM = sizeof(T) == 8 ? (const T*)g_CM164 : (const T*)g_CM132;
  const T* srcS = sizeof(T) == 8 ? (const T*)g_ESC64 : (const T*)g_ESC32;
  constexpr int NS = sizeof(T) == 8 ? TF64_ESC_COUNT : TF32_ESC_COUNT;
  for (int i = threadIdx.x; i < P<T>::E_N; i += blockDim.x) { s.E[i].x = srcE[2 * i]; s.E[i].y = srcE[2 * i + 1]; }
  for (int i = threadIdx.x; i < P<T>::C_N; i += blockDim.x) { s.C[i].x = srcC[2 * i]; s.C[i].y = srcC[2 * i + 1]; }
  for (int i = threadIdx.x; i < P<T>::CM1_N; i += blockDim.x) { s.CM1[i].x = srcM[2 * i]; s.CM1[i].y = srcM[2 * i + 1]; }
  for (int i = threadIdx.x; i < NS; i += blockDim.x) { s.ESC[i].x = srcS[2 * i]; s.ESC[i].y = srcS[2 * i + 1]; }
  const typename V2<T>::t* srcD =
      sizeof(T) == 8 ? (const typename V2<T>::t*)g_SEED64 : (const typename V2<T>::t*)g_SEED32;
  constexpr int ND = sizeof(T) == 8 ? TF64_SEED_COUNT : TF32_SEED_COUNT;
  if (seed) {
    for (int i = threadIdx.x; i < ND; i += blockDim.x) {
      s.SEED[i] = srcD[i];
      s.SEEDM1[i] = sub(srcD[i].x, T(1));
    }
    if (threadIdx.x == 0) {                       // identity entry for tiny arguments
      s.SEED[ND].x = T(1);
      s.SEED[ND].y = T(0);
      s.SEEDM1[ND] = T(0);
    }
  }
}
// seed entries from the staged tables
TF_DEV SeedE64 seed_entry(const STab<double>& tb, int i) {
  return SeedE64{tb.SEED[i].x, tb.SEEDM1[i], tb.SEED[i].y};
}
TF_DEV SeedE32 seed_entry(const STab<float>& tb, int i) {
  return SeedE32{tb.SEED[i].x, tb.SEEDM1[i], tb.SEED[i].y};
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

// the same bands as high words (conservative where marked "<")
constexpr uint32_t H64_TEXP_POS = 0x40862e14u;  // |x| <= 709.76...
constexpr uint32_t H64_TEXP_NEG = 0x408622e1u;  // |x| < 708.3907 (exp normal)
constexpr uint32_t H64_X1_TINY = 0x3e400000u;   // < 2^-27
constexpr uint32_t H64_TINY54 = 0x3c900000u;    // < 2^-54
constexpr uint32_t H64_LN2 = 0x3fe62e42u;       // < LN2 (slightly conservative)
constexpr uint32_t H64_HALF = 0x3fe00000u;      // < 0.5
constexpr uint32_t H64_ONE = 0x3ff00000u;       // < 1
constexpr uint32_t H64_NEAR1 = 0x3eb00000u;     // < 2^-20

// biased exponent that keeps counting down through the subnormals (so a
// subnormal error part still compares by magnitude): 2^(eexp - bias) <= |x|
TF_DEV int eexp(double x) {
  int b = bexp(x);
  unsigned long long m = ubits(x) & 0x000fffffffffffffull;
  return b ? b : 12 - __clzll((long long)m);
}
TF_DEV int eexp(float x) {
  int b = bexp(x);
  return b ? b : 9 - __clz((int)(ubits(x) & 0x7fffffu));
}

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

// Rolled, lane-vectorised Taylor-Horner cores: one loop iteration performs
// one twofold Horner step for all VW lanes, so the VW independent dependency
// chains interleave while the hot code stays a few hundred bytes (a fully
// unrolled 2-lane tlog1p was ~24 KB of SASS and stalled on instruction fetch).
// Coefficients N!/k! come from constant memory with a warp-uniform index.
// t_mul_d (eft.py:214-219) of a twofold whose error part is +0 -- the first
// Horner step of every Taylor core, t = (s, 0): the reference's x1 * b + e
// rounds the product 0 * b, which is exact (+-0 for finite b), so the single
// FMA RN(x1 * b + e) is the same IEEE operation, signed zeros included (the
// sign of an exact-zero sum follows the addition rules in both).  One FP op
// fewer per lane and core.
template <class T> TF_DEV TF<T> t_mul_d_z(TF<T> x, T b) {
  T v = mul(x.v, b);
  T e = fmaop(x.v, b, -v);
  return mk(v, fmaop(x.e, b, e));
}
template <int VW> TF_DEV void taylor_exp_v(const double (&y)[VW], TF<double> (&t)[VW]) {
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    double s = add(y[e], 12.0);
    s = add(mul(s, y[e]), 132.0);
    s = add(mul(s, y[e]), 1320.0);
    t[e] = mk(s, 0.0);
  }
#pragma unroll
  for (int e = 0; e < VW; ++e) t[e] = t_add_d_u(t_mul_d_z(t[e], y[e]), c_texp64[0]);
#pragma unroll
  for (int k = 1; k < 9; ++k) {
    const double c = c_texp64[k];
#pragma unroll
    for (int e = 0; e < VW; ++e) t[e] = t_add_d_u(t_mul_d_u(t[e], y[e]), c);
  }
}
// t_mul_d (eft.py:214-219) for lane pairs without a sign-flip instruction:
// with nb = -b precomputed, fma(x0, nb, v) = RN(v - x0 b) = -e exactly, and
// x1 b + e = x1 b - (-e) is the same IEEE addition.
TF_DEV TF<f2> t_mul_d_p(TF<f2> x, f2 b, f2 nb) {
  f2 v = mul(x.v, b);
  f2 ne = fmaop(x.v, nb, v);
  return mk(v, sub(mul(x.e, b), ne));
}
// the same with x.e = +0 (t_mul_d_z): RN(x1 b - ne) as one FFMA2
TF_DEV TF<f2> t_mul_d_pz(TF<f2> x, f2 b, f2 nb) {
  f2 v = mul(x.v, b);
  f2 ne = fmaop(x.v, nb, v);
  return mk(v, fmaop(x.e, b, -ne));
}

template <int VW> TF_DEV void taylor_exp_v(const float (&y)[VW], TF<float> (&t)[VW]) {
  if constexpr (VW % 2 == 0) {  // lane pairs on FADD2/FMUL2/FFMA2
    constexpr int NP = VW / 2;
    f2 yp[NP], nyp[NP];
    TF<f2> tp[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      yp[p] = pk(y[2 * p], y[2 * p + 1]);
      nyp[p] = pk(-y[2 * p], -y[2 * p + 1]);
      f2 s = add(yp[p], splat(6.0f));
      s = add(mul(s, yp[p]), splat(30.0f));
      tp[p] = mk(s, splat(0.0f));
    }
#pragma unroll
    for (int p = 0; p < NP; ++p)
      tp[p] = t_add_d_u(t_mul_d_pz(tp[p], yp[p], nyp[p]), splat(c_texp32[0]));
#pragma unroll
    for (int k = 1; k < 4; ++k) {
      const f2 c = splat(c_texp32[k]);
#pragma unroll
      for (int p = 0; p < NP; ++p) tp[p] = t_add_d_u(t_mul_d_p(tp[p], yp[p], nyp[p]), c);
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      t[2 * p] = mk(lo(tp[p].v), lo(tp[p].e));
      t[2 * p + 1] = mk(hi(tp[p].v), hi(tp[p].e));
    }
  } else {
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    float s = add(y[e], 6.0f);
    s = add(mul(s, y[e]), 30.0f);
    t[e] = mk(s, 0.0f);
  }
#pragma unroll
  for (int e = 0; e < VW; ++e) t[e] = t_add_d_u(t_mul_d_z(t[e], y[e]), c_texp32[0]);
#pragma unroll
  for (int k = 1; k < 4; ++k) {
    const float c = c_texp32[k];
#pragma unroll
    for (int e = 0; e < VW; ++e) t[e] = t_add_d_u(t_mul_d_u(t[e], y[e]), c);
  }
  }
}
template <int VW> TF_DEV void taylor_expm1_v(const double (&y)[VW], TF<double> (&t)[VW]) {
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    double s = add(y[e], 10.0);
    s = add(mul(s, y[e]), 90.0);
    s = add(mul(s, y[e]), 720.0);
    t[e] = mk(s, 0.0);
  }
#pragma unroll
  for (int e = 0; e < VW; ++e) t[e] = t_add_d_u(t_mul_d_z(t[e], y[e]), c_texpm1_64[0]);
#pragma unroll
  for (int k = 1; k < 6; ++k) {
    const double c = c_texpm1_64[k];
#pragma unroll
    for (int e = 0; e < VW; ++e) t[e] = t_add_d_u(t_mul_d_u(t[e], y[e]), c);
  }
#pragma unroll
  for (int e = 0; e < VW; ++e)
    t[e] = t_mul_u(t_mul_d_u(t[e], y[e]), mk(P<double>::INVF_V, P<double>::INVF_E));
}
template <int VW> TF_DEV void taylor_expm1_v(const float (&y)[VW], TF<float> (&t)[VW]) {
  if constexpr (VW % 2 == 0) {
    constexpr int NP = VW / 2;
    f2 yp[NP], nyp[NP];
    TF<f2> tp[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      yp[p] = pk(y[2 * p], y[2 * p + 1]);
      nyp[p] = pk(-y[2 * p], -y[2 * p + 1]);
      f2 s = add(yp[p], splat(5.0f));
      s = add(mul(s, yp[p]), splat(20.0f));
      tp[p] = mk(s, splat(0.0f));
    }
#pragma unroll
    for (int p = 0; p < NP; ++p)
      tp[p] = t_add_d_u(t_mul_d_pz(tp[p], yp[p], nyp[p]), splat(c_texpm1_32[0]));
#pragma unroll
    for (int k = 1; k < 2; ++k) {
      const f2 c = splat(c_texpm1_32[k]);
#pragma unroll
      for (int p = 0; p < NP; ++p) tp[p] = t_add_d_u(t_mul_d_p(tp[p], yp[p], nyp[p]), c);
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      tp[p] = t_mul_u(t_mul_d_p(tp[p], yp[p], nyp[p]), mk(splat(P<float>::INVF_V), splat(P<float>::INVF_E)));
      t[2 * p] = mk(lo(tp[p].v), lo(tp[p].e));
      t[2 * p + 1] = mk(hi(tp[p].v), hi(tp[p].e));
    }
  } else {
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    float s = add(y[e], 5.0f);
    s = add(mul(s, y[e]), 20.0f);
    t[e] = mk(s, 0.0f);
  }
#pragma unroll
  for (int e = 0; e < VW; ++e) t[e] = t_add_d_u(t_mul_d_z(t[e], y[e]), c_texpm1_32[0]);
#pragma unroll
  for (int k = 1; k < 2; ++k) {
    const float c = c_texpm1_32[k];
#pragma unroll
    for (int e = 0; e < VW; ++e) t[e] = t_add_d_u(t_mul_d_u(t[e], y[e]), c);
  }
#pragma unroll
  for (int e = 0; e < VW; ++e)
    t[e] = t_mul_u(t_mul_d_u(t[e], y[e]), mk(P<float>::INVF_V, P<float>::INVF_E));
  }
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

// pexpm10_raw, in-band branch only (expcore.py:142-146), VW lanes
template <class T, int VW>
TF_DEV void pexpm10_inband_v(const STab<T>& tb, const T (&x)[VW], TF<T> (&w)[VW]) {
  T y[VW];
  int n[VW];
#pragma unroll
  for (int e = 0; e < VW; ++e) decomp_expm1_u(x[e], n[e], y[e]);
  TF<T> t[VW];
  taylor_expm1_v<VW>(y, t);
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    TF<T> c = tv<T>(tb.CM1[n[e] - P<T>::CM1_LO]);
    w[e] = t_add_u(t_mul_u(c, t[e]), t_add_u(c, t[e]));
  }
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
// conservative integer form of explog.py:201/429 (binary64 arithmetic there).
TF_DEV bool newton_quiet(double r1, double r0) {
  int e1 = bexp(r1), e0 = bexp(r0);
  return e1 + 22 <= max(e0, 1023);
}
TF_DEV bool newton_quiet(float r1, float r0) {
  // on the FP pipe (the binary32 kernels are ALU-bound): |r1| < 2^-21 max(|r0|, 1),
  // which implies the reference's |r1| <= 2^-20 (|r0| + 1) with a factor 2 to spare
  return fabsf(r1) < 0x1p-21f * fmaxf(fabsf(r0), 1.0f);
}

// binary32 value part RN(h + l) from a twofold core: flag the element when
// h + l lies within 2^TOL |z| of a rounding boundary, so the rare-element
// drain decides it with the binary64 library (or the exact path).  The
// reference's twofold results are accurate to ~2^-37 at worst (PAPER.md:745-755,
// the near-1 log lanes), but the value-part sums of the fast kernels are far
// better: built with TOL = -40, 2^30 config-4 samples per function show no
// fast/exact difference (tools/guard_probe.py), so TOL = -36 keeps a 16x
// margin while flagging only ~2^-11 of the elements.
// rho = (h + l) - z is at most half an ulp (|z| < 2^(e+1): half = 2^(e-24),
// 2^TOL |z| <= 2^(TOL+25) half), so "within 2^TOL |z| of the boundary" implies
// |rho| k > half for k = 1 + eps + 2 eps^2, eps = 2^(TOL+25) ((1 - eps) k > 1),
// where z + rho k crosses the midpoint and rounds away from z: one FFMA and
// one compare, flagging |rho| >~ (1 - eps) half (~2^(TOL+25) of the
// elements).  Below an exact power of two the midpoint is half / 2, which the
// same rounding detects.
// rounding-guard tolerances (2^TOL |z|) of the binary32 logarithms and
// exponentials
#ifndef TF_TOL32_LOG
#define TF_TOL32_LOG -36
#endif
#ifndef TF_TOL32_EXP
#define TF_TOL32_EXP -36
#endif
#ifndef TF_GUARD_TIGHT
#define TF_GUARD_TIGHT 1
#endif
template <int TOL = -32> TF_DEV float kguard() {
  // 2 eps^2 below 2^-23: one ulp of k still satisfies (1 - eps) k > 1
  constexpr int SQ = 23 + 2 * (TOL + 25) + 1;
  if (TF_GUARD_TIGHT)
    return __int_as_float(0x3f800000 + (1 << (23 + TOL + 25)) + (SQ > 0 ? 1 << SQ : 1));
  return __int_as_float(0x3f800000 + (1 << (23 + TOL + 26)));   // 1 + 2 eps
}
template <int TOL = -32> TF_DEV float rn_guard(float h, float l, bool& hard) {
  float z = add(h, l);
  float rho = add(sub(h, z), l);                    // (h + l) - z
  hard = fmaop(rho, kguard<TOL>(), z) != z;
  return z;
}
// binary32 log(1 + d) for an exact |d| <= 2^-7 (the logarithms' near-1
// lanes): d - d^2/2 with d^2 split exactly by an FMA, then the d^3 .. d^7
// terms (truncation d^8/8 <= 2^-59), rounded under the guard: the series'
// own rounding error is ~2^-41 |z| at |d| = 2^-7, and a correctly rounded
// value needs the midpoint test like every other binary32 value part
// (tools/guard_probe.py found y = 0x1.01ed9ap+0 misrounded by the earlier
// unguarded degree-5 series).
TF_DEV float log_near1_g(float d, bool& hard) {
  const float q = mul(d, d);
  const float qe = fmaop(d, d, -q);
  float p = fmaop(d, 0x1.24924ap-3f, -0x1.555556p-3f);      // 1/7, -1/6
  p = fmaop(d, p, 0x1.99999ap-3f);                          // 1/5
  p = fmaop(d, p, -0.25f);
  p = fmaop(d, p, 0x1.555556p-2f);                          // 1/3
  const float c = mul(mul(q, d), p);
  const float lo = fmaop(-0.5f, qe, c);
  const TF<float> s = fast_two_sum_u(d, mul(-0.5f, q));
  return rn_guard<TF_TOL32_LOG>(s.v, add(s.e, lo), hard);
}
template <int TOL = -32>
TF_DEV double rn_guard(double h, double l, bool& hard) {  // binary64 cores: ~2^-100, no guard
  hard = false;
  return add(h, l);
}

// binary32 value part from the binary64 library (rare-element drain only):
// CUDA's binary64 exp/expm1/log/log1p are within 1 ulp, so RN32 of the result
// is the correctly rounded binary32 value unless it lies within 2 binary64
// ulps of a binary32 rounding midpoint (hard: exact path).  Normal binary32
// results only (29 dropped bits).
TF_DEV float cr32_of(double v, bool& hard) {
  const long long b = (long long)(ubits(v) & ((1ull << 29) - 1));
  const long long dm = b - (1ll << 28);
  hard = dm <= 2 && dm >= -2;
  return __double2float_rn(v);
}
enum DFn { DF_EXP = 0, DF_EXPM1 = 1, DF_LOG = 2, DF_LOG1P = 3 };
template <int F> TF_DEV float cr32_lib(float x, bool& hard) {
  const double d = (double)x;
  const double v = F == DF_EXP ? exp(d) : F == DF_EXPM1 ? expm1(d) : F == DF_LOG ? log(d)
                                                                        : log1p(d);
  return cr32_of(v, hard);
}

// ================================================================ texp
// Classes of x0 by raw bits (the sign-magnitude order of IEEE bit patterns):
//   core   lo_bound <= x0 < hi_bound            pexp0_raw's table path
//   below  -inf <= x0 < lo_bound                pexp0_raw = (0, 0)  (expcore.py:125-126)
//   above  hi_bound <= x0 <= +inf               (inf, inf)          (expcore.py:127-128,
//          x0 == hi_bound too: its product overflows and texp's guard returns (inf, inf))
//   NaN                                         (NaN, NaN)          (expcore.py:123-124)
// The main kernels run the core on the band where the result is normal and
// below 2^1023 (cheap high-word tests); the rare-element drain resolves the
// saturated classes with selects (texp_special) and evaluates the rest of the
// core -- subnormal results, x0 up to hi_bound -- with WIDE = true (fast_alt),
// so the exact path sees no finite x0 with a tiny tail at all.
constexpr uint64_t U64_HI = 0x40862e42fefa39f0ull;     // hi_bound
constexpr uint64_t U64_LO_NEG = 0xc0874385446d71c4ull; // lo_bound (negative)
constexpr uint64_t U64_UNF_NEG = 0xc0874910d52d3052ull; // EXP_UNF: exp(x) rounds to 0 below
constexpr uint64_t U64_PINF = 0x7ff0000000000000ull, U64_NINF = 0xfff0000000000000ull;
constexpr uint64_t U64_SIGN = 0x8000000000000000ull;

// PM = true: pexp0 = renorm_fast(pexp0_raw(x0)) (explog.py:101-103), no libm value
template <int VW, bool PM = false, bool WIDE = false>
TF_DEV void fast_texp(const STab<double>& tb, const double (&x0)[VW], const double (&x1)[VW],
                      double (&z0)[VW], double (&z1)[VW], bool (&ok)[VW]) {
  double y[VW];
  int m[VW], n[VW];
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    if constexpr (WIDE) {
      const uint64_t b = ubits(x0[e]);
      ok[e] = (b < U64_HI || (b >= U64_SIGN && b <= U64_LO_NEG)) && ahi(x1[e]) < H64_X1_TINY;
    } else {
      ok[e] = ahi(x0[e]) <= (sgn(x0[e]) ? H64_TEXP_NEG : H64_TEXP_POS) &&
              ahi(x1[e]) < H64_X1_TINY;
    }
    decomp_exp_u(ok[e] ? x0[e] : 0.0, m[e], n[e], y[e]);
  }
  TF<double> t[VW];
  taylor_exp_v<VW>(y, t);
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    TF<double> ct = t_mul_u(tv<double>(tb.C[n[e] - P<double>::C_LO]), t[e]);
    TF<double> v = t_mul_u(tv<double>(tb.E[m[e] - P<double>::E_LO]), ct);
    if constexpr (PM) {
      TF<double> r = fast_two_sum_u(v.v, v.e);
      z0[e] = r.v;
      z1[e] = r.e;
      continue;
    }
    double zz = add(v.v, v.e);                                  // CR exp(x0)
    if (m[e] <= TF64_ESC_LO + TF64_ESC_COUNT - 1) {
      // e^x < 2^-987: the unscaled product's residuals underflow, so round the
      // value part from the 2^128-scaled coarse entry (result normal: exact
      // unscale; WIDE: onto the subnormal grid, the exact path's rounding)
      TF<double> vs = t_mul_u(tv<double>(tb.ESC[m[e] - TF64_ESC_LO]), ct);
      zz = WIDE ? round_unscale128(vs.v, vs.e) : mul(add(vs.v, vs.e), 0x1p-128);
    }
    z0[e] = zz;
    z1[e] = add(mul(zz, t1_tiny(x1[e])), add(v.e, sub(v.v, zz)));  // explog.py:125
  }
}

// texp's saturated classes (drain): (NaN, NaN) for NaN x0 and (inf, inf) for
// x0 >= hi_bound whatever x1 (explog.py:119-122: the guard returns before t1;
// NaN propagates through z1), and for x0 < lo_bound with a tiny tail
// pexp0_raw = (0, 0), z0 = exp(x0) in {2^-1074, 0}, z1 by the texp epilogue.
TF_DEV bool texp_special(double x0, double x1, double& z0, double& z1) {
  const uint64_t b = ubits(x0);
  if (b > U64_PINF && b != U64_SIGN && !(b >= U64_SIGN && b <= U64_NINF)) {
    z0 = z1 = Lim<double>::qnan();
    return true;
  }
  if (b >= U64_HI && b <= U64_PINF) {
    z0 = z1 = Lim<double>::inf();
    return true;
  }
  if (b > U64_LO_NEG && b <= U64_NINF && ahi(x1) < H64_X1_TINY) {
    const double zz = b < U64_UNF_NEG ? 0x1p-1074 : 0.0;
    z0 = zz;
    z1 = add(mul(zz, t1_tiny(x1)), add(0.0, sub(0.0, zz)));
    return true;
  }
  return false;
}

// DBLV: value part from the binary64 library (cr32_lib), rare-element drain
template <int VW, bool PM = false, bool DBLV = false>
TF_DEV void fast_texp(const STab<float>& tb, const float (&x0)[VW], const float (&x1)[VW],
                      float (&z0)[VW], float (&z1)[VW], bool (&ok)[VW]) {
  float y[VW];
  int m[VW], n[VW];
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    // band tests on the FP pipe (the binary32 kernels are ALU-bound)
    ok[e] = x0[e] >= -__uint_as_float(B32_TEXP_NEG) && x0[e] <= __uint_as_float(B32_TEXP_POS) &&
            fabsf(x1[e]) < __uint_as_float(B32_X1_TINY);
    decomp_exp_u(ok[e] ? x0[e] : 0.0f, m[e], n[e], y[e]);
  }
  TF<float> t[VW];
  taylor_exp_v<VW>(y, t);
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    TF<float> ct = t_mul_u(tv<float>(tb.C[n[e] - P<float>::C_LO]), t[e]);
    TF<float> ev = tv<float>(tb.E[m[e] - P<float>::E_LO]);
    TF<float> v = t_mul_u(ev, ct);
    if constexpr (PM) {
      TF<float> r = fast_two_sum_u(v.v, v.e);
      z0[e] = r.v;
      z1[e] = r.e;
      continue;
    }
    // value part: near the subnormal range use the 2^64-scaled coarse table so
    // the twofold keeps full precision (result is normal: exact unscaling)
    bool scaled = m[e] <= -35;  // e^(2m) < 2^-100: residuals would underflow
    TF<float> es = tv<float>(tb.ESC[scaled ? m[e] - TF32_ESC_LO : 0]);
    TF<float> vs = t_mul_u(scaled ? es : ev, ct);
    bool hard;
    if constexpr (DBLV) z0[e] = cr32_lib<DF_EXP>(x0[e], hard);
    else z0[e] = mul(rn_guard<TF_TOL32_EXP>(vs.v, vs.e, hard), scaled ? 0x1p-64f : 1.0f);
    ok[e] = ok[e] && !hard;
    z1[e] = add(mul(z0[e], t1_tiny(x1[e])), add(v.e, sub(v.v, z0[e])));
  }
}

// ============================================================== texpm1
// binary64: the in-band core is the bulk (cfg 2: 99.5%)
// PM = true: pexpm10 = renorm_fast(pexpm10_raw(x0)) (explog.py:135-137)
template <int VW, bool PM = false>
TF_DEV void fast_texpm1(const STab<double>& tb, const double (&x0)[VW], const double (&x1)[VW],
                        double (&z0)[VW], double (&z1)[VW], bool (&ok)[VW]) {
  double xs[VW];
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    ok[e] = ahi(x0[e]) < H64_LN2 && ahi(x1[e]) < H64_X1_TINY;
    xs[e] = ok[e] ? x0[e] : 0.0;
  }
  TF<double> w[VW];
  pexpm10_inband_v<double, VW>(tb, xs, w);
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    if constexpr (PM) {
      TF<double> r = fast_two_sum_u(w[e].v, w[e].e);
      z0[e] = r.v;
      z1[e] = r.e;
      continue;
    }
    z0[e] = ahi(xs[e]) < H64_TINY54 ? xs[e] : add(w[e].v, w[e].e);   // CR expm1(x0)
    double tail = add(w[e].e, sub(w[e].v, z0[e]));
    z1[e] = add(mul(add(z0[e], 1.0), t1_tiny(x1[e])), tail);          // explog.py:159-160
  }
}

// binary64 fallback branch (|x0| >= ln2, expcore.py:147): pexp0_raw(x0) - 1.
// Not the main path at the BASELINE configs (cfg 2: 0.5% of elements); the
// rare-element drain runs it before resorting to the exact path.
template <int VW, bool PM = false>
TF_DEV void fast_texpm1_fb(const STab<double>& tb, const double (&x0)[VW],
                           const double (&x1)[VW], double (&z0)[VW], double (&z1)[VW],
                           bool (&ok)[VW]) {
  double y[VW];
  int m[VW], n[VW];
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    ok[e] = abits(x0[e]) > B64_LN2 &&                          // out of band (expcore.py:142)
            ahi(x0[e]) <= (sgn(x0[e]) ? H64_TEXP_NEG : H64_TEXP_POS) &&
            ahi(x1[e]) < H64_X1_TINY;
    decomp_exp_u(ok[e] ? x0[e] : 1.0, m[e], n[e], y[e]);
  }
  TF<double> t[VW];
  taylor_exp_v<VW>(y, t);
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    TF<double> v = t_mul_u(tv<double>(tb.E[m[e] - P<double>::E_LO]),
                           t_mul_u(tv<double>(tb.C[n[e] - P<double>::C_LO]), t[e]));
    TF<double> w = t_add_d_u(v, -1.0);                          // expcore.py:147
    if constexpr (PM) {
      TF<double> r = fast_two_sum_u(w.v, w.e);
      z0[e] = r.v;
      z1[e] = r.e;
      continue;
    }
    z0[e] = add(w.v, w.e);                                      // CR expm1(x0)
    double tail = add(w.e, sub(w.v, z0[e]));
    z1[e] = add(mul(add(z0[e], 1.0), t1_tiny(x1[e])), tail);
  }
}

// binary32: the pexp0 - 1 fallback is the bulk (cfg 4: 99.2%)
template <int VW, bool PM = false, bool DBLV = false>
TF_DEV void fast_texpm1(const STab<float>& tb, const float (&x0)[VW], const float (&x1)[VW],
                        float (&z0)[VW], float (&z1)[VW], bool (&ok)[VW]) {
  float y[VW];
  int m[VW], n[VW];
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    ok[e] = fabsf(x0[e]) > __uint_as_float(B32_LN2) && x0[e] >= -__uint_as_float(B32_LO) &&
            x0[e] <= __uint_as_float(B32_TEXP_POS) && fabsf(x1[e]) < __uint_as_float(B32_X1_TINY);
    decomp_exp_u(ok[e] ? x0[e] : 1.0f, m[e], n[e], y[e]);
  }
  TF<float> t[VW];
  taylor_exp_v<VW>(y, t);
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    TF<float> v = t_mul_u(tv<float>(tb.E[m[e] - P<float>::E_LO]),
                          t_mul_u(tv<float>(tb.C[n[e] - P<float>::C_LO]), t[e]));
    TF<float> w = t_add_d_u(v, -1.0f);                          // expcore.py:147
    if constexpr (PM) {
      TF<float> r = fast_two_sum_u(w.v, w.e);
      z0[e] = r.v;
      z1[e] = r.e;
      continue;
    }
    bool hard;
    if constexpr (DBLV) z0[e] = cr32_lib<DF_EXPM1>(x0[e], hard);
    else z0[e] = rn_guard<TF_TOL32_EXP>(w.v, w.e, hard);
    ok[e] = ok[e] && !hard;
    float tail = add(w.e, sub(w.v, z0[e]));
    z1[e] = add(mul(add(z0[e], 1.0f), t1_tiny(x1[e])), tail);
  }
}

// binary32 in-band branch (|x0| <= LN2, expcore.py:142-146), drain only: the
// main binary32 kernel takes the fallback branch (cfg 4: 99.2% of elements)
template <bool PM = false>
TF_DEV void fast_texpm1_inb32(const STab<float>& tb, float x0, float x1, float& z0, float& z1,
                              bool& ok) {
  ok = abits(x0) <= B32_LN2 && ahi(x1) < B32_X1_TINY;
  float xs[1] = {ok ? x0 : 0.0f};
  TF<float> w[1];
  pexpm10_inband_v<float, 1>(tb, xs, w);
  if constexpr (PM) {
    TF<float> r = fast_two_sum_u(w[0].v, w[0].e);
    z0 = r.v;
    z1 = r.e;
    return;
  }
  bool hard;
  z0 = rn_guard<TF_TOL32_EXP>(w[0].v, w[0].e, hard);        // binary64 library only when
  if (hard) z0 = cr32_lib<DF_EXPM1>(xs[0], hard);  // the core cannot decide
  if (ahi(xs[0]) < B32_TINY25) {                    // expm1(x) rounds to x (keeps -0)
    z0 = xs[0];
    hard = false;
  }
  ok = ok && !hard;
  float tail = add(w[0].e, sub(w[0].v, z0));
  z1 = add(mul(add(z0, 1.0f), t1_tiny(x1)), tail);
}

// ================================================================= tlog
// explog.py:244-249 -> _log_core (188-208) -> _newton_log_z (170-186),
// with the value part replaced by a correctly rounded log(y0):
//   log(y0) = log(v) - log1p(d),  d = y1 / y0  (renorm is error-free: v - y0 == y1),
// and near 1 by the exact-d series (log_near1).
template <class T> struct LogC;
template <> struct LogC<double> {
  static constexpr uint32_t NORM_SPAN = 2044u;   // positive normal and < 2^1022: 2^-n normal
  // |d| < 2^-50 (tlog value part): log(y0) = core - d drops d^2/2, which must
  // stay far below an ulp of |log y0| >= 2^-20 (coupled inputs have |d| <= 2^-53)
  static constexpr uint32_t DMAX = (1023u - 50u) << 20;
  static constexpr int SMALL = 50, EBIAS = 1022;
  static constexpr int SUBSH = 54;
  static constexpr double SUBSCALE = 0x1p54;
  static constexpr uint64_t HALF = B64_HALF, TWO = B64_TWO;
  static constexpr uint32_t NEAR1H = H64_NEAR1;
  TF_DEV static uint32_t eb(double x) { return (uint32_t)hi32(x) >> 20; }
  TF_DEV static int n_of(double v) { return (int)(ubits(v) >> 52) - 1022; }
  TF_DEV static double mant(double v) {
    return __longlong_as_double((ubits(v) & 0x800fffffffffffffull) | (1022ull << 52));
  }
  TF_DEV static double p2(int k) { return p2d_bf(k); }
  // |r| <= LN2 (the table value): pexpm10_raw's in-band test (expcore.py:142),
  // exact; a seed of exactly -LN2 (argument a power of two) stays in band
  TF_DEV static bool in_ln2(double r) { return abits(r) <= B64_LN2; }
  // 2^k for k in [-1022, 1023] (normal), two integer ops
  TF_DEV static double p2n(int k) { return __hiloint2double((k + 1023) << 20, 0); }
  TF_DEV static double rcp(double x) { return rcp_nr(x); }
};
template <> struct LogC<float> {
  static constexpr uint32_t NORM_SPAN = 254u;           // (2^-n may be subnormal: p2n = p2)
  static constexpr uint32_t DMAX = (127u - 21u) << 23;   // |d| < 2^-21
  static constexpr int SMALL = 21, EBIAS = 126;
  static constexpr int SUBSH = 25;
  static constexpr float SUBSCALE = 0x1p25f;
  static constexpr uint32_t HALF = B32_HALF, TWO = B32_TWO;
  static constexpr uint32_t NEAR1H = NEAR1_32 + 1u;
  TF_DEV static uint32_t eb(float x) { return ubits(x) >> 23; }
  TF_DEV static int n_of(float v) { return (int)(ubits(v) >> 23) - 126; }
  TF_DEV static float mant(float v) {
    return __int_as_float((ubits(v) & 0x807fffffu) | (126u << 23));
  }
  TF_DEV static float p2(int k) { return p2f_bf(k); }
  TF_DEV static bool in_ln2(float r) { return abits(r) <= B32_LN2; }
  TF_DEV static float p2n(int k) { return p2f_bf(k); }
  TF_DEV static float rcp(float x) { return rcp_approx(x); }
};

// tlog / tlog0 / tlogp inputs whose result is a constant (_correct, explog.py:
// 216-223, with the library value log(y0)): y0 NaN or negative (not -0) ->
// log(y0) = NaN -> (NaN, NaN) whatever y1; y0 = +-0 and y1 = +-0 -> the core is
// (-inf, NaN) and log(0) = -inf -> (-inf, -inf); y0 = +inf, y1 finite -> the
// core's value part is +inf -> (inf, inf).  Resolved in the rare-element drain
// (special_const) instead of the exact path.
enum LogConst { LC_NONE = 0, LC_NAN = 1, LC_NINF = 2, LC_PINF = 3 };
TF_DEV int log_const_class(double y0, double y1) {
  const uint64_t b0 = ubits(y0), b1 = ubits(y1);
  if (b0 > U64_PINF && b0 != U64_SIGN) return LC_NAN;
  if ((b0 << 1) == 0 && (b1 << 1) == 0) return LC_NINF;
  if (b0 == U64_PINF && is_finite(y1)) return LC_PINF;
  return LC_NONE;
}
TF_DEV int log_const_class(float y0, float y1) {
  const uint32_t b0 = ubits(y0), b1 = ubits(y1);
  if (b0 > 0x7f800000u && b0 != 0x80000000u) return LC_NAN;
  if ((b0 << 1) == 0 && (b1 << 1) == 0) return LC_NINF;
  if (b0 == 0x7f800000u && is_finite(y1)) return LC_PINF;
  return LC_NONE;
}
template <class T> TF_DEV bool log_const_apply(int c, T& z0, T& z1) {
  if (c == LC_NAN) { z0 = Lim<T>::qnan(); z1 = Lim<T>::qnan(); }
  if (c == LC_NINF) { z0 = -Lim<T>::inf(); z1 = -Lim<T>::inf(); }
  if (c == LC_PINF) { z0 = Lim<T>::inf(); z1 = Lim<T>::inf(); }
  return c != LC_NONE;
}

// Variants (explog.py:225-258): RENORM = false evaluates the core on (y0, y1)
// as given (tlogp, plog; tlog0 / plog0 have y1 = 0, where renorm is the
// identity); PM = true returns renorm_fast(core) instead of the _correct'ed
// value part (plog0, plog).
// FULLR (binary64 drain only): the top binade y0 >= 2^1022 too, scaling by a
// possibly subnormal 2^-n (p2 instead of the two-op p2n)
template <class T, int VW, bool RENORM = true, bool PM = false, bool DBLV = false,
          bool FULLR = false>
TF_DEV void fast_tlog(const STab<T>& tb, const T (&y0i)[VW], const T (&y1i)[VW], T (&z0)[VW],
                      T (&z1)[VW], bool (&ok)[VW]) {
  using C = LogC<T>;
  constexpr uint32_t SPAN = FULLR ? C::NORM_SPAN + 2u : C::NORM_SPAN;
  auto p2s = [](int k) { return FULLR ? C::p2(k) : C::p2n(k); };
  T y0[VW], y1[VW], zc0[VW], zc1[VW], r0[VW], mr0[VW];
  int n[VW];
  TF<T> v[VW];
  int nsc[VW];  // exponent of the tail scaling 2^-n (0 for pre-scaled subnormals)
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    // FULLR (drain): a positive subnormal y0 with y1 = 0 is scaled by 2^SUBSH
    // first (exact), so frexp's exponent is n_of(y0 2^SUBSH) - SUBSH
    bool subn = false;
    if constexpr (FULLR)
      subn = C::eb(y0i[e]) == 0u && !sgn(y0i[e]) && !zbits(y0i[e]) && zbits(y1i[e]);
    const T y0s = subn ? mul(y0i[e], C::SUBSCALE) : y0i[e];
    // positive normal y0 (below 2^1022 / 2^126) and finite y1; how small y1 is
    // against y0 is checked on d = y1/y0 below, where it matters
    ok[e] = C::eb(y0s) - 1u < SPAN && is_finite(y1i[e]);
    if constexpr (sizeof(T) == 8) {
      // binary64: rejected lanes compute on whatever they hold (no selects
      // here): the seed index is clamped and the CM1 index masked below
      y0[e] = y0s;
      y1[e] = y1i[e];
    } else {
      y0[e] = ok[e] ? y0s : T(1);
      y1[e] = ok[e] ? y1i[e] : T(0);
    }
    v[e] = RENORM ? renorm_u(mk(y0[e], y1[e])) : mk(y0[e], y1[e]);
    ok[e] = ok[e] && C::eb(v[e].v) - 1u < SPAN;
    if (sizeof(T) == 4 && !ok[e]) v[e] = mk(T(1), T(0));
    auto vb = ubits(v[e].v);
    bool band = vb >= C::HALF && vb <= C::TWO;
    n[e] = band ? 0 : C::n_of(v[e].v) - (subn ? C::SUBSH : 0);
    nsc[e] = subn ? 0 : -n[e];
    zc0[e] = band ? v[e].v : C::mant(v[e].v);
    zc1[e] = band ? v[e].e : (zbits(v[e].e) ? T(0) : mul(v[e].e, p2s(nsc[e])));
    r0[e] = seed_log1p_t(add(sub(zc0[e], T(1)), zc1[e]),      // explog.py:196-199
                         [&](int i) { return seed_entry(tb, i); });
    ok[e] = ok[e] && C::in_ln2(r0[e]);
    // keeps the CM1 index in range for rejected lanes (tlogp / plog take y1
    // unrenormalised, so the seed of a non-coupled input can be anything)
    mr0[e] = ok[e] ? -r0[e] : T(0);
  }
  TF<T> s[VW];
  pexpm10_inband_v<T, VW>(tb, mr0, s);
  T dl[VW], cv[VW], ce[VW];
  unsigned near = 0;
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    TF<T> w = fast_two_sum_u(sub(zc0[e], T(1)), zc1[e]);
    TF<T> u = t_add_u(t_mul_u(mk(zc0[e], zc1[e]), s[e]), w);
    T r1 = add(u.v, u.e);
    ok[e] = ok[e] && newton_quiet(r1, r0[e]);
    TF<T> nl = t_mul_d_u(mk(P<T>::LN2_V, P<T>::LN2_E), (T)n[e]);
    TF<T> core = t_add_u(mk(r0[e], r1), nl);
    if constexpr (PM) {                                 // explog.py:205-208, 258
      TF<T> r = n[e] == 0 ? fast_two_sum_u(r0[e], r1) : fast_two_sum_u(core.v, core.e);
      z0[e] = r.v;
      z1[e] = r.e;
      continue;
    }
    // Away from 1 (|y0 - 1| >= 2^-20, 2^-7 in binary32) |log y0| is large next
    // to d = y1/y0 (|d| <= 2^-50 |log y0|, 2^-17 in binary32), so
    // log(y0) = core - d to well below an ulp with d known to ~2^-22:
    // y1 * 2^-n over zc0 (= v0 * 2^-n, within an ulp of y0 * 2^-n).
    T d0 = mul(mul(y1[e], p2s(nsc[e])), C::rcp(zc0[e]));
    ok[e] = ok[e] && ahi(d0) < C::DMAX;
    // binary64: d carries the reciprocal's 2^-40 relative error, which must
    // stay ~2^-30 below an ulp of log(y0): |d| <= 2^-42 |core| away from the
    // near-1 series (only |log y0| < ~2^-11 is sent away)
    const bool dsmall = sizeof(T) == 4 || ahi(d0) + (42u << 20) <= ahi(core.v);
    bool hard;
    if constexpr (sizeof(T) == 8) {
      // |y0 - 1| < 2^-20 on the bit pattern (no DADD); y0 - 1 (exact there) is
      // formed in the near-1 pass only
      dl[e] = y0[e];
      z0[e] = rn_guard<TF_TOL32_LOG>(core.v, sub(core.e, d0), hard);
      if (ubits(y0[e]) - 0x3FEFFFFE00000001ull < 0x3FF0000010000000ull - 0x3FEFFFFE00000001ull)
        near |= 1u << e;
      else ok[e] = ok[e] && !hard && dsmall;
    } else if constexpr (DBLV) {
      dl[e] = sub(y0[e], T(1));
      z0[e] = cr32_lib<DF_LOG>(y0[e], hard);
      ok[e] = ok[e] && !hard;
    } else {
      dl[e] = sub(y0[e], T(1));                       // exact near 1
      z0[e] = rn_guard<TF_TOL32_LOG>(core.v, sub(core.e, d0), hard);
      if (ahi(dl[e]) < C::NEAR1H) near |= 1u << e;
      else ok[e] = ok[e] && !hard && dsmall;
    }
    cv[e] = core.v;
    ce[e] = core.e;
  }
  // near-1 value parts (cfg 3: 5% of elements): one log_near1 per pass for the
  // lowest flagged lane, so a warp pays for one series, not one per lane
  while (near) {
    T d = dl[0];
#pragma unroll
    for (int e = VW - 1; e > 0; --e)
      if (near >> e & 1u) d = dl[e];
    if (near & 1u) d = dl[0];
    const unsigned low = near & (0u - near);
    bool hn = false;
    T r;
    if constexpr (sizeof(T) == 4) r = log_near1_g(d, hn);
    else r = log_near1(sub(d, T(1)));                 // dl holds y0 (binary64)
#pragma unroll
    for (int e = 0; e < VW; ++e)
      if (low == 1u << e) { z0[e] = r; ok[e] = ok[e] && !hn; }
    near &= near - 1u;
  }
  if constexpr (!PM) {
#pragma unroll
    for (int e = 0; e < VW; ++e) {
      z1[e] = add(ce[e], sub(cv[e], z0[e]));  // _correct (222-223)
    }
  }
}

// ------------------------------------------- binary32 tlog, lane pairs
// The binary32 kernels are issue-bound: every scalar FP32 op costs an issue
// slot.  This variant of fast_tlog<float> (RENORM / tlogp flavours of the main
// kernels) runs the whole twofold pipeline -- renorm, seed polynomial, the
// expm1 core, the Newton step, n ln2, the value part -- on f32x2 pairs
// (FADD2 / FFMA2: one issue slot for two lanes).  The operation sequence per
// lane is exactly fast_tlog<float>'s; classification and table indexing stay
// per lane on the integer pipe.
TF_DEV TF<f2> pk2(TF<float> a, TF<float> b) { return mk(pk(a.v, b.v), pk(a.e, b.e)); }

// expm1 Taylor core on a lane pair (taylor_expm1_v's packed body)
TF_DEV TF<f2> taylor_expm1_p(f2 yp) {
  const f2 nyp = -yp;
  f2 s = add(yp, splat(5.0f));
  s = add(mul(s, yp), splat(20.0f));
  TF<f2> tp = mk(s, splat(0.0f));
  tp = t_add_d_u(t_mul_d_pz(tp, yp, nyp), splat(c_texpm1_32[0]));
  tp = t_add_d_u(t_mul_d_p(tp, yp, nyp), splat(c_texpm1_32[1]));
  return t_mul_u(t_mul_d_p(tp, yp, nyp), mk(splat(P<float>::INVF_V), splat(P<float>::INVF_E)));
}

// table-driven seed log1p (seed_log1p_t<float>) on a lane pair
// One 32-bit shared-memory load per half of a lane pair (TF_SPLIT_LDS): the two
// lanes read different table entries, and loading each entry's (v, e) as one
// 64-bit word leaves v0, v1 in two different register pairs, which ptxas then
// copies into place (IMAD.MOV, on the busy fmaheavy pipe) for the packed
// consumers.  The loads are volatile because ptxas merges adjacent plain
// ld.shared.f32 back into LDS.64.  +6% tlog f32, +4% tlog1p f32.
#ifndef TF_SPLIT_LDS
#define TF_SPLIT_LDS 1
#endif
// 32-bit shared-window address of a shared-memory object; the table bases are
// loop invariant, so each lookup costs one index scaling (the (v, e) halves
// share it through the load's immediate offset) instead of a generic-to-shared
// conversion per load (which ptxas emits as IMADs on the busy FMA pipe)
TF_DEV uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
TF_DEV float lds32a(uint32_t a) {
  float r;
  asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(r) : "r"(a));
  return r;
}
TF_DEV float lds32(const float* p) { return lds32a(saddr(p)); }
// TF_BOUNDS_CHECK (diagnostic builds, tools/sanitize_target.py): trap on a table
// index outside the staged table; the pool has no compute-sanitizer
#ifndef TF_BOUNDS_CHECK
#define TF_BOUNDS_CHECK 0
#endif
TF_DEV void bounds(int i, int n) {
  if (TF_BOUNDS_CHECK && (unsigned)i >= (unsigned)n) __trap();
}
template <int N>
TF_DEV TF<f2> ldpair(const float2 (&t)[N], int i0, int i1) {
  bounds(i0, N);
  bounds(i1, N);
  if (TF_SPLIT_LDS) {
    const uint32_t b = saddr(&t[0]);
    const uint32_t a0 = b + (uint32_t)i0 * 8u, a1 = b + (uint32_t)i1 * 8u;
    return mk(pk(lds32a(a0), lds32a(a1)), pk(lds32a(a0 + 4u), lds32a(a1 + 4u)));
  }
  const float2 a = t[i0], b = t[i1];
  return mk(pk(a.x, b.x), pk(a.y, b.y));
}

TF_DEV f2 seed_log1p_p(const STab<float>& tb, f2 a) {
  constexpr int B = TF32_SEED_BITS, NB = 1 << B;
  const f2 f = add(splat(1.0f), a);
  int idx[2];
  const float ax[2] = {lo(a), hi(a)}, fx[2] = {lo(f), hi(f)};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    // (exponent, leading B mantissa bits) of f in [1/2, 2] is one field:
    // ((e - 126) << B) | m = (fb >> (23 - B)) - (126 << B), in [0, 2 NB]; the
    // unsigned clamp keeps rejected lanes' garbage in range
    const uint32_t i = (ubits(fx[h]) >> (23 - B)) - (126u << B);
    idx[h] = fabsf(ax[h]) < 0x1p-8f ? 2 * NB + 1 : (int)min(i, 2u * NB);   // FP pipe test
  }
  const TF<f2> t = ldpair(tb.SEED, idx[0], idx[1]);       // (invc, logc)
  bounds(idx[0], TF32_SEED_COUNT + 1);
  bounds(idx[1], TF32_SEED_COUNT + 1);
  const uint32_t bm = saddr(&tb.SEEDM1[0]);
  const f2 m1 = TF_SPLIT_LDS ? pk(lds32a(bm + (uint32_t)idx[0] * 4u), lds32a(bm + (uint32_t)idx[1] * 4u))
                             : pk(tb.SEEDM1[idx[0]], tb.SEEDM1[idx[1]]);
  const f2 r = fmaop(a, t.v, m1);                          // (1 + a) invc - 1, one rounding
  const f2 q = mul(r, r);                                  // seed_poly<float>
  f2 pp = fmaop(r, splat(-0.25f), splat(0x1.555556p-2f));
  pp = fmaop(r, pp, splat(-0.5f));
  pp = fmaop(q, pp, r);
  return add(t.e, pp);
}

// pexpm10_raw(mx), in-band branch (expcore.py:142-146), on a lane pair:
// decompose_expm1 by the magic constant, the packed Taylor core, and the
// coupled CM1 entry recombination
TF_DEV TF<f2> pexpm10_inband_p(const STab<float>& tb, f2 mx) {
  const f2 tq = fmaop(mx, splat(128.0f), splat(12582912.0f));
  const int n0 = (int)ubits(lo(tq)) - 0x4b400000, n1 = (int)ubits(hi(tq)) - 0x4b400000;
  const f2 ym = fmaop(sub(tq, splat(12582912.0f)), splat(-0.0078125f), mx);
  const TF<f2> tt = taylor_expm1_p(ym);
  const TF<f2> cm = ldpair(tb.CM1, n0 - P<float>::CM1_LO, n1 - P<float>::CM1_LO);
  return t_add_u(t_mul_u(cm, tt), t_add_u(cm, tt));
}

// rn_guard<TF_TOL32_LOG> on a lane pair: packed sums and crossing test
template <int TOL = TF_TOL32_LOG>
TF_DEV f2 rn_guard_p(f2 h, f2 l, bool (&hard)[2]) {
  const f2 zs = add(h, l);
  const f2 rho = add(sub(h, zs), l);
  const f2 cr = fmaop(rho, splat(kguard<TOL>()), zs);
  hard[0] = lo(cr) != lo(zs);
  hard[1] = hi(cr) != hi(zs);
  return zs;
}

// per-lane select of two lane pairs: (c0 ? a.lo : b.lo, c1 ? a.hi : b.hi)
// (a select on the bit patterns compiles to the same FSEL / SEL mix: ptxas
// picks the pipe)
TF_DEV f2 sel2(bool c0, bool c1, f2 a, f2 b) {
  return pk(c0 ? lo(a) : lo(b), c1 ? hi(a) : hi(b));
}

template <int VW, bool RENORM>
TF_DEV void fast_tlog_p(const STab<float>& tb, const float (&y0i)[VW], const float (&y1i)[VW],
                        float (&z0)[VW], float (&z1)[VW], bool (&ok)[VW]) {
  static_assert(VW % 2 == 0, "lane pairs");
  constexpr int NP = VW / 2;
  using C = LogC<float>;
  float y0[VW], y1[VW], r0[VW], dl[VW];
  int n[VW];
  unsigned near = 0;
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    // classification on the FP pipe (FSETP) where an integer test would load
    // the ALU pipe: positive normal y0, finite y1.  With RENORM the finiteness
    // tests are implied by the positive-normal test of v = renorm(y) below (an
    // infinite or NaN operand, or an overflowing sum, makes v0 NaN)
    ok[e] = RENORM ? y0i[e] >= 0x1p-126f
                   : y0i[e] >= 0x1p-126f && y0i[e] <= 0x1.fffffep127f &&
                         fabsf(y1i[e]) <= 0x1.fffffep127f;
    // rejected lanes compute on whatever they hold: every table index below is
    // clamped or derived from a masked value, and their results are discarded
    y0[e] = y0i[e];
    y1[e] = y1i[e];
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const int a = 2 * p, b = 2 * p + 1;
    TF<f2> v = mk(pk(y0[a], y0[b]), pk(y1[a], y1[b]));
    if (RENORM) v = renorm_u(v);
    // per-lane classification and frexp on the integer pipe
    float vv[2] = {lo(v.v), hi(v.v)}, ve[2] = {lo(v.e), hi(v.e)};
    float c0[2], p2[2], z1a[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = 2 * p + h;
      ok[e] = ok[e] && vv[h] >= 0x1p-126f && vv[h] <= 0x1.fffffep127f;
      bool band = vv[h] >= 0.5f && vv[h] <= 2.0f;
      n[e] = band ? 0 : C::n_of(vv[h]);
      c0[h] = band ? vv[h] : C::mant(vv[h]);
      p2[h] = band ? 1.0f : C::p2n(-n[e]);            // band: v.e * 1 == v.e exactly
      z1a[h] = band ? -0.0f : 0.0f;
    }
    const f2 zc0 = pk(c0[0], c0[1]);
    // v.e 2^-n, and 0.0 for a zero v.e out of band (explog.py:190, "if y1 != 0.0
    // else 0.0"): one FFMA2 whose +0 addend turns -0 into +0 and leaves every
    // other product unchanged (the band keeps v.e as is: addend -0)
    const f2 zc1 = fmaop(pk(ve[0], ve[1]), pk(p2[0], p2[1]), pk(z1a[0], z1a[1]));
    const f2 rs = seed_log1p_p(tb, add(sub(zc0, splat(1.0f)), zc1));   // explog.py:196-199
    float rr[2] = {lo(rs), hi(rs)};
    float mr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = 2 * p + h;
      r0[e] = rr[h];
      ok[e] = ok[e] && fabsf(rr[h]) <= P<float>::LN2_V;
      mr[h] = ok[e] ? -rr[h] : 0.0f;                     // keeps the CM1 index in range
    }
    // s = pexpm10_raw(-r0), in-band branch (expcore.py:142-146)
    const TF<f2> s = pexpm10_inband_p(tb, pk(mr[0], mr[1]));
    // Newton step (_newton_log_z, explog.py:170-186)
    const TF<f2> w = fast_two_sum_u(sub(zc0, splat(1.0f)), zc1);
    const TF<f2> u = t_add_u(t_mul_u(mk(zc0, zc1), s), w);
    const f2 r1 = add(u.v, u.e);
    const f2 r0p = pk(r0[2 * p], r0[2 * p + 1]);
    // newton_quiet on the FP pipe: |r1| < 2^-21 max(|r0|, 1) (exact scaling)
    const f2 lim = mul(pk(fmaxf(fabsf(r0[2 * p]), 1.0f), fmaxf(fabsf(r0[2 * p + 1]), 1.0f)),
                       splat(0x1p-21f));
#pragma unroll
    for (int h = 0; h < 2; ++h)
      ok[2 * p + h] = ok[2 * p + h] && fabsf(h ? hi(r1) : lo(r1)) < (h ? hi(lim) : lo(lim));
    const TF<f2> nl = t_mul_d_u(mk(splat(P<float>::LN2_V), splat(P<float>::LN2_E)),
                                pk((float)n[2 * p], (float)n[2 * p + 1]));
    const TF<f2> core = t_add_u(mk(r0p, r1), nl);
    // value part: log(y0) = core - d, d = y1 2^-n / zc0
    const f2 rc = pk(C::rcp(c0[0]), C::rcp(c0[1]));
    const f2 d0 = mul(mul(pk(y1[2 * p], y1[2 * p + 1]), pk(p2[0], p2[1])), rc);
    bool hard[2];
    const f2 zs = rn_guard_p(core.v, sub(core.e, d0), hard);   // |z| >= 2^-8 away from 1
    float zx[2] = {lo(zs), hi(zs)}, dx[2] = {lo(d0), hi(d0)};
    const f2 dlp = sub(pk(y0[2 * p], y0[2 * p + 1]), splat(1.0f));   // exact near 1
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = 2 * p + h;
      ok[e] = ok[e] && fabsf(dx[h]) < 0x1p-21f;             // C::DMAX
      z0[e] = zx[h];
      dl[e] = h ? hi(dlp) : lo(dlp);
      if (fabsf(dl[e]) <= 0x1p-7f) near |= 1u << e;          // C::NEAR1H
      else ok[e] = ok[e] && !hard[h];
    }
    // z1 = core.e + (core.v - z0) (_correct, explog.py:222-223), after near-1 fix-ups
    z1[2 * p] = lo(core.v);
    z1[2 * p + 1] = hi(core.v);
    y1[2 * p] = lo(core.e);
    y1[2 * p + 1] = hi(core.e);
  }
  while (near) {
    float d = dl[0];
#pragma unroll
    for (int e = VW - 1; e > 0; --e)
      if (near >> e & 1u) d = dl[e];
    if (near & 1u) d = dl[0];
    const unsigned low = near & (0u - near);
    bool hn;
    const float r = log_near1_g(d, hn);
#pragma unroll
    for (int e = 0; e < VW; ++e)
      if (low == 1u << e) { z0[e] = r; ok[e] = ok[e] && !hn; }
    near &= near - 1u;
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const f2 cv = pk(z1[2 * p], z1[2 * p + 1]), ce = pk(y1[2 * p], y1[2 * p + 1]);
    const f2 r = add(ce, sub(cv, pk(z0[2 * p], z0[2 * p + 1])));
    z1[2 * p] = lo(r);
    z1[2 * p + 1] = hi(r);
  }
}

// =============================================================== tlog1p
// _plog1p_raw (explog.py:290-294) with both branches sharing ONE in-band
// pexpm10 evaluation (the Taylor core is ~3/4 of the work):
//   in-band  (-1/2 <= v0 <= 1): _log1p_core (276-282) -> _newton_log1p_in_band
//            (260-274), seed log1p(v0);
//   out-of-band: w = renorm(v + 1), tlogp(w) = _correct(_log_core(w), log(w0))
//            (239-242, 188-208), seed log1p((z0 - 1) + z1) after frexp.
// UNIFIED=false (binary64, cfg 2: 0.45% out-of-band) sends the out-of-band
// lanes to the exact path instead; UNIFIED=true (binary32, cfg 4: 50/50)
// evaluates them here with a lane-selected prologue/epilogue.
// Value parts: log1p(y0) = log1p(v) - log1p(d), d = y1/(1 + y0) (renorm is
// error-free); log(w0) = log(w) - log1p(w1/w0).
// Variants (explog.py:284-325): RENORM = false evaluates (y0, y1) as given
// (tlog1pp, plog1p; the dotted ones have y1 = 0); INNER = false is
// _plog1p0_raw's out-of-band branch, the raw _log_core of renorm(1 + y0)
// without tlogp's inner _correct (tlog1p0, plog1p0); PM = true returns
// renorm_fast of the raw result (plog1p0, plog1p).
template <class T, int VW, bool RENORM = true, bool PM = false, bool INNER = true, int UNI = -1,
          bool DBLV = false>
TF_DEV void fast_tlog1p(const STab<T>& tb, const T (&y0i)[VW], const T (&y1i)[VW], T (&z0)[VW],
                        T (&z1)[VW], bool (&ok)[VW]) {
  constexpr bool D = sizeof(T) == 8;
  constexpr bool UNIFIED = UNI < 0 ? !D : UNI > 0;
  // out-of-band value part: log1p(d) = d - d^2/2 to the lane's precision needs
  // |d| = |y1 / (1 + y0)| <= 2^-13 (binary32); binary64 also needs the
  // reciprocal's 2^-40 error in d far below an ulp: |d| <= 2^-51 (coupled
  // arguments have |d| <= 2^-53)
  constexpr int DSEP = D ? 52 : 14;
  using C = LogC<T>;
  T y0[VW], y1[VW], sd[VW], ms[VW], zc0[VW], zc1[VW];
  T wv[DBLV ? VW : 1];
  int n[VW];
  bool inb[VW];
  TF<T> v[VW];
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    // finite inputs; the size of y1 is checked where it matters, on d below
    if constexpr (D) ok[e] = is_finite(y0i[e]) && is_finite(y1i[e]);
    else ok[e] = fabsf(y0i[e]) <= 0x1.fffffep127f && fabsf(y1i[e]) <= 0x1.fffffep127f;
    // binary32 (ALU-bound): rejected lanes keep their values; the prologue's
    // `if (!ok) arg = 0` below keeps every table index in range
    y0[e] = (D && !ok[e]) ? T(0) : y0i[e];
    y1[e] = (D && !ok[e]) ? T(0) : y1i[e];
    v[e] = RENORM ? renorm_u(mk(y0[e], y1[e])) : mk(y0[e], y1[e]);
    // in band: -1/2 <= v0 <= 1 (explog.py:291).  The unified branch needs the
    // exact test (v0 = 1 or -1/2 must not go out of band); without it, the
    // binary64 high-word test keeps a margin inside the band (|log1p(v0)| then
    // stays below LN2 whatever the seed's last bit) and sends the rest away.
    if (D && !UNIFIED) inb[e] = ahi(v[e].v) < (sgn(v[e].v) ? H64_HALF : H64_ONE);
    else if (D) inb[e] = abits(v[e].v) <= (sgn(v[e].v) ? B64_HALF : B64_ONE);
    else inb[e] = v[e].v >= -0.5f && v[e].v <= 1.0f;     // FP pipe (binary32 is ALU-bound)
    T arg = v[e].v;
    n[e] = 0;
    zc0[e] = T(1);
    zc1[e] = T(0);
    if (UNIFIED && !inb[e]) {
      // out-of-band prologue; v0 > -1 keeps w0 = 1 + v0 positive and normal
      if constexpr (D) ok[e] = ok[e] && (inb[e] || !sgn(v[e].v) || ahi(v[e].v) < H64_ONE);
      else ok[e] = ok[e] && (inb[e] || v[e].v > -1.0f);
      TF<T> w = renorm_u(t_add_d_u(v[e], T(1)));
      if constexpr (DBLV) wv[e] = w.v;
      // |d| = |y1 / (1 + y0)| <= ~2^-13 so log1p(d) = d - d^2/2 suffices below
      if constexpr (D) ok[e] = ok[e] && (inb[e] || zbits(y1[e]) || bexp(y1[e]) + DSEP <= bexp(w.v));
      else ok[e] = ok[e] && (inb[e] || fabsf(y1[e]) * 0x1p14f <= fabsf(w.v));  // stricter
      bool band;
      if constexpr (D) band = ubits(w.v) >= C::HALF && ubits(w.v) <= C::TWO;
      else band = w.v >= 0.5f && w.v <= 2.0f;
      int nn = band ? 0 : C::n_of(w.v);
      T c0 = band ? w.v : C::mant(w.v);
      T c1 = band ? w.e : (zbits(w.e) ? T(0) : mul(w.e, C::p2(-nn)));
      if (!inb[e]) {
        n[e] = nn;
        zc0[e] = c0;
        zc1[e] = c1;
        arg = add(sub(c0, T(1)), c1);
      }
    } else {
      ok[e] = ok[e] && inb[e];
    }
    if (!ok[e]) { arg = T(0); inb[e] = true; }
    sd[e] = seed_log1p_t(arg, [&](int i) { return seed_entry(tb, i); });  // explog.py:197-199, 277
    // pexpm10_raw(-sd) must take its in-band branch (|sd| <= LN2); in band this
    // can fail only at v0 = -1/2 or 1 with a seed one ulp beyond ln 2
    if (D && !UNIFIED) ok[e] = ok[e] && (inb[e] || C::in_ln2(sd[e]));
    else if (D) ok[e] = ok[e] && C::in_ln2(sd[e]);
    else ok[e] = ok[e] && fabsf(sd[e]) <= T(P<T>::LN2_V);
    ms[e] = -sd[e];
  }
  TF<T> s[VW];
  pexpm10_inband_v<T, VW>(tb, ms, s);
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    if (inb[e]) {
      TF<T> u;
      if (v[e].e == T(0)) {                              // explog.py:268-270
        TF<T> w = fast_two_sum_u(T(1), v[e].v);
        u = t_add_d_u(t_mul_u(w, s[e]), v[e].v);
      } else {                                           // explog.py:271-273
        TF<T> ys = t_mul_u(v[e], s[e]);
        u = t_add_u(t_add_u(ys, v[e]), s[e]);
      }
      T x1 = add(u.v, u.e);
      ok[e] = ok[e] && newton_quiet(x1, sd[e]);
      if constexpr (PM) {                                 // renorm_fast(_log1p_core)
        TF<T> r = fast_two_sum_u(sd[e], x1);
        z0[e] = r.v;
        z1[e] = r.e;
        continue;
      }
      bool tiny;
      if constexpr (D) tiny = ahi(y0[e]) < H64_TINY54;
      else tiny = fabsf(y0[e]) < 0x1p-25f;
      // v - y0 == y1 exactly; with |d| <= 2^-48 |log1p(y0)| (2^-21 binary32)
      // ~2^-22 accuracy of d suffices; below 2^-54 the value part is y0 itself
      // binary64 needs the refined reciprocal: MUFU alone is 2^-19.9
      // (tools/micro/rcp_acc.cu), which would misround ~1e-6 of the z0
      T d = mul(y1[e], C::rcp(add(T(1), y0[e])));
      if constexpr (D) ok[e] = ok[e] && (tiny || ahi(d) + (48u << 20) <= ahi(sd[e]));
      else ok[e] = ok[e] && (tiny || fabsf(d) * 0x1p21f <= fabsf(sd[e]));
      bool hard;
      T zz;
      if constexpr (DBLV && !D) zz = cr32_lib<DF_LOG1P>(y0[e], hard);
      else zz = rn_guard<TF_TOL32_LOG>(sd[e], sub(x1, d), hard);
      z0[e] = tiny ? y0[e] : zz;
      ok[e] = ok[e] && (tiny || !hard);
      z1[e] = add(x1, sub(sd[e], z0[e]));               // _correct (222-223)
    } else if (UNIFIED) {
      // _newton_log_z (170-186) on (zc0, zc1), then + n ln2 (206-208)
      TF<T> wz = fast_two_sum_u(sub(zc0[e], T(1)), zc1[e]);
      TF<T> u = t_add_u(t_mul_u(mk(zc0[e], zc1[e]), s[e]), wz);
      T r1 = add(u.v, u.e);
      ok[e] = ok[e] && newton_quiet(r1, sd[e]);
      TF<T> nl = t_mul_d_u(mk(P<T>::LN2_V, P<T>::LN2_E), (T)n[e]);
      TF<T> core = t_add_u(mk(sd[e], r1), nl);
      if constexpr (PM && !INNER) {                       // renorm_fast(_log_core(w))
        TF<T> r = n[e] == 0 ? fast_two_sum_u(sd[e], r1) : fast_two_sum_u(core.v, core.e);
        z0[e] = r.v;
        z1[e] = r.e;
        continue;
      }
      // tlogp's value part log(w0) (_correct, 216-223): w1/w0 = zc1/zc0
      // (out-of-band: |log w0| >= ln 2 - tiny, |w1/w0| <= 2^-24)
      T rc = rcp_nr(zc0[e]);
      bool hard0;
      T t0;
      if constexpr (DBLV && !D) {
        t0 = cr32_lib<DF_LOG>(wv[e], hard0);                 // log(w0)
      } else {
        t0 = rn_guard<TF_TOL32_LOG>(core.v, sub(core.e, mul(zc1[e], rc)), hard0);
      }
      ok[e] = ok[e] && !hard0;
      T t1 = add(core.e, sub(core.v, t0));
      if constexpr (PM) {                                 // renorm_fast(tlogp(w))
        TF<T> r = fast_two_sum_u(t0, t1);
        z0[e] = r.v;
        z1[e] = r.e;
        continue;
      }
      // final value part log1p(y0) = log(w) - log1p(y1 / (1 + y0))
      // 1 + y0 ~ w0 = zc0 * 2^n: divide in the scaled domain (1/(1 + y0) can
      // underflow the approximate reciprocal when y0 ~ FLT_MAX)
      T dd = mul(mul(y1[e], C::p2(-n[e])), rc);
      bool hard;
      T zz;
      if constexpr (DBLV && !D) zz = cr32_lib<DF_LOG1P>(y0[e], hard);
      else zz = rn_guard<TF_TOL32_LOG>(core.v, sub(core.e, fmaop(mul(T(-0.5), dd), dd, dd)), hard);
      ok[e] = ok[e] && !hard;
      z0[e] = zz;
      if constexpr (INNER) z1[e] = add(t1, sub(t0, zz));  // _correct (222-223)
      else z1[e] = add(core.e, sub(core.v, zz));
    }
  }
}

// ------------------------------------------ binary32 tlog1p, lane pairs
// fast_tlog1p<float> (UNIFIED, PM = false, INNER = true) with the twofold
// pipeline on f32x2 pairs.  The two branches of _plog1p_raw (explog.py:290-294)
// share one seed, one pexpm10 and one twofold product of the Newton step, with
// per-lane operand selects where they differ:
//   in band:     u = ((v s) + v) + s                (explog.py:271-273)
//   out of band: u = (zc s) + ((zc0 - 1) + zc1)     (explog.py:182-184)
// so both lanes of a pair run one instruction stream whatever their branch.
// The per-lane operation sequence is exactly fast_tlog1p<float>'s; in-band
// lanes with v1 == 0 (explog.py:268-270) take a warp-uniform extra step.
template <int VW, bool RENORM>
TF_DEV void fast_tlog1p_p(const STab<float>& tb, const float (&y0i)[VW], const float (&y1i)[VW],
                          float (&z0)[VW], float (&z1)[VW], bool (&ok)[VW]) {
  static_assert(VW % 2 == 0, "lane pairs");
  constexpr int NP = VW / 2;
  using C = LogC<float>;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const int a = 2 * p, b = 2 * p + 1;
    const float yy0[2] = {y0i[a], y0i[b]}, yy1[2] = {y1i[a], y1i[b]};
    const f2 y0 = pk(yy0[0], yy0[1]), y1 = pk(yy1[0], yy1[1]);
    TF<f2> v = mk(y0, y1);
    if (RENORM) v = renorm_u(v);
    // out-of-band prologue for both lanes: w = renorm(v + 1), then frexp
    const TF<f2> w = renorm_u(t_add_d_u(v, splat(1.0f)));
    const float vv[2] = {lo(v.v), hi(v.v)}, ve[2] = {lo(v.e), hi(v.e)};
    const float wv[2] = {lo(w.v), hi(w.v)}, we[2] = {lo(w.e), hi(w.e)};
    bool k[2], inb[2];
    int n[2];
    float xv[2], xe[2], p2[2], one[2], z1a[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      // finite operands; with RENORM implied by the tests on v below (an
      // infinite or NaN operand or an overflowing sum makes v0 NaN, which is
      // neither in band nor > -1)
      k[h] = RENORM || ((fabsf(yy0[h]) <= 0x1.fffffep127f) & (fabsf(yy1[h]) <= 0x1.fffffep127f));
      inb[h] = (vv[h] >= -0.5f) & (vv[h] <= 1.0f);         // explog.py:291
#ifdef TF_T1P32_PURE
      // measurement builds only (tools/pure_probe.py): branch-pure
      // code, 1 = in band only, 2 = out of band only; other lanes are rejected
      k[h] &= (TF_T1P32_PURE == 1) == inb[h];
      inb[h] = TF_T1P32_PURE == 1;
#endif
      // out of band: v0 > -1 and |y1 / (1 + y0)| <= 2^-14 (log1p(d) = d - d^2/2)
      k[h] &= inb[h] | ((vv[h] > -1.0f) & (fabsf(yy1[h]) * 0x1p14f <= fabsf(wv[h])));
      const bool band = (wv[h] >= 0.5f) & (wv[h] <= 2.0f);
      const int nn = band ? 0 : C::n_of(wv[h]);
      n[h] = inb[h] ? 0 : nn;
      // the Newton product's left operand x: v in band, zc = (zc0, w1 2^-n) out
      xv[h] = inb[h] ? vv[h] : band ? wv[h] : C::mant(wv[h]);
      xe[h] = inb[h] ? ve[h] : we[h];
      p2[h] = (inb[h] | band) ? 1.0f : C::p2(-nn);         // x1 * 1 == x1 exactly
      z1a[h] = (inb[h] | band) ? -0.0f : 0.0f;             // see fast_tlog_p
      one[h] = inb[h] ? 0.0f : 1.0f;
    }
    const f2 xm_v = pk(xv[0], xv[1]);
    const f2 xm_e = fmaop(pk(xe[0], xe[1]), pk(p2[0], p2[1]), pk(z1a[0], z1a[1]));
    const f2 pa = sub(xm_v, pk(one[0], one[1]));           // v0 in band, zc0 - 1 out (exact)
    f2 arg;
    TF<f2> yw;
    if constexpr (RENORM) {
      // renormalised v: RN(v0 + v1) == v0 and fast_two_sum(v0, v1) == (v0, v1)
      // bitwise, so one expression serves both branches
      arg = add(pa, xm_e);
      yw = fast_two_sum_u(pa, xm_e);
    } else {
      arg = sel2(inb[0], inb[1], v.v, add(pa, xm_e));
      const TF<f2> wz = fast_two_sum_u(pa, xm_e);
      yw = mk(sel2(inb[0], inb[1], v.v, wz.v), sel2(inb[0], inb[1], v.e, wz.e));
    }
    const f2 sd = seed_log1p_p(tb, arg);                   // explog.py:197-199, 277
    const float sx[2] = {lo(sd), hi(sd)};
    float ms[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      k[h] &= fabsf(sx[h]) <= P<float>::LN2_V;
      ms[h] = k[h] ? -sx[h] : 0.0f;                         // keeps the CM1 index in range
    }
    const TF<f2> s = pexpm10_inband_p(tb, pk(ms[0], ms[1]));
    // Newton step: one product x s, then + v + s in band, + wz out of band.
    // In band with v1 == 0 (explog.py:268-270) the reference computes
    // t_add_d(t_mul(w, s), v0), w = fast_two_sum(1, v0): the same product and
    // addition with x = w, since yw is (v0, +-0) there and adding a zero error
    // part changes no bit for v0 != 0 (v0 = +-0 goes to the drain).
    f2 xmv = xm_v, xme = xm_e;
    const bool dot[2] = {bool(inb[0] & (ve[0] == 0.0f)), bool(inb[1] & (ve[1] == 0.0f))};
    if (__any_sync(0xffffffffu, dot[0] | dot[1])) {
      const TF<f2> w1 = fast_two_sum_u(splat(1.0f), v.v);
      xmv = sel2(dot[0], dot[1], w1.v, xm_v);
      xme = sel2(dot[0], dot[1], w1.e, xm_e);
#pragma unroll
      for (int h = 0; h < 2; ++h) k[h] &= !(dot[h] & (vv[h] == 0.0f));
    }
    const TF<f2> u1 = t_add_u(t_mul_u(mk(xmv, xme), s), yw);
    const TF<f2> u2 = t_add_u(u1, s);
    const bool two[2] = {bool(inb[0] & !dot[0]), bool(inb[1] & !dot[1])};
    const TF<f2> u = mk(sel2(two[0], two[1], u2.v, u1.v), sel2(two[0], two[1], u2.e, u1.e));
    const f2 x1 = add(u.v, u.e);
    // newton_quiet: |x1| < 2^-21 max(|sd|, 1)
    const f2 lim = mul(pk(fmaxf(fabsf(sx[0]), 1.0f), fmaxf(fabsf(sx[1]), 1.0f)), splat(0x1p-21f));
    const float xx[2] = {lo(x1), hi(x1)}, lm[2] = {lo(lim), hi(lim)};
#pragma unroll
    for (int h = 0; h < 2; ++h) k[h] &= fabsf(xx[h]) < lm[h];
    // + n ln2 (explog.py:206-208).  In band n = 0 and core == (sd, x1) (up to
    // the sign of a zero x1, which no result below can see)
    const TF<f2> nl = t_mul_d_u(mk(splat(P<float>::LN2_V), splat(P<float>::LN2_E)),
                                pk((float)n[0], (float)n[1]));
    const TF<f2> core = t_add_u(mk(sd, x1), nl);
    // one reciprocal per lane: 1 / (1 + y0) in band, 1 / zc0 out of band
    const f2 q = sel2(inb[0], inb[1], add(splat(1.0f), y0), xm_v);
    const f2 r = pk(rcp_approx(lo(q)), rcp_approx(hi(q)));
    const f2 rc = fmaop(r, fmaop(-q, r, splat(1.0f)), r);   // rcp_nr
    // tlogp's value part t0 = log(w0) (_correct, explog.py:216-223); in band
    // t0 = RN(sd - 0) = sd, so that the final _correct below is x1 + (sd - z0)
    bool hard0[2], hard[2];
    const f2 t0 = rn_guard_p(core.v, sel2(inb[0], inb[1], splat(-0.0f), sub(core.e, mul(xm_e, rc))),
                             hard0);
    const f2 t1 = add(core.e, sub(core.v, t0));
    // d = y1 / (1 + y0): in band y1 r, out of band (y1 2^-n) / zc0, which enters
    // as log1p(d) = d - d^2/2 (fast_tlog1p<float>)
    const f2 dd = mul(mul(y1, pk(p2[0], p2[1])), rc);
    const f2 g = fmaop(mul(splat(-0.5f), dd), dd, dd);
    const f2 zz = rn_guard_p(core.v, sub(core.e, sel2(inb[0], inb[1], dd, g)), hard);
    const float dx[2] = {lo(dd), hi(dd)};
    float zx[2] = {lo(zz), hi(zz)};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool tiny = inb[h] & (fabsf(yy0[h]) < 0x1p-25f);
      const bool okin = tiny | ((fabsf(dx[h]) * 0x1p21f <= fabsf(sx[h])) & !hard[h]);
      k[h] &= inb[h] ? okin : !(hard0[h] | hard[h]);
      zx[h] = tiny ? yy0[h] : zx[h];
    }
    const f2 zr = add(t1, sub(t0, pk(zx[0], zx[1])));      // _correct (222-223)
    z0[a] = zx[0];
    z0[b] = zx[1];
    z1[a] = lo(zr);
    z1[b] = hi(zr);
    ok[a] = k[0];
    ok[b] = k[1];
  }
}

// ------------------------------------- binary32 texp / texpm1, lane pairs
// fast_texp<float> / fast_texpm1<float> with the recombination on f32x2
// pairs too: C and E entries of the two lanes loaded straight into register
// pairs (ldpair), the two twofold products, the value-part guard and z1 packed.
// The per-lane operation sequence is exactly the scalar kernels'.
TF_DEV TF<f2> taylor_exp_p(f2 yp) {                 // taylor_exp_v<float>'s packed body
  const f2 nyp = -yp;
  f2 s = add(yp, splat(6.0f));
  s = add(mul(s, yp), splat(30.0f));
  TF<f2> tp = mk(s, splat(0.0f));
  tp = t_add_d_u(t_mul_d_pz(tp, yp, nyp), splat(c_texp32[0]));
#pragma unroll
  for (int k = 1; k < 4; ++k) tp = t_add_d_u(t_mul_d_p(tp, yp, nyp), splat(c_texp32[k]));
  return tp;
}

// decompose_exp (expcore.py:35-48) of a lane pair: M = RNE(32 x) by the magic
// constant and the exact y = x - M/32 as two packed FMAs and one FADD2 (the
// same IEEE ops per lane as decomp_exp_u), then m, n = sign(M) (|M| div/mod 64)
// as (M + (M < 0 ? 63 : 0)) >> 6 and M - 64 m.  Rejected lanes take M = 0 (the
// table indices stay in range; their y is discarded with their result).
TF_DEV f2 decomp_exp_p(f2 x, const bool (&okp)[2], int (&m)[2], int (&n)[2]) {
  const f2 mg = splat(12582912.0f);                     // 1.5 * 2^23
  const f2 t = fmaop(x, splat(32.0f), mg);
  const f2 y = fmaop(sub(t, mg), splat(-0.03125f), x);
  const float tl[2] = {lo(t), hi(t)};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int M = okp[h] ? (int)ubits(tl[h]) - 0x4b400000 : 0;
    m[h] = (M + ((M >> 31) & 63)) >> 6;
    n[h] = M - (m[h] << 6);
  }
  return y;
}

template <int VW, bool PM = false>
TF_DEV void fast_texp_p(const STab<float>& tb, const float (&x0)[VW], const float (&x1)[VW],
                        float (&z0)[VW], float (&z1)[VW], bool (&ok)[VW]) {
  static_assert(VW % 2 == 0, "lane pairs");
  int m[VW], n[VW];
#pragma unroll
  for (int e = 0; e < VW; ++e)
    ok[e] = x0[e] >= -__uint_as_float(B32_TEXP_NEG) && x0[e] <= __uint_as_float(B32_TEXP_POS) &&
            fabsf(x1[e]) < __uint_as_float(B32_X1_TINY);
#pragma unroll
  for (int p = 0; p < VW / 2; ++p) {
    const int a = 2 * p, b = 2 * p + 1;
    int mm[2], nn[2];
    const f2 yp = decomp_exp_p(pk(x0[a], x0[b]), {ok[a], ok[b]}, mm, nn);
    m[a] = mm[0]; m[b] = mm[1]; n[a] = nn[0]; n[b] = nn[1];
    const TF<f2> t = taylor_exp_p(yp);
    const TF<f2> ct = t_mul_u(ldpair(tb.C, n[a] - P<float>::C_LO, n[b] - P<float>::C_LO), t);
    const TF<f2> ev = ldpair(tb.E, m[a] - P<float>::E_LO, m[b] - P<float>::E_LO);
    const TF<f2> v = t_mul_u(ev, ct);
    if constexpr (PM) {
      const TF<f2> r = fast_two_sum_u(v.v, v.e);
      z0[a] = lo(r.v); z0[b] = hi(r.v);
      z1[a] = lo(r.e); z1[b] = hi(r.e);
      continue;
    }
    // value part near the subnormal range from the 2^64-scaled coarse table
    const bool sc0 = m[a] <= -35, sc1 = m[b] <= -35;
    const TF<f2> es = ldpair(tb.ESC, sc0 ? m[a] - TF32_ESC_LO : 0, sc1 ? m[b] - TF32_ESC_LO : 0);
    const TF<f2> vs = t_mul_u(mk(sel2(sc0, sc1, es.v, ev.v), sel2(sc0, sc1, es.e, ev.e)), ct);
    bool hard[2];
    const f2 zz = mul(rn_guard_p<TF_TOL32_EXP>(vs.v, vs.e, hard),
                      pk(sc0 ? 0x1p-64f : 1.0f, sc1 ? 0x1p-64f : 1.0f));
    ok[a] = ok[a] && !hard[0];
    ok[b] = ok[b] && !hard[1];
    const f2 t1 = pk(t1_tiny(x1[a]), t1_tiny(x1[b]));
    const f2 zr = add(mul(zz, t1), add(v.e, sub(v.v, zz)));   // explog.py:125
    z0[a] = lo(zz); z0[b] = hi(zz);
    z1[a] = lo(zr); z1[b] = hi(zr);
  }
}

template <int VW, bool PM = false>
TF_DEV void fast_texpm1_p(const STab<float>& tb, const float (&x0)[VW], const float (&x1)[VW],
                          float (&z0)[VW], float (&z1)[VW], bool (&ok)[VW]) {
  static_assert(VW % 2 == 0, "lane pairs");
  int m[VW], n[VW];
#pragma unroll
  for (int e = 0; e < VW; ++e)
    ok[e] = fabsf(x0[e]) > __uint_as_float(B32_LN2) && x0[e] >= -__uint_as_float(B32_LO) &&
            x0[e] <= __uint_as_float(B32_TEXP_POS) && fabsf(x1[e]) < __uint_as_float(B32_X1_TINY);
#pragma unroll
  for (int p = 0; p < VW / 2; ++p) {
    const int a = 2 * p, b = 2 * p + 1;
    int mm[2], nn[2];
    const f2 yp = decomp_exp_p(pk(x0[a], x0[b]), {ok[a], ok[b]}, mm, nn);
    m[a] = mm[0]; m[b] = mm[1]; n[a] = nn[0]; n[b] = nn[1];
    const TF<f2> t = taylor_exp_p(yp);
    const TF<f2> v = t_mul_u(ldpair(tb.E, m[a] - P<float>::E_LO, m[b] - P<float>::E_LO),
                             t_mul_u(ldpair(tb.C, n[a] - P<float>::C_LO, n[b] - P<float>::C_LO), t));
    const TF<f2> w = t_add_d_u(v, splat(-1.0f));             // expcore.py:147
    if constexpr (PM) {
      const TF<f2> r = fast_two_sum_u(w.v, w.e);
      z0[a] = lo(r.v); z0[b] = hi(r.v);
      z1[a] = lo(r.e); z1[b] = hi(r.e);
      continue;
    }
    bool hard[2];
    const f2 zz = rn_guard_p<TF_TOL32_EXP>(w.v, w.e, hard);
    ok[a] = ok[a] && !hard[0];
    ok[b] = ok[b] && !hard[1];
    const f2 tail = add(w.e, sub(w.v, zz));
    const f2 t1 = pk(t1_tiny(x1[a]), t1_tiny(x1[b]));
    const f2 zr = add(mul(add(zz, splat(1.0f)), t1), tail);   // explog.py:159-160
    z0[a] = lo(zz); z0[b] = hi(zz);
    z1[a] = lo(zr); z1[b] = hi(zr);
  }
}

// Per-warp exchange buffer for class-sorting the 32 x VW elements of a warp
// iteration (binary32 tlog1p, whose in-band / out-of-band split is ~50/50).
template <int VW> struct Xch {
  float a[32 * VW], b[32 * VW];
  unsigned char src[32 * VW], okb[32 * VW];
};

// binary32 tlog1p: sort the warp's elements by branch before evaluating, so
// that every lane index except one holds a single class across the warp and
// the in-band / out-of-band epilogues no longer run back to back under
// divergence.  Element k = e*32 + lane goes to slot rank_A(k) (in-band) or
// n_A + rank_B(k); results travel back through the same buffer.
template <int VW, bool RENORM, bool PM, bool INNER>
TF_DEV void tlog1p_sorted(const STab<float>& tb, Xch<VW>* xw, const float (&x0)[VW],
                          const float (&x1)[VW], float (&z0)[VW], float (&z1)[VW],
                          bool (&ok)[VW]) {
  const int lane = threadIdx.x & 31;
  unsigned m[VW];
  int pre[VW], nA = 0;
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    bool fin = fabsf(x0[e]) <= 0x1.fffffep127f && fabsf(x1[e]) <= 0x1.fffffep127f;
    TF<float> v = mk(fin ? x0[e] : 0.0f, fin ? x1[e] : 0.0f);
    if (RENORM) v = renorm_u(v);
    bool inb = v.v >= -0.5f && v.v <= 1.0f;
    m[e] = __ballot_sync(0xffffffffu, inb);
    pre[e] = nA;
    nA += __popc(m[e]);
  }
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    int k = e * 32 + lane;
    int ra = pre[e] + __popc(m[e] & lt);
    int dst = (m[e] >> lane & 1u) ? ra : nA + (k - ra);
    xw->a[dst] = x0[e];
    xw->b[dst] = x1[e];
    xw->src[dst] = (unsigned char)k;
  }
  __syncwarp();
  float p0[VW], p1[VW], q0[VW], q1[VW];
  int sk[VW];
  bool pok[VW];
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    p0[e] = xw->a[e * 32 + lane];
    p1[e] = xw->b[e * 32 + lane];
    sk[e] = xw->src[e * 32 + lane];
  }
  __syncwarp();
  // (a lane-pair f32x2 variant of this body was tried: register pressure at
  // 64 registers made it 5% slower, and 512-thread CTAs without spills 11%)
  fast_tlog1p<float, VW, RENORM, PM, INNER>(tb, p0, p1, q0, q1, pok);
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    xw->a[sk[e]] = q0[e];
    xw->b[sk[e]] = q1[e];
    xw->okb[sk[e]] = pok[e];
  }
  __syncwarp();
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    z0[e] = xw->a[e * 32 + lane];
    z1[e] = xw->b[e * 32 + lane];
    ok[e] = xw->okb[e * 32 + lane] != 0;
  }
  __syncwarp();
}

// Second-chance evaluator of the rare-element drain (binary64): the branch the
// main fast path leaves out -- texpm1's pexp0 - 1 fallback, tlog1p's
// out-of-band tlogp(renorm(1 + y)) -- run lane-scalar on the queued elements;
// elements it does not admit go on to the exact path.  Exact-path cost per
// element is ~10x this, and these branches are most of cfg 2's rare elements.
template <class T, int FN> struct HasAlt {
  static constexpr bool value =
      sizeof(T) == 4 ||
      (FN == FN_TEXP || FN == FN_TEXPP || FN == FN_TEXP0 || FN == FN_PEXP0 ||
       FN == FN_TEXPM1 || FN == FN_TEXPM10 || FN == FN_PEXPM10 || FN == FN_PEXPM1 ||
       FN == FN_TLOG1P || FN == FN_TLOG1P0 || FN == FN_TLOG1PP || FN == FN_PLOG1P ||
       FN == FN_PLOG1P0 || FN == FN_TLOG || FN == FN_TLOG0 || FN == FN_TLOGP ||
       FN == FN_PLOG || FN == FN_PLOG0);
};

// binary32 second chance: the same fast cores with the value part from the
// binary64 library instead of the 2^-36 rounding guard (which sends ~0.05% of
// elements away), and texpm1's in-band branch
template <int FN>
TF_DEV bool fast_alt32(const STab<float>& tb, float x0, float x1, float& z0, float& z1) {
  float a[1] = {x0}, b[1] = {x1}, r0[1], r1[1];
  bool ok[1];
  if constexpr (FN == FN_TEXP || FN == FN_TEXPP || FN == FN_TEXP0 || FN == FN_PEXP) {
    fast_texp<1, false, true>(tb, a, b, r0, r1, ok);
  } else if constexpr (FN == FN_PEXP0) {
    return false;                                  // no value part to guard
  } else if constexpr (FN == FN_TEXPM1 || FN == FN_TEXPM1P || FN == FN_TEXPM10 ||
                       FN == FN_PEXPM1 || FN == FN_PEXPM10) {
    constexpr bool PM = FN == FN_PEXPM10;
    if (abits(x0) <= B32_LN2) fast_texpm1_inb32<PM>(tb, x0, x1, r0[0], r1[0], ok[0]);
    else if constexpr (PM) return false;
    else fast_texpm1<1, false, true>(tb, a, b, r0, r1, ok);
  } else if constexpr (FN == FN_TLOG || FN == FN_TLOG0) {
    fast_tlog<float, 1, true, false, true>(tb, a, b, r0, r1, ok);
  } else if constexpr (FN == FN_TLOGP) {
    fast_tlog<float, 1, false, false, true>(tb, a, b, r0, r1, ok);
  } else if constexpr (FN == FN_PLOG0 || FN == FN_PLOG) {
    return false;
  } else {
    constexpr bool RENORM = FN == FN_TLOG1P;
    constexpr bool PM = FN == FN_PLOG1P0 || FN == FN_PLOG1P;
    constexpr bool INNER = !(FN == FN_TLOG1P0 || FN == FN_PLOG1P0);
    fast_tlog1p<float, 1, RENORM, PM, INNER, 1, true>(tb, a, b, r0, r1, ok);
  }
  if constexpr (FN == FN_PEXP || FN == FN_PEXPM1) {
    TF<float> r = fast_two_sum_u(r0[0], r1[0]);
    r0[0] = r.v;
    r1[0] = r.e;
  }
  z0 = r0[0];
  z1 = r1[0];
  return ok[0];
}
// binary64 out-of-band tlog1p / tlog1pp / plog1p when 1 + y0 is exact (e.g.
// cfg 2's clamp value y0 = -1 + 2^-52, whose tail y1 is O(1 + y0), so the
// unified branch's d = y1 / (1 + y0) is not small): tlogp(w), w = renorm(1 + v)
// (explog.py:290-294, 239-242), and the value part CR log1p(y0) = CR log(1 + y0)
// from a second tlog core on the exact argument.
template <int FN>
TF_DEV bool alt_log1p_exact1p(const STab<double>& tb, double y0, double y1, double& z0,
                              double& z1) {
  constexpr bool RENORM = FN == FN_TLOG1P;
  constexpr bool PM = FN == FN_PLOG1P;
  if (!is_finite(y0) || !is_finite(y1)) return false;
  TF<double> v = RENORM ? renorm_u(mk(y0, y1)) : mk(y0, y1);
  if (!(v.v < -0.5 || v.v > 1.0) || !(v.v > -1.0)) return false;
  TF<double> w = renorm_u(t_add_d_u(v, 1.0));
  double a[1] = {w.v}, b[1] = {w.e}, t0[1], t1[1];
  bool ok[1];
  fast_tlog<double, 1, false>(tb, a, b, t0, t1, ok);         // tlogp(w)
  if (!ok[0]) return false;
  if constexpr (PM) {                                          // renorm_fast(tlogp(w))
    TF<double> r = fast_two_sum_u(t0[0], t1[0]);
    z0 = r.v;
    z1 = r.e;
    return true;
  } else {
    TF<double> u = two_sum_u(1.0, y0);
    if (!zbits(u.e)) return false;                             // 1 + y0 not exact
    double c[1] = {u.v}, d[1] = {0.0}, l0[1], l1[1];
    fast_tlog<double, 1, false>(tb, c, d, l0, l1, ok);       // CR log(1 + y0)
    if (!ok[0]) return false;
    z0 = l0[0];
    z1 = add(t1[0], sub(t0[0], z0));                          // _correct (222-223)
    return true;
  }
}

// DR queued elements per lane at once (independent chains: the drain's
// evaluation is latency-bound with one)
template <int FN, int DR>
TF_DEV void fast_alt64_v(const STab<double>& tb, const double (&x0)[DR], const double (&x1)[DR],
                         double (&z0)[DR], double (&z1)[DR], bool (&ok)[DR]) {
  using T = double;
  constexpr bool L1P = FN == FN_TLOG1P || FN == FN_TLOG1PP || FN == FN_PLOG1P;
  // log1p family: the unified branch below admits |y1| <= 2^-52 |1 + y0| (its
  // d test) with one evaluation; alt_log1p_exact1p costs two and serves the
  // arguments with a larger tail (cfg 2's clamp value y0 = -1 + 2^-52), so it
  // goes first only for those
  bool small_d[DR], pre[DR];
#pragma unroll
  for (int k = 0; k < DR; ++k) {
    small_d[k] = true;
    pre[k] = false;
    if constexpr (L1P) {
      small_d[k] = zbits(x1[k]) || bexp(x1[k]) + 52 <= bexp(add(1.0, x0[k]));
      if (!small_d[k]) pre[k] = alt_log1p_exact1p<FN>(tb, x0[k], x1[k], z0[k], z1[k]);
    }
  }
  T r0[DR], r1[DR];
  if constexpr (FN == FN_TEXP || FN == FN_TEXPP || FN == FN_TEXP0) {   // subnormal / near-overflow
    fast_texp<DR, false, true>(tb, x0, x1, r0, r1, ok);
  } else if constexpr (FN == FN_PEXP0) {
    fast_texp<DR, true, true>(tb, x0, x1, r0, r1, ok);
  } else if constexpr (FN == FN_TEXPM1 || FN == FN_TEXPM10 || FN == FN_PEXPM1) {
    fast_texpm1_fb<DR>(tb, x0, x1, r0, r1, ok);
    if constexpr (FN == FN_PEXPM1) {
#pragma unroll
      for (int k = 0; k < DR; ++k) {
        TF<T> r = fast_two_sum_u(r0[k], r1[k]);
        r0[k] = r.v;
        r1[k] = r.e;
      }
    }
  } else if constexpr (FN == FN_PEXPM10) {
    fast_texpm1_fb<DR, true>(tb, x0, x1, r0, r1, ok);
  } else if constexpr (FN == FN_TLOG || FN == FN_TLOG0) {       // top binade
    fast_tlog<T, DR, true, false, false, true>(tb, x0, x1, r0, r1, ok);
  } else if constexpr (FN == FN_TLOGP) {
    fast_tlog<T, DR, false, false, false, true>(tb, x0, x1, r0, r1, ok);
  } else if constexpr (FN == FN_PLOG0 || FN == FN_PLOG) {
    fast_tlog<T, DR, false, true, false, true>(tb, x0, x1, r0, r1, ok);
  } else {
    constexpr bool RENORM = FN == FN_TLOG1P;
    constexpr bool PM = FN == FN_PLOG1P0 || FN == FN_PLOG1P;
    constexpr bool INNER = !(FN == FN_TLOG1P0 || FN == FN_PLOG1P0);
    fast_tlog1p<T, DR, RENORM, PM, INNER, 1>(tb, x0, x1, r0, r1, ok);
  }
#pragma unroll
  for (int k = 0; k < DR; ++k) {
    if (pre[k]) {
      ok[k] = true;                                 // z0 / z1 set by alt_log1p_exact1p
      continue;
    }
    if constexpr (L1P)
      if (!ok[k] && small_d[k]) {
        ok[k] = alt_log1p_exact1p<FN>(tb, x0[k], x1[k], z0[k], z1[k]);
        continue;
      }
    z0[k] = r0[k];
    z1[k] = r1[k];
  }
}

template <int FN>
TF_DEV bool fast_alt64(const STab<double>& tb, double x0, double x1, double& z0, double& z1) {
  double a[1] = {x0}, b[1] = {x1}, r0[1], r1[1];
  bool ok[1];
  fast_alt64_v<FN, 1>(tb, a, b, r0, r1, ok);
  z0 = r0[0];
  z1 = r1[0];
  return ok[0];
}

// texpm1 / texpm1p / texpm10 saturated classes (explog.py:149-160 with
// pexpm10_raw's fallback t_add_d(pexp0_raw(x0), -1), expcore.py:138-147):
// NaN -> (NaN, NaN); x0 >= hi_bound -> (inf, inf) (the guard, explog.py:155);
// x0 < lo_bound with a tiny tail -> w = (-1, +0), z0 = expm1(x0) = -1 and z1 by
// the texpm1 epilogue (+0 for finite tiny x1).
template <class T> TF_DEV bool texpm1_special(T x0, T x1, T& z0, T& z1) {
  if (is_nan(x0)) {
    z0 = z1 = Lim<T>::qnan();
    return true;
  }
  if (x0 >= P<T>::HI) {
    z0 = z1 = Lim<T>::inf();
    return true;
  }
  const bool tiny1 = sizeof(T) == 8 ? ahi(x1) < H64_X1_TINY : (uint32_t)ahi(x1) < B32_X1_TINY;
  if (x0 < P<T>::LO && tiny1) {
    const T w0 = T(-1), w1 = T(0);
    z0 = T(-1);
    const T tail = add(w1, sub(w0, z0));
    z1 = add(mul(add(z0, T(1)), t1_tiny(x1)), tail);
    return true;
  }
  return false;
}

// tlog1p / tlog1pp / tlog1p0 constant classes (_correct with log1p(y0),
// explog.py:216-223, 305-317): y0 NaN or below -1 -> log1p(y0) = NaN ->
// (NaN, NaN); y0 = -1 with y1 = +-0 -> the core is tlogp(0, 0) = (-inf, -inf)
// and log1p(-1) = -inf -> (-inf, -inf); y0 = +inf, y1 finite -> (inf, inf).
template <class T> TF_DEV bool log1p_special(T y0, T y1, T& z0, T& z1) {
  if (is_nan(y0) || y0 < T(-1)) {
    z0 = z1 = Lim<T>::qnan();
    return true;
  }
  if (y0 == T(-1) && y1 == T(0)) {
    z0 = z1 = -Lim<T>::inf();
    return true;
  }
  if (is_inf(y0) && y0 > T(0) && is_finite(y1)) {
    z0 = z1 = Lim<T>::inf();
    return true;
  }
  return false;
}

// Constant-result classes of the rare elements (specials), resolved in the
// drain with a few selects before any evaluation: texp / texpp / texp0
// (texp_special), texpm1 / texpm1p / texpm10, tlog / tlog0 / tlogp
// (log_const_class) and tlog1p / tlog1pp / tlog1p0.
template <class T, int FN>
TF_DEV bool special_const(T x0, T x1, T& z0, T& z1) {
  if constexpr (sizeof(T) == 8 && (FN == FN_TEXP || FN == FN_TEXPP || FN == FN_TEXP0)) {
    return texp_special(x0, x1, z0, z1);
  } else if constexpr (FN == FN_TEXPM1 || FN == FN_TEXPM1P || FN == FN_TEXPM10) {
    return texpm1_special(x0, x1, z0, z1);
  } else if constexpr (FN == FN_TLOG || FN == FN_TLOG0 || FN == FN_TLOGP) {
    return log_const_apply(log_const_class(x0, x1), z0, z1);
  } else if constexpr (FN == FN_TLOG1P || FN == FN_TLOG1PP || FN == FN_TLOG1P0) {
    return log1p_special(x0, x1, z0, z1);
  } else {
    return false;
  }
}

template <class T, int FN>
TF_DEV bool fast_alt(const STab<T>& tb, T x0, T x1, T& z0, T& z1) {
  if constexpr (sizeof(T) == 4) {
    return fast_alt32<FN>(tb, x0, x1, z0, z1);
  } else {
    return fast_alt64<FN>(tb, x0, x1, z0, z1);
  }
}

// binary32 exponential families with the recombination on lane pairs
#ifndef TF_EXP32_PACKED
#define TF_EXP32_PACKED 1
#endif
// binary32 tlog1p / tlog1pp run on lane pairs (fast_tlog1p_p); the other
// log1p-family functions are class-sorted (tlog1p_sorted)
#ifndef TF_TLOG1P32_PACKED
#define TF_TLOG1P32_PACKED 1
#endif
__host__ __device__ constexpr bool log1p_packed32(int fn) {
  return TF_TLOG1P32_PACKED && (fn == FN_TLOG1P || fn == FN_TLOG1PP);
}
__host__ __device__ constexpr bool log1p_fn(int fn) {
  return !log1p_packed32(fn) && (fn == FN_TLOG1P || fn == FN_TLOG1P0 || fn == FN_TLOG1PP ||
                                 fn == FN_PLOG1P || fn == FN_PLOG1P0);
}

// All twenty functions (explog.py:101-325) on the admission-band cores.  The
// dotted ones arrive with x1 = 0: texp0 / texpm10 / tlog0 are then bitwise the
// twofold functions (t1 = expm1(0) = 0 adds +0 to a nonzero-or-+0 tail; renorm
// of (y0, 0) is the identity), which tests/test_gpu_parity.py checks against
// the exact path.
template <class T, int FN, int VW>
TF_DEV void fast_eval(const STab<T>& tb, void* xch, const T (&x0)[VW], const T (&x1)[VW],
                      T (&z0)[VW], T (&z1)[VW], bool (&ok)[VW]) {
  constexpr bool PK = sizeof(T) == 4 && VW % 2 == 0 && TF_EXP32_PACKED;
  if constexpr (FN == FN_TEXP || FN == FN_TEXPP || FN == FN_TEXP0 || FN == FN_PEXP) {
    if constexpr (PK) fast_texp_p<VW>(tb, x0, x1, z0, z1, ok);
    else fast_texp<VW>(tb, x0, x1, z0, z1, ok);
  } else if constexpr (FN == FN_PEXP0) {
    if constexpr (PK) fast_texp_p<VW, true>(tb, x0, x1, z0, z1, ok);
    else fast_texp<VW, true>(tb, x0, x1, z0, z1, ok);
  } else if constexpr (FN == FN_TEXPM1 || FN == FN_TEXPM1P || FN == FN_TEXPM10 ||
                       FN == FN_PEXPM1) {
    if constexpr (PK) fast_texpm1_p<VW>(tb, x0, x1, z0, z1, ok);
    else fast_texpm1<VW>(tb, x0, x1, z0, z1, ok);
  } else if constexpr (FN == FN_PEXPM10) {
    if constexpr (PK) fast_texpm1_p<VW, true>(tb, x0, x1, z0, z1, ok);
    else fast_texpm1<VW, true>(tb, x0, x1, z0, z1, ok);
  } else if constexpr (FN == FN_TLOG || FN == FN_TLOG0) {
    if constexpr (sizeof(T) == 4 && VW % 2 == 0) fast_tlog_p<VW, true>(tb, x0, x1, z0, z1, ok);
    else fast_tlog<T, VW>(tb, x0, x1, z0, z1, ok);
  } else if constexpr (FN == FN_TLOGP) {
    if constexpr (sizeof(T) == 4 && VW % 2 == 0) fast_tlog_p<VW, false>(tb, x0, x1, z0, z1, ok);
    else fast_tlog<T, VW, false>(tb, x0, x1, z0, z1, ok);
  } else if constexpr (FN == FN_PLOG0 || FN == FN_PLOG) {
    fast_tlog<T, VW, false, true>(tb, x0, x1, z0, z1, ok);
  } else {
    constexpr bool RENORM = FN == FN_TLOG1P;
    constexpr bool PM = FN == FN_PLOG1P0 || FN == FN_PLOG1P;
    constexpr bool INNER = !(FN == FN_TLOG1P0 || FN == FN_PLOG1P0);
    if constexpr (sizeof(T) == 4 && VW % 2 == 0 && log1p_packed32(FN))
      fast_tlog1p_p<VW, RENORM>(tb, x0, x1, z0, z1, ok);
    else if constexpr (sizeof(T) == 4 && VW >= 2)
      tlog1p_sorted<VW, RENORM, PM, INNER>(tb, static_cast<Xch<VW>*>(xch), x0, x1, z0, z1, ok);
    else
      fast_tlog1p<T, VW, RENORM, PM, INNER>(tb, x0, x1, z0, z1, ok);
  }
  if constexpr (FN == FN_PEXP || FN == FN_PEXPM1) {
    // renorm_fast(texpp / texpm1p) (explog.py:131-133, 165-166); a non-finite
    // sum takes the _special policy (eft.py:65-74): exact path
#pragma unroll
    for (int e = 0; e < VW; ++e) {
      TF<T> r = fast_two_sum_u(z0[e], z1[e]);
      z0[e] = r.v;
      z1[e] = r.e;
      ok[e] = ok[e] && is_finite(r.v);
    }
  }
}

}  // namespace tf
