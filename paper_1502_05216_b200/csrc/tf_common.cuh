// tf_common.cuh -- device twofold arithmetic for the B200 kernels.
//
// Every primitive is written with explicit round-to-nearest intrinsics
// (__dadd_rn/__dmul_rn/__fma_rn and the float forms), which nvcc never
// contracts or reassociates, so each kernel executes the same IEEE operation
// sequence as the reference package (pkg/src/twofold/eft.py:77-237,
// eft32.py:36-190) with the "fma" residual backend (eft.py:254-255).
// The TU is additionally compiled with -fmad=false -ftz=false.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tf_tables.h"

#define TF_DEV __device__ __forceinline__

namespace tf {

// ---------------------------------------------------------------- IEEE ops
TF_DEV double add(double a, double b) { return __dadd_rn(a, b); }
TF_DEV double sub(double a, double b) { return __dsub_rn(a, b); }
TF_DEV double mul(double a, double b) { return __dmul_rn(a, b); }
TF_DEV double fmaop(double a, double b, double c) { return __fma_rn(a, b, c); }
TF_DEV float add(float a, float b) { return __fadd_rn(a, b); }
TF_DEV float sub(float a, float b) { return __fsub_rn(a, b); }
TF_DEV float mul(float a, float b) { return __fmul_rn(a, b); }
TF_DEV float fmaop(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// Packed binary32 pairs: Blackwell's FADD2/FMUL2/FFMA2 evaluate two IEEE
// round-to-nearest binary32 ops per instruction (same FP32 pipe rate, half the
// issue slots).  Two independent lanes of a binary32 kernel ride in one f2.
struct f2 { unsigned long long u; };
TF_DEV f2 pk(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.u) : "f"(a), "f"(b));
  return r;
}
TF_DEV float lo(f2 x) { return __uint_as_float((unsigned)(x.u & 0xffffffffull)); }
TF_DEV float hi(f2 x) { return __uint_as_float((unsigned)(x.u >> 32)); }
TF_DEV f2 add(f2 a, f2 b) { f2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(a.u), "l"(b.u)); return r; }
TF_DEV f2 sub(f2 a, f2 b) { f2 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(a.u), "l"(b.u)); return r; }
// ptxas (CUDA 12.9) contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even
// under -fmad=false (and rewrites fma(a, b, -0) back into FMUL2 first), which
// would change the reference's rounding.  A product is therefore issued as
// fma(a, b, z) with z = (-0, -0) read from constant memory: RN(a*b) exactly,
// but opaque to ptxas, so it can neither be turned into FMUL2 nor fused.
__constant__ unsigned long long c_nz2 = 0x8000000080000000ull;
TF_DEV f2 mul(f2 a, f2 b) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.u) : "l"(a.u), "l"(b.u), "l"(c_nz2));
  return r;
}
TF_DEV f2 fmaop(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.u) : "l"(a.u), "l"(b.u), "l"(c.u));
  return r;
}
// sign flip per half as neg.f32: ptxas folds it into the consuming FFMA2 /
// FADD2 as an operand modifier (a 64-bit XOR would cost two LOP3s)
TF_DEV f2 operator-(f2 a) { return pk(-lo(a), -hi(a)); }
TF_DEV f2 splat(float c) { return pk(c, c); }

// ------------------------------------------------- integer-pipe classifiers
TF_DEV int hi32(double x) { return __double2hiint(x); }
TF_DEV uint32_t ubits(float x) { return __float_as_uint(x); }
TF_DEV uint64_t ubits(double x) { return (uint64_t)__double_as_longlong(x); }
// |x| as ordered integer bits (NaN sorts above +inf)
TF_DEV uint64_t abits(double x) { return ubits(x) & 0x7fffffffffffffffull; }
TF_DEV uint32_t abits(float x) { return ubits(x) & 0x7fffffffu; }
TF_DEV bool is_finite(double x) { return (hi32(x) & 0x7ff00000) != 0x7ff00000; }
TF_DEV bool is_finite(float x) { return (ubits(x) & 0x7f800000u) != 0x7f800000u; }
TF_DEV bool is_nan(double x) { return abits(x) > 0x7ff0000000000000ull; }
TF_DEV bool is_nan(float x) { return abits(x) > 0x7f800000u; }
TF_DEV bool is_inf(double x) { return abits(x) == 0x7ff0000000000000ull; }
TF_DEV bool is_inf(float x) { return abits(x) == 0x7f800000u; }
// |x| high word / zero test on the integer pipe (a 64-bit "& 0x7fff..." mask
// is pattern-matched into DADD |x|, which would burn an FP64 pipe slot)
TF_DEV uint32_t ahi(double x) { return (uint32_t)__double2hiint(x) & 0x7fffffffu; }
TF_DEV uint32_t ahi(float x) { return __float_as_uint(x) & 0x7fffffffu; }
TF_DEV bool zbits(double x) { return ((__double2hiint(x) & 0x7fffffff) | __double2loint(x)) == 0; }
TF_DEV bool zbits(float x) { return (__float_as_uint(x) & 0x7fffffffu) == 0; }
// biased exponent field
TF_DEV int bexp(double x) { return (hi32(x) >> 20) & 0x7ff; }
TF_DEV int bexp(float x) { return (int)((ubits(x) >> 23) & 0xff); }

template <class T> struct Lim;
template <> struct Lim<double> {
  TF_DEV static double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }
  TF_DEV static double inf() { return __longlong_as_double(0x7ff0000000000000ll); }
};
template <> struct Lim<float> {
  TF_DEV static float qnan() { return __int_as_float(0x7fc00000); }
  TF_DEV static float inf() { return __int_as_float(0x7f800000); }
};

// ---------------------------------------------------------------- twofold
template <class T> struct TF { T v, e; };
template <class T> TF_DEV TF<T> mk(T v, T e) { TF<T> r; r.v = v; r.e = e; return r; }

// Reference non-finite policy _special (eft.py:65-74).
template <class T> TF_DEV TF<T> special(T v, bool any_nan) {
  if (is_nan(v)) return mk(v, v);
  return mk(v, any_nan ? Lim<T>::qnan() : v);
}

// -- unchecked primitives: identical op sequences, no finiteness test.  Used
//    on the fast paths, whose admission band proves every value finite.
template <class T> TF_DEV TF<T> fast_two_sum_u(T a, T b) {     // eft.py:77-82
  T s = add(a, b);
  return mk(s, sub(b, sub(s, a)));
}
template <class T> TF_DEV TF<T> two_sum_u(T a, T b) {          // eft.py:85-92
  T s = add(a, b);
  T bp = sub(s, a);
  T ap = sub(s, bp);
  return mk(s, add(sub(a, ap), sub(b, bp)));
}
template <class T> TF_DEV TF<T> renorm_u(TF<T> x) {            // eft.py:168-171
  TF<T> t = two_sum_u(x.v, x.e);
  return fast_two_sum_u(t.v, t.e);
}
template <class T> TF_DEV TF<T> t_add_u(TF<T> x, TF<T> y) {    // eft.py:182-189
  T s = add(x.v, y.v);
  T bp = sub(s, x.v);
  T ap = sub(s, bp);
  T e = add(sub(x.v, ap), sub(y.v, bp));
  return mk(s, add(e, add(x.e, y.e)));
}
template <class T> TF_DEV TF<T> t_add_d_u(TF<T> x, T b) {      // eft.py:192-199
  T s = add(x.v, b);
  T bp = sub(s, x.v);
  T ap = sub(s, bp);
  T e = add(sub(x.v, ap), sub(b, bp));
  return mk(s, add(e, x.e));
}
template <class T> TF_DEV TF<T> t_mul_u(TF<T> x, TF<T> y) {    // eft.py:207-212
  T v = mul(x.v, y.v);
  T e = fmaop(x.v, y.v, -v);
  return mk(v, add(e, add(mul(x.v, y.e), mul(x.e, y.v))));
}
template <class T> TF_DEV TF<T> t_mul_d_u(TF<T> x, T b) {      // eft.py:214-219
  T v = mul(x.v, b);
  T e = fmaop(x.v, b, -v);
  return mk(v, add(mul(x.e, b), e));
}

// -- checked primitives: full reference semantics incl. _special.
template <class T> TF_DEV bool n2(T a, T b) { return is_nan(a) | is_nan(b); }
template <class T> TF_DEV bool n3(T a, T b, T c) { return is_nan(a) | is_nan(b) | is_nan(c); }
template <class T> TF_DEV bool n4(T a, T b, T c, T d) {
  return is_nan(a) | is_nan(b) | is_nan(c) | is_nan(d);
}
template <class T> TF_DEV TF<T> fast_two_sum_c(T a, T b) {
  T s = add(a, b);
  if (is_finite(s)) return mk(s, sub(b, sub(s, a)));
  return special(s, n2(a, b));
}
template <class T> TF_DEV TF<T> two_sum_c(T a, T b) {
  T s = add(a, b);
  if (is_finite(s)) {
    T bp = sub(s, a);
    T ap = sub(s, bp);
    return mk(s, add(sub(a, ap), sub(b, bp)));
  }
  return special(s, n2(a, b));
}
template <class T> TF_DEV TF<T> renorm_c(TF<T> x) {
  TF<T> t = two_sum_c(x.v, x.e);
  return fast_two_sum_c(t.v, t.e);
}
template <class T> TF_DEV TF<T> t_add_c(TF<T> x, TF<T> y) {
  T s = add(x.v, y.v);
  if (!is_finite(s)) return special(s, n4(x.v, x.e, y.v, y.e));
  T bp = sub(s, x.v);
  T ap = sub(s, bp);
  T e = add(sub(x.v, ap), sub(y.v, bp));
  return mk(s, add(e, add(x.e, y.e)));
}
template <class T> TF_DEV TF<T> t_add_d_c(TF<T> x, T b) {
  T s = add(x.v, b);
  if (!is_finite(s)) return special(s, n3(x.v, x.e, b));
  T bp = sub(s, x.v);
  T ap = sub(s, bp);
  T e = add(sub(x.v, ap), sub(b, bp));
  return mk(s, add(e, x.e));
}
template <class T> TF_DEV TF<T> t_mul_c(TF<T> x, TF<T> y) {
  T v = mul(x.v, y.v);
  if (!is_finite(v)) return special(v, n4(x.v, x.e, y.v, y.e));
  T e = fmaop(x.v, y.v, -v);
  return mk(v, add(e, add(mul(x.v, y.e), mul(x.e, y.v))));
}
template <class T> TF_DEV TF<T> t_mul_d_c(TF<T> x, T b) {
  T v = mul(x.v, b);
  if (!is_finite(v)) return special(v, n3(x.v, x.e, b));
  T e = fmaop(x.v, b, -v);
  return mk(v, add(mul(x.e, b), e));
}

// ------------------------------------------------------ method parameters
// params.py:62-98
template <class T> struct P;
template <> struct P<double> {
  static constexpr double LO = -0x1.74385446d71c4p+9;
  static constexpr double HI = 0x1.62e42fefa39f0p+9;
  static constexpr int SPAN_SHIFT = 7;  // L + K = 2 + 5
  static constexpr double LN2_V = TF64_LN2_V, LN2_E = TF64_LN2_E;
  static constexpr double INVF_V = TF64_INVFACT_V, INVF_E = TF64_INVFACT_E;
  static constexpr int E_LO = TF64_E_LO, C_LO = TF64_C_LO, CM1_LO = TF64_CM1_LO;
  static constexpr int E_N = TF64_E_COUNT, C_N = TF64_C_COUNT, CM1_N = TF64_CM1_COUNT;
};
template <> struct P<float> {
  static constexpr float LO = -0x1.9d1da0p+6f;
  static constexpr float HI = 0x1.62e430p+6f;
  static constexpr int SPAN_SHIFT = 6;  // L + K = 1 + 5
  static constexpr float LN2_V = TF32_LN2_V, LN2_E = TF32_LN2_E;
  static constexpr float INVF_V = TF32_INVFACT_V, INVF_E = TF32_INVFACT_E;
  static constexpr int E_LO = TF32_E_LO, C_LO = TF32_C_LO, CM1_LO = TF32_CM1_LO;
  static constexpr int E_N = TF32_E_COUNT, C_N = TF32_C_COUNT, CM1_N = TF32_CM1_COUNT;
};

// Round-to-nearest-even "magic" constant: fma(x, 2^K, 1.5*2^52) leaves
// round(x * 2^K) in the low word for |x * 2^K| < 2^31.
constexpr double MAGIC = 6755399441055744.0;  // 1.5 * 2^52
constexpr int MAGIC_HI = 0x43380000;

}  // namespace tf
