// tf_eft.cu -- element-wise error-free transformations and twofold arithmetic
// over device arrays (libtwofold_b200.so).
//
// The reference's scalar substrate (pkg/src/twofold/eft.py:77-237 binary64,
// eft32.py:36-214 binary32): fast_two_sum, two_sum, two_diff, two_prod
// (fused or Dekker-Veltkamp residual), split, renorm_fast, renorm, t_add,
// t_add_d, t_mul, t_mul_d, t_div, t_sqrt -- same IEEE operation sequences,
// same non-finite policy (_special, eft.py:65-74), both residual backends
// ("fma" = one hardware FMA, "dv" = Veltkamp split + Dekker product, and
// fma_sim for the division / square-root remainders), bit for bit.
//
// These ops are pure streaming work (8..24 bytes in, 8..16 bytes out per
// element, a handful of flops): HBM-bound.  One persistent grid of
// SMs x 8 CTAs x 256 threads, 4 independent elements per thread per pass
// (coalesced, each warp-wide load/store one contiguous segment) to keep
// enough bytes in flight.
#include <cstdio>

#include "tf_common.cuh"
#include "tf_abi.h"

namespace tf {
namespace eft {

TF_DEV double div(double a, double b) { return __ddiv_rn(a, b); }
TF_DEV float div(float a, float b) { return __fdiv_rn(a, b); }
TF_DEV double sqrt_rn(double a) { return __dsqrt_rn(a); }
TF_DEV float sqrt_rn(float a) { return __fsqrt_rn(a); }

template <class T> struct SplitC;
template <> struct SplitC<double> {  // eft.py:107-112
  static constexpr double S = 134217729.0, BIG = 0x1p996, DOWN = 0x1p-28, UP = 0x1p28;
  static constexpr double TOP = 0x1p996, SHED = 0x1p970;
};
template <> struct SplitC<float> {   // eft32.py:63-67
  static constexpr float S = 4097.0f, BIG = 0x1p115f, DOWN = 0x1p-13f, UP = 0x1p13f;
  static constexpr float TOP = 0x1p115f, SHED = 0x1p103f;
};

// Veltkamp split (eft.py:115-128, eft32.py:70-82)
template <class T> TF_DEV TF<T> split(T x) {
  using C = SplitC<T>;
  if (fabs(x) > C::BIG) {
    T xs = mul(x, C::DOWN);
    T a = mul(C::S, xs);
    T b = sub(a, xs);
    T h = sub(a, b);
    if (fabs(h) == C::TOP) h = copysign(sub(C::TOP, C::SHED), h);
    return mk(mul(h, C::UP), mul(sub(xs, h), C::UP));
  }
  T a = mul(C::S, x);
  T b = sub(a, x);
  T h = sub(a, b);
  return mk(h, sub(x, h));
}

// exact product residual x*y - v (eft.py:254-264, eft32.py:180-190)
template <class T, bool DV> TF_DEV T prod_err(T x, T y, T v) {
  if constexpr (!DV) {
    return fmaop(x, y, -v);
  } else {
    TF<T> xs = split(x), ys = split(y);
    T e0 = sub(v, mul(xs.v, ys.v));
    T e1 = sub(e0, mul(xs.v, ys.e));
    T e2 = sub(e1, mul(xs.e, ys.v));
    return sub(mul(xs.e, ys.e), e2);
  }
}

// two_prod_fma / two_prod_dv (eft.py:131-149)
template <class T, bool DV> TF_DEV TF<T> two_prod(T x, T y) {
  T v = mul(x, y);
  if (!is_finite(v)) return special(v, n2(x, y));
  return mk(v, prod_err<T, DV>(x, y, v));
}

// fma_sim (eft.py:152-160): (z + p) + t with (p, t) = two_prod_dv(x, y)
template <class T> TF_DEV T fma_sim(T x, T y, T z) {
  TF<T> p = two_prod<T, true>(x, y);
  return add(add(z, p.v), p.e);
}

// a - q*b, exact (_rem_fma / _rem_dv, eft.py:267-272)
template <class T, bool DV> TF_DEV T rem(T q, T b, T a) {
  if constexpr (!DV) return fmaop(-q, b, a);
  else return fma_sim(-q, b, a);
}

// two_diff (eft.py:95-104)
template <class T> TF_DEV TF<T> two_diff(T a, T b) {
  T d = sub(a, b);
  if (!is_finite(d)) return special(d, n2(a, b));
  T bp = sub(d, a);
  T ap = sub(d, bp);
  T bs = add(b, bp);
  T as = sub(a, ap);
  return mk(d, sub(as, bs));
}

// t_mul / t_mul_d with either residual (eft.py:207-219)
template <class T, bool DV> TF_DEV TF<T> t_mul(TF<T> x, TF<T> y) {
  T v = mul(x.v, y.v);
  if (!is_finite(v)) return special(v, n4(x.v, x.e, y.v, y.e));
  T e = prod_err<T, DV>(x.v, y.v, v);
  return mk(v, add(e, add(mul(x.v, y.e), mul(x.e, y.v))));
}
template <class T, bool DV> TF_DEV TF<T> t_mul_d(TF<T> x, T b) {
  T v = mul(x.v, b);
  if (!is_finite(v)) return special(v, n3(x.v, x.e, b));
  T e = prod_err<T, DV>(x.v, b, v);
  return mk(v, add(mul(x.e, b), e));
}

// t_div (eft.py:221-226)
template <class T, bool DV> TF_DEV TF<T> t_div(TF<T> x, TF<T> y) {
  T q = div(x.v, y.v);
  if (!is_finite(q)) return special(q, n4(x.v, x.e, y.v, y.e));
  T r = rem<T, DV>(q, y.v, x.v);
  return mk(q, div(add(r, sub(x.e, mul(q, y.e))), y.v));
}

// t_sqrt (eft.py:228-235)
template <class T, bool DV> TF_DEV TF<T> t_sqrt(TF<T> x) {
  T q = sqrt_rn(x.v);
  if (!is_finite(q)) return special(q, n2(x.v, x.e));
  if (x.v == T(0)) return mk(q, T(0));
  T r = rem<T, DV>(q, q, x.v);
  return mk(q, div(add(r, x.e), add(q, q)));
}

// op codes: TF_OP_* of include/twofold_b200.h
enum Op {
  FAST_TWO_SUM = 0, TWO_SUM = 1, TWO_DIFF = 2, TWO_PROD = 3, SPLIT = 4, RENORM_FAST = 5,
  RENORM = 6, T_ADD = 7, T_ADD_D = 8, T_MUL = 9, T_MUL_D = 10, T_DIV = 11, T_SQRT = 12,
  OP_COUNT = 13
};
__host__ __device__ constexpr bool reads_a1(int op) {
  return op >= RENORM_FAST;
}
__host__ __device__ constexpr bool reads_b0(int op) {
  return op <= TWO_PROD || op == T_ADD || op == T_ADD_D || op == T_MUL || op == T_MUL_D ||
         op == T_DIV;
}
__host__ __device__ constexpr bool reads_b1(int op) {
  return op == T_ADD || op == T_MUL || op == T_DIV;
}
__host__ __device__ constexpr bool uses_backend(int op) {
  return op == TWO_PROD || op == T_MUL || op == T_MUL_D || op == T_DIV || op == T_SQRT;
}

template <class T, int OP, bool DV> TF_DEV TF<T> apply(T a0, T a1, T b0, T b1) {
  if constexpr (OP == FAST_TWO_SUM) return fast_two_sum_c(a0, b0);
  else if constexpr (OP == TWO_SUM) return two_sum_c(a0, b0);
  else if constexpr (OP == TWO_DIFF) return two_diff(a0, b0);
  else if constexpr (OP == TWO_PROD) return two_prod<T, DV>(a0, b0);
  else if constexpr (OP == SPLIT) return split(a0);
  else if constexpr (OP == RENORM_FAST) return fast_two_sum_c(a0, a1);
  else if constexpr (OP == RENORM) return renorm_c(mk(a0, a1));
  else if constexpr (OP == T_ADD) return t_add_c(mk(a0, a1), mk(b0, b1));
  else if constexpr (OP == T_ADD_D) return t_add_d_c(mk(a0, a1), b0);
  else if constexpr (OP == T_MUL) return t_mul<T, DV>(mk(a0, a1), mk(b0, b1));
  else if constexpr (OP == T_MUL_D) return t_mul_d<T, DV>(mk(a0, a1), b0);
  else if constexpr (OP == T_DIV) return t_div<T, DV>(mk(a0, a1), mk(b0, b1));
  else return t_sqrt<T, DV>(mk(a0, a1));
}

constexpr int ILP = 4;

template <class T, int OP, bool DV>
__global__ void __launch_bounds__(256) k_eft(const T* __restrict__ a0, const T* __restrict__ a1,
                                             const T* __restrict__ b0, const T* __restrict__ b1,
                                             T* __restrict__ z0, T* __restrict__ z1, uint64_t n) {
  const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += ILP * gs) {
    T x0[ILP], x1[ILP], y0[ILP], y1[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      uint64_t i = i0 + k * gs;
      bool v = i < n;
      x0[k] = v ? __ldcs(a0 + i) : T(0);
      x1[k] = (reads_a1(OP) && v) ? __ldcs(a1 + i) : T(0);
      y0[k] = (reads_b0(OP) && v) ? __ldcs(b0 + i) : T(0);
      y1[k] = (reads_b1(OP) && v) ? __ldcs(b1 + i) : T(0);
    }
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      uint64_t i = i0 + k * gs;
      if (i < n) {
        TF<T> r = apply<T, OP, DV>(x0[k], x1[k], y0[k], y1[k]);
        __stcs(z0 + i, r.v);
        __stcs(z1 + i, r.e);
      }
    }
  }
}

}  // namespace eft
}  // namespace tf

namespace {
using tfabi::cuda_check;
using tfabi::device_sms;
using tfabi::fail;

template <class T, int OP, bool DV>
int launch_eft(const T* a0, const T* a1, const T* b0, const T* b1, T* z0, T* z1, int64_t n,
               cudaStream_t s) {
  int64_t grid = (int64_t)device_sms() * 8;
  int64_t need = (n + 256 * tf::eft::ILP - 1) / (256 * tf::eft::ILP);
  if (need < grid) grid = need > 0 ? need : 1;
  tf::eft::k_eft<T, OP, DV><<<(unsigned)grid, 256, 0, s>>>(a0, a1, b0, b1, z0, z1, (uint64_t)n);
  return cuda_check("k_eft launch");
}

template <class T, int OP>
int dispatch_dv(bool dv, const T* a0, const T* a1, const T* b0, const T* b1, T* z0, T* z1,
                int64_t n, cudaStream_t s) {
  if constexpr (tf::eft::uses_backend(OP)) {
    if (dv) return launch_eft<T, OP, true>(a0, a1, b0, b1, z0, z1, n, s);
  }
  return launch_eft<T, OP, false>(a0, a1, b0, b1, z0, z1, n, s);
}

template <class T>
int dispatch(int op, bool dv, const T* a0, const T* a1, const T* b0, const T* b1, T* z0, T* z1,
             int64_t n, cudaStream_t s) {
  using namespace tf::eft;
  switch (op) {
    case FAST_TWO_SUM: return dispatch_dv<T, FAST_TWO_SUM>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case TWO_SUM: return dispatch_dv<T, TWO_SUM>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case TWO_DIFF: return dispatch_dv<T, TWO_DIFF>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case TWO_PROD: return dispatch_dv<T, TWO_PROD>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case SPLIT: return dispatch_dv<T, SPLIT>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case RENORM_FAST: return dispatch_dv<T, RENORM_FAST>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case RENORM: return dispatch_dv<T, RENORM>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case T_ADD: return dispatch_dv<T, T_ADD>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case T_ADD_D: return dispatch_dv<T, T_ADD_D>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case T_MUL: return dispatch_dv<T, T_MUL>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case T_MUL_D: return dispatch_dv<T, T_MUL_D>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case T_DIV: return dispatch_dv<T, T_DIV>(dv, a0, a1, b0, b1, z0, z1, n, s);
    case T_SQRT: return dispatch_dv<T, T_SQRT>(dv, a0, a1, b0, b1, z0, z1, n, s);
  }
  return fail(TF_ERR_ARG, "unknown op code%s");
}
}  // namespace

extern "C" {

TF_API int tf_eft(int op, int width, int backend, const void* a0, const void* a1, const void* b0,
                  const void* b1, void* z0, void* z1, int64_t n, void* stream) {
  using namespace tf::eft;
  if (op < 0 || op >= OP_COUNT) return fail(TF_ERR_ARG, "unknown op code%s");
  if (backend != 0 && backend != 1) return fail(TF_ERR_ARG, "unknown backend (0 fma, 1 dv)%s");
  if (width != 32 && width != 64) return fail(TF_ERR_ARG, "unsupported width (expected 32 or 64)%s");
  if (n < 0) return fail(TF_ERR_ARG, "negative element count%s");
  if (n == 0) return TF_OK;
  if (!a0 || !z0 || !z1 || (reads_a1(op) && !a1) || (reads_b0(op) && !b0) ||
      (reads_b1(op) && !b1))
    return fail(TF_ERR_ARG, "null pointer%s");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (width == 64)
    return dispatch<double>(op, backend == 1, (const double*)a0, (const double*)a1,
                            (const double*)b0, (const double*)b1, (double*)z0, (double*)z1, n, s);
  return dispatch<float>(op, backend == 1, (const float*)a0, (const float*)a1, (const float*)b0,
                         (const float*)b1, (float*)z0, (float*)z1, n, s);
}

}  // extern "C"
