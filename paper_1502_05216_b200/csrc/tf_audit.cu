// tf_audit.cu -- GPU accuracy audit and benchmark checksum (libtwofold_b200.so).
//
// The reference's audit (pkg/src/twofold/audit.py:207-286) measures, per
// sample, the relative error |(z0 + z1) - ref| / |ref| of a function result
// against a high-precision etalon, after excluding non-finite results and
// results below the error floor (audit.py:248-249), arguments outside the
// etalon's domain (250-256) and zero references (absolute fallback, 258-260).
// Here one thread handles one sample: the triple-double etalon
// (tf_etalon.cuh) for etalon "oracle", or the binary64 library at x0 + x1
// for etalon "lib" (binary32 only; oracle.py:158-167), and writes the error
// and an exclusion state; paper_1502_05216_b200/audit.py reduces them.
//
// run_bench's checksum (audit.py:344-349) is the XOR of bits64(value) over
// all results; k_xor64 computes it on the device from the result array.
#include <cstdio>

#include "tf_etalon.cuh"
#include "tf_abi.h"

namespace tf {

// exclusion states of one audit sample
enum : unsigned char { ST_INCLUDED = 0, ST_FLOOR = 1, ST_DOMAIN = 2, ST_ABSOLUTE = 3 };

template <class T>
__global__ void __launch_bounds__(128) k_audit(int fam, int kind, const T* __restrict__ x0,
                                               const T* __restrict__ x1, const T* __restrict__ z0,
                                               const T* __restrict__ z1, uint64_t n, double floor,
                                               double* __restrict__ err,
                                               unsigned char* __restrict__ state) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    double v = (double)z0[i], w = (double)z1[i];
    double a = (double)x0[i], b = (double)x1[i];
    unsigned char st = ST_INCLUDED;
    double e = 0.0;
    if (!(fabs(v) <= 1.79769313486231570e308) || fabs(v) < floor) {
      st = ST_FLOOR;
    } else if (kind == 1) {
      // binary64 library etalon at the binary64 sum (oracle.py:158-167)
      double s = add(a, b);
      double ref = fam == et::EXP ? exp(s) : fam == et::EXPM1 ? expm1(s)
                   : fam == et::LOG ? log(s) : log1p(s);
      double d = add(sub(v, ref), w);
      if (ref == 0.0) st = ST_ABSOLUTE;
      else e = fabs(d / ref);
    } else {
      et::TD m;
      int k;
      if (!et::etalon(fam, a, b, m, k)) {
        st = ST_DOMAIN;
      } else if (m.a == 0.0) {
        st = ST_ABSOLUTE;
      } else {
        // (z0 + z1) 2^-k - m, exact scalings (the results are >= the floor)
        et::TD d = et::add_d(et::add_d(et::neg(m), ldexp(v, -k)), ldexp(w, -k));
        e = fabs(d.a) / fabs(m.a);
      }
    }
    err[i] = e;
    state[i] = st;
  }
}

// the etalon itself, m = (a, b, c) * 2^k, SoA
__global__ void __launch_bounds__(128) k_etalon(int fam, const double* __restrict__ x0,
                                                const double* __restrict__ x1, uint64_t n,
                                                double* __restrict__ m, int* __restrict__ kout) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    et::TD r;
    int k;
    bool ok = et::etalon(fam, x0[i], x1[i], r, k);
    const double q = __longlong_as_double(0x7ff8000000000000ull);
    m[i] = ok ? r.a : q;
    m[n + i] = ok ? r.b : q;
    m[2 * n + i] = ok ? r.c : q;
    kout[i] = ok ? k : 0;
  }
}

// XOR of bits64((double) z[i]) over all i
template <class T>
__global__ void __launch_bounds__(256) k_xor64(const T* __restrict__ z, uint64_t n,
                                               unsigned long long* out) {
  unsigned long long h = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    h ^= (unsigned long long)__double_as_longlong((double)z[i]);
  for (int o = 16; o > 0; o >>= 1) h ^= __shfl_down_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0 && h) atomicXor(out, h);
}

}  // namespace tf

namespace {
using tfabi::cuda_check;
using tfabi::device_sms;
using tfabi::fail;

unsigned grid_for(int64_t n, int block, int per_sm) {
  int64_t g = (int64_t)device_sms() * per_sm;
  int64_t need = (n + block - 1) / block;
  return (unsigned)(need < g ? (need > 0 ? need : 1) : g);
}
}  // namespace

extern "C" {

TF_API int tf_audit_errors(int family, int width, int etalon_kind, const void* x0, const void* x1,
                           const void* z0, const void* z1, int64_t n, double* err,
                           unsigned char* state, void* stream) {
  if (n < 0) return fail(TF_ERR_ARG, "negative element count%s");
  if (family < 0 || family > 3) return fail(TF_ERR_ARG, "unknown function family%s");
  if (etalon_kind != 0 && etalon_kind != 1) return fail(TF_ERR_ARG, "unknown etalon%s");
  if (etalon_kind == 1 && width != 32)
    return fail(TF_ERR_ARG, "library etalon is only meaningful for binary32%s");
  if (n == 0) return TF_OK;
  if (!x0 || !x1 || !z0 || !z1 || !err || !state) return fail(TF_ERR_ARG, "null pointer%s");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned g = grid_for(n, 128, 8);
  if (width == 64) {
    tf::k_audit<double><<<g, 128, 0, s>>>(family, etalon_kind, (const double*)x0,
                                          (const double*)x1, (const double*)z0,
                                          (const double*)z1, (uint64_t)n, 0x1p-969, err, state);
  } else if (width == 32) {
    tf::k_audit<float><<<g, 128, 0, s>>>(family, etalon_kind, (const float*)x0, (const float*)x1,
                                         (const float*)z0, (const float*)z1, (uint64_t)n,
                                         0x1p-102, err, state);
  } else {
    return fail(TF_ERR_ARG, "unsupported width (expected 32 or 64)%s");
  }
  return cuda_check("k_audit launch");
}

TF_API int tf_etalon(int family, const double* x0, const double* x1, int64_t n, double* m,
                     int* k, void* stream) {
  if (n < 0) return fail(TF_ERR_ARG, "negative element count%s");
  if (family < 0 || family > 3) return fail(TF_ERR_ARG, "unknown function family%s");
  if (n == 0) return TF_OK;
  if (!x0 || !x1 || !m || !k) return fail(TF_ERR_ARG, "null pointer%s");
  tf::k_etalon<<<grid_for(n, 128, 8), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      family, x0, x1, (uint64_t)n, m, k);
  return cuda_check("k_etalon launch");
}

TF_API int tf_checksum(int width, const void* z0, int64_t n, unsigned long long* out,
                       void* stream) {
  if (n < 0) return fail(TF_ERR_ARG, "negative element count%s");
  if (!out) return fail(TF_ERR_ARG, "null pointer%s");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(out, 0, sizeof(unsigned long long), s) != cudaSuccess)
    return cuda_check("checksum reset");
  if (n == 0) return TF_OK;
  if (!z0) return fail(TF_ERR_ARG, "null pointer%s");
  unsigned g = grid_for(n, 256, 4);
  if (width == 64)
    tf::k_xor64<double><<<g, 256, 0, s>>>((const double*)z0, (uint64_t)n, out);
  else if (width == 32)
    tf::k_xor64<float><<<g, 256, 0, s>>>((const float*)z0, (uint64_t)n, out);
  else
    return fail(TF_ERR_ARG, "unsupported width (expected 32 or 64)%s");
  return cuda_check("k_xor64 launch");
}

}  // extern "C"
