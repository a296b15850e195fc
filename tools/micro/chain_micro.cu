// FP32 pipe utilisation against ILP: CH dependent FADD2 chains per thread, one
// 1024-thread CTA per SM (the f32 log kernels' shape), optionally with scalar
// FSETP+FSEL (ALU) or IMAD (fmaheavy) work interleaved.  Prints lane-ops/s.
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
  u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
template <int CH, int MIX> __global__ void __launch_bounds__(1024, 1) k(float* out, int iters) {
  u64 p[CH];
  unsigned q[CH];
  float f[CH];
  for (int i = 0; i < CH; ++i) { p[i] = ((u64)__float_as_uint(threadIdx.x * 1e-9f + i) << 32) | 0x3f800000u; q[i] = threadIdx.x + i; f[i] = i; }
  const u64 m = 0x3380000033800000ull;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      p[i] = fadd2(p[i], m);
      p[i] = fadd2(p[i], m);
      if (MIX == 1) {  // scalar compare + select per two packed ops
        float lo = __uint_as_float((unsigned)p[i]);
        f[i] = lo > f[i] ? f[i] + 0.f : lo;
      }
      if (MIX == 2) q[i] = q[i] * 3u + (unsigned)p[i];   // IMAD
      if (MIX == 3) {  // the same compare + select on the bit patterns (ISETP + SEL)
        unsigned lo = (unsigned)p[i], fb = __float_as_uint(f[i]);
        unsigned r;
        asm("{ .reg .pred q; setp.gt.s32 q, %1, %2; selp.b32 %0, %2, %1, q; }" : "=r"(r) : "r"(lo), "r"(fb));
        f[i] = __uint_as_float(r);
      }
      if (MIX == 4) q[i] = (q[i] ^ (unsigned)p[i]) + 3u;  // LOP3 + IADD (ALU)
    }
  }
  float s = 0;
  for (int i = 0; i < CH; ++i) s += __uint_as_float((unsigned)p[i]) + f[i] + q[i];
  if (s == -1.f) out[0] = s;
}
template <int CH, int MIX> void run(const char* name, float* d, int sms) {
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<CH, MIX><<<sms, 1024>>>(d, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("%-12s CH=%d %7.2f T lane-ops/s\n", name, CH,
                    (double)sms * 1024 * iters * CH * 4 / (ms * 1e-3) / 1e12);
  }
}
int main() {
  float* d; cudaMalloc(&d, 4); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1, 0>("FADD2", d, sms); run<2, 0>("FADD2", d, sms); run<4, 0>("FADD2", d, sms);
  run<1, 1>("+FSETP/FSEL", d, sms); run<2, 1>("+FSETP/FSEL", d, sms); run<4, 1>("+FSETP/FSEL", d, sms);
  run<1, 2>("+IMAD", d, sms); run<2, 2>("+IMAD", d, sms); run<4, 2>("+IMAD", d, sms);
  run<2, 3>("+ISETP/SEL", d, sms); run<4, 3>("+ISETP/SEL", d, sms);
  run<2, 4>("+LOP3/IADD", d, sms); run<4, 4>("+LOP3/IADD", d, sms);
  return 0;
}
