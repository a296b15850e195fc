// throughput of FFMA2 vs FFMA
#include <cstdio>
template <int P> __global__ void k(float* out, int iters) {
  float c[16];
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
    if (P) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        unsigned long long x, r; float2 v = make_float2(c[i], c[i+1]);
        x = *reinterpret_cast<unsigned long long*>(&v);
        asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(r) : "l"(x));
        float2 w = *reinterpret_cast<float2*>(&r); c[i] = w.x; c[i+1] = w.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) c[i] = __fmaf_rn(c[i], c[i], c[i]);
    }
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += c[i];
  if (s == -1.f) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int P = 0; P < 2; ++P) for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    if (P) k<1><<<sms*8, 256>>>(d, 4096); else k<0><<<sms*8, 256>>>(d, 4096);
    cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s %.2f T fma/s\n", P ? "FFMA2" : "FFMA", (double)sms*8*256*4096*16/(ms*1e-3)/1e12);
  }
}
