// FP64 pipe utilisation against ILP: CH dependent DADD chains per thread in
// one CTA of B threads per SM (the binary64 kernels: 512 threads x 4 lanes).
#include <cstdio>
template <int CH> __global__ void k(double* out, int iters) {
  double p[CH];
  for (int i = 0; i < CH; ++i) p[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) p[i] = __dadd_rn(p[i], 1e-17);
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) s += p[i];
  if (s == -1.0) out[0] = s;
}
template <int CH> void run(double* d, int sms, int B) {
  const int iters = 8192;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<CH><<<sms, B>>>(d, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("DADD B=%4d CH=%d  %6.2f T op/s\n", B, CH, (double)sms * B * iters * CH / (ms * 1e-3) / 1e12);
  }
}
int main() {
  double* d; cudaMalloc(&d, 8); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int B : {512, 1024}) { run<1>(d, sms, B); run<2>(d, sms, B); run<4>(d, sms, B); run<8>(d, sms, B); }
  return 0;
}
