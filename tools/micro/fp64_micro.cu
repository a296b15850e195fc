// FP64 pipe microbenchmarks on B200: throughput per opcode and dependent-chain latency.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP, int CH>
__global__ void k(double* out, int iters, double a, double b) {
  double c[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (OP == 0) c[i] = __fma_rn(c[i], a, b);
      if (OP == 1) c[i] = __dadd_rn(c[i], b);
      if (OP == 2) c[i] = __dmul_rn(c[i], a);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i];
  if (s == -1.2345) out[0] = s;
}
template <int OP, int CH>
void run(const char* name, int blocks, int threads) {
  double* d; cudaMalloc(&d, 8);
  int iters = 4096;
  k<OP, CH><<<blocks, threads>>>(d, iters, 0.9999999, 1e-9);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP, CH><<<blocks, threads>>>(d, iters, 0.9999999, 1e-9);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * iters * CH;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  // per-SMSP cycles per dependent op = (time * clk) / (ops per chain)
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-8s ch=%d blocks=%d thr=%d : %.2f Top/s   cycles/iter-per-chain %.2f\n", name, CH, blocks, threads,
         ops / (ms * 1e-3) / 1e12, cyc / iters);
  cudaFree(d);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, 8>("dfma", sms * 8, 256);
  run<1, 8>("dadd", sms * 8, 256);
  run<2, 8>("dmul", sms * 8, 256);
  // latency: one warp per SMSP, one chain
  run<0, 1>("dfma-lat", sms, 128);
  run<1, 1>("dadd-lat", sms, 128);
  run<2, 1>("dmul-lat", sms, 128);
  // occupancy sweep for 2 chains per thread (like VW=2)
  for (int w : {4, 6, 8, 12, 16}) {
    run<1, 2>("dadd", sms, 128 * w);
  }
  return 0;
}
