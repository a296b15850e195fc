// max relative error of rcp.approx.ftz.f64 (MUFU.RCP64H path) on random inputs
#include <cstdio>
#include <cstdint>
__global__ void k(double* worst, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
  h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
  double x = 1.0 + (double)(h >> 11) * 0x1p-53;   // [1, 2)
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fabs(fma(-x, r, 1.0));               // |1 - x r| = relative error
  unsigned long long* w = (unsigned long long*)worst;
  atomicMax(w, (unsigned long long)__double_as_longlong(e));
}
int main() {
  double* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  int n = 1 << 26;
  k<<<n / 256, 256>>>(d, n);
  double h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("rcp.approx.ftz.f64 worst relative error %.3e = 2^%.2f\n", h, log2(h));
  return 0;
}
