// Check packed f32x2 ops against scalar IEEE ops bit for bit on random inputs.
#include <cstdio>
#include <cstdint>
__device__ uint32_t h32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__global__ void k(unsigned long long* bad, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float a0 = __uint_as_float((h32(i * 6 + 0) & 0x3fffffff) | 0x38000000) * ((i & 1) ? -1.f : 1.f);
  float a1 = __uint_as_float((h32(i * 6 + 1) & 0x3fffffff) | 0x38000000);
  float b0 = __uint_as_float((h32(i * 6 + 2) & 0x3fffffff) | 0x38000000);
  float b1 = __uint_as_float((h32(i * 6 + 3) & 0x3fffffff) | 0x38000000) * ((i & 2) ? -1.f : 1.f);
  float c0 = -__fmul_rn(a0, b0), c1 = -__fmul_rn(a1, b1);
  unsigned long long A, B, C, R, S, M, D;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(c0), "f"(c1));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(R) : "l"(A), "l"(B), "l"(C));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(S) : "l"(A), "l"(B));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(M) : "l"(A), "l"(B));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
  float r0, r1, s0, s1, m0, m1, d0, d1;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r0), "=f"(r1) : "l"(R));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(s0), "=f"(s1) : "l"(S));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(m0), "=f"(m1) : "l"(M));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(D));
  if (__float_as_uint(r0) != __float_as_uint(__fmaf_rn(a0, b0, c0))) atomicAdd(&bad[0], 1ull);
  if (__float_as_uint(r1) != __float_as_uint(__fmaf_rn(a1, b1, c1))) atomicAdd(&bad[0], 1ull);
  if (__float_as_uint(s0) != __float_as_uint(__fadd_rn(a0, b0)) || __float_as_uint(s1) != __float_as_uint(__fadd_rn(a1, b1))) atomicAdd(&bad[1], 1ull);
  if (__float_as_uint(m0) != __float_as_uint(__fmul_rn(a0, b0)) || __float_as_uint(m1) != __float_as_uint(__fmul_rn(a1, b1))) atomicAdd(&bad[2], 1ull);
  if (__float_as_uint(d0) != __float_as_uint(__fsub_rn(a0, b0)) || __float_as_uint(d1) != __float_as_uint(__fsub_rn(a1, b1))) atomicAdd(&bad[3], 1ull);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 32); cudaMemset(d, 0, 32);
  int n = 1 << 26;
  k<<<n / 256, 256>>>(d, n);
  unsigned long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("mismatches of %d: fma %llu add %llu mul %llu sub %llu\n", n, h[0], h[1], h[2], h[3]);
}
