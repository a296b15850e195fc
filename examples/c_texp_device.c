/* C client evaluating texp / tlog1p on device arrays through the C ABI:
 *
 *   gcc -std=c99 -I include -I /usr/local/cuda/include examples/c_texp_device.c \
 *       -L paper_1502_05216_b200/lib -ltwofold_b200 -L /usr/local/cuda/lib64 -lcudart \
 *       -o /tmp/tf_texp && LD_LIBRARY_PATH=paper_1502_05216_b200/lib /tmp/tf_texp
 *
 * Prints z0, z1 of texp((1, 0)) and tlog1p((1, 0)); z0 must be the correctly
 * rounded e and ln 2. */
#include <stdio.h>
#include <cuda_runtime.h>
#include "twofold_b200.h"

int main(void) {
  const int n = 4;
  double hx0[4] = {1.0, 0.5, -2.0, 10.0}, hx1[4] = {0.0, 0.0, 0.0, 0.0};
  double hz0[4], hz1[4];
  double *x0, *x1, *z0, *z1;
  if (tf_init(0) != TF_OK) {
    printf("tf_init failed: %s\n", tf_last_error());
    return 1;
  }
  cudaMalloc((void**)&x0, n * sizeof(double));
  cudaMalloc((void**)&x1, n * sizeof(double));
  cudaMalloc((void**)&z0, n * sizeof(double));
  cudaMalloc((void**)&z1, n * sizeof(double));
  cudaMemcpy(x0, hx0, sizeof hx0, cudaMemcpyHostToDevice);
  cudaMemcpy(x1, hx1, sizeof hx1, cudaMemcpyHostToDevice);
  if (tf_texp_f64(x0, x1, z0, z1, n, NULL) != TF_OK) {
    printf("tf_texp_f64: %s\n", tf_last_error());
    return 1;
  }
  cudaMemcpy(hz0, z0, sizeof hz0, cudaMemcpyDeviceToHost);
  cudaMemcpy(hz1, z1, sizeof hz1, cudaMemcpyDeviceToHost);
  printf("texp(1) = %a + %a\n", hz0[0], hz1[0]);
  if (tf_eval(TF_FN_TLOG1P, 64, x0, x1, z0, z1, n, NULL, 0) != TF_OK) {
    printf("tf_eval: %s\n", tf_last_error());
    return 1;
  }
  cudaMemcpy(hz0, z0, sizeof hz0, cudaMemcpyDeviceToHost);
  cudaMemcpy(hz1, z1, sizeof hz1, cudaMemcpyDeviceToHost);
  printf("tlog1p(1) = %a + %a\n", hz0[0], hz1[0]);
  cudaFree(x0);
  cudaFree(x1);
  cudaFree(z0);
  cudaFree(z1);
  return 0;
}
