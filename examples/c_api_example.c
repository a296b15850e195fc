/* Minimal C client of libtwofold_b200.so (C99, no CUDA headers needed):
 *
 *   gcc -std=c99 -I include examples/c_api_example.c \
 *       -L paper_1502_05216_b200/lib -ltwofold_b200 -o /tmp/tf_example
 *   LD_LIBRARY_PATH=paper_1502_05216_b200/lib /tmp/tf_example
 *
 * It exercises the error conventions of the ABI (status codes plus
 * tf_last_error(), never an abort) and, when a device is present, evaluates
 * texp and tlog1p over plain host arrays through tf_eval_host -- the client
 * needs no CUDA code at all.  Device-pointer use: examples/c_texp_device.c. */
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include "twofold_b200.h"

int main(void) {
  printf("twofold_b200 ABI version %d\n", tf_version());
  /* argument errors are reported, never thrown */
  int rc = tf_eval(TF_FN_TEXP, 64, NULL, NULL, NULL, NULL, -1, NULL, 0);
  printf("negative count -> %d (%s)\n", rc, tf_last_error());
  rc = tf_eval(99, 64, NULL, NULL, NULL, NULL, 4, NULL, 0);
  printf("unknown function -> %d (%s)\n", rc, tf_last_error());
  rc = tf_eft(TF_OP_T_ADD, 64, 0, NULL, NULL, NULL, NULL, NULL, NULL, 0, NULL);
  printf("empty t_add -> %d\n", rc);
  rc = tf_init(0);
  if (rc != TF_OK) {
    printf("no usable CUDA device: %d (%s)\n", rc, tf_last_error());
    return 0;
  }
  printf("device 0 initialised\n");
  /* host arrays (pageable here; pinned memory streams at full PCIe speed) */
  double x0[4] = {1.0, -2.5, 0.0, 700.0}, x1[4] = {0.0, 1e-17, 0.0, 0.0}, z0[4], z1[4];
  rc = tf_eval_host(TF_FN_TEXP, 64, x0, x1, z0, z1, 4, 0, NULL, 0);
  if (rc != TF_OK) {
    printf("tf_eval_host failed: %d (%s)\n", rc, tf_last_error());
    return 1;
  }
  printf("host texp(1) = %a + %a\n", z0[0], z1[0]);
  double y0[1] = {1.0}, y1[1] = {0.0};
  rc = tf_eval_host(TF_FN_TLOG1P, 64, y0, y1, z0, z1, 1, 0, NULL, 0);
  if (rc != TF_OK) {
    printf("tf_eval_host failed: %d (%s)\n", rc, tf_last_error());
    return 1;
  }
  printf("host tlog1p(1) = %a + %a\n", z0[0], z1[0]);
  return 0;
}
