/* Minimal C client of libtwofold_b200.so (C99, no CUDA headers needed):
 *
 *   gcc -std=c99 -I include examples/c_api_example.c \
 *       -L paper_1502_05216_b200/lib -ltwofold_b200 -o /tmp/tf_example
 *   LD_LIBRARY_PATH=paper_1502_05216_b200/lib /tmp/tf_example
 *
 * It exercises the error conventions of the ABI (status codes plus
 * tf_last_error(), never an abort) and initialises device 0 when one is
 * present.  Evaluating arrays needs device pointers from the caller's own CUDA
 * code: see INTEGRATION.md, "From C/C++". */
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
  return 0;
}
