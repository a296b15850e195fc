/*
 * twofold_b200.h -- C ABI of libtwofold_b200.so (B200 / sm_100a).
 *
 * Batch twofold elementary functions over structure-of-arrays operands:
 * element i is the twofold x0[i] + x1[i]; the result is z0[i] + z1[i] with
 * z0[i] the correctly rounded value of the standard function at x0[i] and
 * z1[i] the error part of the reference algorithm.
 *
 * Each entry point replaces, for a whole array, the per-element reference
 * call of the Python package (/root/reference/pkg/src/twofold):
 *   tf_texp_f64   <- ExpLog(64).texp(x)    explog.py:115-125
 *   tf_texpm1_f64 <- ExpLog(64).texpm1(x)  explog.py:149-160
 *   tf_tlog_f64   <- ExpLog(64).tlog(y)    explog.py:244-249
 *   tf_tlog1p_f64 <- ExpLog(64).tlog1p(y)  explog.py:314-317
 *   tf_*_f32      <- the same methods of ExpLog(32) (binary32 lane)
 * (api(width) / get_function(name, width), explog.py:333-349, resolve to them).
 * The paper's scalar C form z0 = texp(x0, x1, &z1)
 * is the n == 1 case.
 *
 * Conventions
 *   - x0, x1, z0, z1 are DEVICE pointers of the current device (tf_init),
 *     same element type; z may alias x only element-for-element (in place).
 *   - 16-byte aligned pointers take the vectorised path; any element-aligned
 *     pointer is accepted.
 *   - stream is a cudaStream_t (NULL = legacy default stream); every call is
 *     asynchronous and thread-safe.
 *   - return 0 on success, negative TF_ERR_* on error (message in
 *     tf_last_error(), thread-local).  Numerics never fail: non-finite inputs
 *     produce the reference's IEEE special results.
 */
#ifndef TWOFOLD_B200_H
#define TWOFOLD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define TF_API __declspec(dllexport)
#else
#define TF_API __attribute__((visibility("default")))
#endif

#define TF_ABI_VERSION 1

/* status codes */
#define TF_OK 0
#define TF_ERR_ARG (-1)  /* invalid argument (the reference raises ValueError) */
#define TF_ERR_CUDA (-2) /* CUDA runtime / launch error */

/* function codes for tf_eval: the four TWOFOLD_ARG hot-path functions first,
 * then the other sixteen names of FUNCTION_NAMES (explog.py:44-53).  Codes
 * marked (dotted) take the plain argument x0 only; x1 may be NULL. */
#define TF_FN_TEXP 0
#define TF_FN_TEXPM1 1
#define TF_FN_TLOG 2
#define TF_FN_TLOG1P 3
#define TF_FN_PEXP0 4    /* (dotted) */
#define TF_FN_TEXP0 5    /* (dotted) */
#define TF_FN_TEXPP 6
#define TF_FN_PEXP 7
#define TF_FN_PEXPM10 8  /* (dotted) */
#define TF_FN_TEXPM10 9  /* (dotted) */
#define TF_FN_TEXPM1P 10
#define TF_FN_PEXPM1 11
#define TF_FN_PLOG0 12   /* (dotted) */
#define TF_FN_TLOG0 13   /* (dotted) */
#define TF_FN_TLOGP 14
#define TF_FN_PLOG 15
#define TF_FN_PLOG1P0 16 /* (dotted) */
#define TF_FN_TLOG1P0 17 /* (dotted) */
#define TF_FN_TLOG1PP 18
#define TF_FN_PLOG1P 19
#define TF_FN_COUNT 20

/* tf_eval flags */
#define TF_FLAG_FORCE_EXACT 1 /* route every element through the exact path (testing) */
#define TF_FLAG_COUNT_EXACT 2 /* count exact-path elements (tf_exact_count) */
#define TF_FLAG_MARK_EXACT 4  /* diagnostics: write (NaN, -12345) instead of evaluating them */

/* synthetic distributions for tf_generate (BASELINE.json configs; workloads.py) */
#define TF_DIST_EXP64 0
#define TF_DIST_POW10 1
#define TF_DIST_POW10C 2
#define TF_DIST_LOG64 3
#define TF_DIST_EXP32 4
#define TF_DIST_LOG32 5
#define TF_DIST_EXP64S 6
#define TF_DIST_LOGU64S 7
#define TF_DIST_COUNT 8

TF_API int tf_version(void);
TF_API const char* tf_last_error(void);

/* Select the device (device < 0: keep the current one) and upload constants. */
TF_API int tf_init(int device);

TF_API int tf_texp_f64(const double* x0, const double* x1, double* z0, double* z1, int64_t n, void* stream);
TF_API int tf_texpm1_f64(const double* x0, const double* x1, double* z0, double* z1, int64_t n, void* stream);
TF_API int tf_tlog_f64(const double* x0, const double* x1, double* z0, double* z1, int64_t n, void* stream);
TF_API int tf_tlog1p_f64(const double* x0, const double* x1, double* z0, double* z1, int64_t n, void* stream);
TF_API int tf_texp_f32(const float* x0, const float* x1, float* z0, float* z1, int64_t n, void* stream);
TF_API int tf_texpm1_f32(const float* x0, const float* x1, float* z0, float* z1, int64_t n, void* stream);
TF_API int tf_tlog_f32(const float* x0, const float* x1, float* z0, float* z1, int64_t n, void* stream);
TF_API int tf_tlog1p_f32(const float* x0, const float* x1, float* z0, float* z1, int64_t n, void* stream);

/* Generic dispatcher: fn = TF_FN_*, width = 32 or 64, flags = TF_FLAG_*. */
TF_API int tf_eval(int fn, int width, const void* x0, const void* x1, void* z0, void* z1,
                   int64_t n, void* stream, int flags);

/* Host-buffer evaluation (the reference's own calling convention: api(width)
 * methods on host numpy arrays, explog.py:333-349).  x0, x1, z0, z1 are HOST
 * arrays -- pinned (cudaHostAlloc / torch pin_memory) for full PCIe speed,
 * pageable memory works at the driver's staged rate.  The n elements stream
 * through a three-stage chunk pipeline on the current device (H2D on two copy
 * streams, the kernel, D2H on two copy streams, over a ring of device buffers)
 * that starts after the work queued on `stream`; the call returns when z0, z1
 * hold the results.  chunk = elements per pipeline chunk, 0 = default (2^20).
 * Small calls (n <= 1024, chunk == 0) use a mapped pinned buffer instead; up to
 * 32 elements travel by value with a one-warp launch whose completion the call
 * detects from a mapped flag (no stream synchronisation).  Dotted functions
 * take x1 = NULL.  Thread-safe: each device has two pipelines, so two calls
 * from different host threads run concurrently; further calls queue. */
TF_API int tf_eval_host(int fn, int width, const void* x0, const void* x1, void* z0, void* z1,
                        int64_t n, int64_t chunk, void* stream, int flags);

/* Shard-invariant synthetic inputs: elements [start, start+n) of distribution
 * `dist` for `seed` (bit-identical to workloads.generate). */
TF_API int tf_generate(int dist, uint64_t seed, int64_t start, int64_t n, void* x0, void* x1,
                       void* stream);

/* Accumulate parity statistics of (z0, z1) against (r0, r1) into the 6
 * counters at stats_dev (device memory, caller-zeroed):
 * [elements, z0 bit mismatches, z0 mismatches > 1 ulp, |dz| > max(rel|r|, abs_guard, 2 ulp(r1)),
 *  non-finite class mismatches, z1 bit mismatches]. */
TF_API int tf_compare(int width, const void* z0, const void* z1, const void* r0, const void* r1,
                      int64_t n, double rel, double abs_guard, unsigned long long* stats_dev,
                      void* stream);

/* Parity / error statistics of one shard: the tf_compare counters plus the
 * accuracy audit's (sum, max, count) of relative errors (reference
 * audit.py:205-269 run_accuracy; SPEC.md "merge of (sum, max, count) is
 * order-independent").  err_max is -inf when no error was recorded. */
typedef struct tf_stats {
  uint64_t n;              /* elements compared */
  uint64_t z0_mismatch;    /* z0 bit mismatches */
  uint64_t z0_gt1ulp;      /* z0 mismatches beyond 1 ulp */
  uint64_t tol_violations; /* |(z0 + z1) - (r0 + r1)| beyond the tolerance */
  uint64_t class_mismatch; /* non-finite class mismatches */
  uint64_t z1_mismatch;    /* z1 bit mismatches */
  uint64_t included;       /* samples in the error sum (audit) */
  uint64_t warnings;       /* errors above the L0 threshold (audit) */
  double err_sum;          /* sum of relative errors (audit L1 numerator) */
  double err_max;          /* max relative error (audit L0, or log2 of it) */
} tf_stats;

/* Merge nparts shard statistics into *out: counts and sums add, maxima take
 * the max (NaN entries ignored).  Host memory only, no device work; the
 * contiguous shards of a multi-GPU run merge to the single-process result
 * (the one small cross-rank reduction of SURVEY.md 8(e)).  nparts == 0 gives
 * the empty record. */
TF_API int tf_reduce_stats(const tf_stats* parts, int64_t nparts, tf_stats* out);

/* FP-pipe calibration: `blocks` CTAs x 256 threads x `iters` x 8 independent
 * ops of the given width; width + 100 selects DADD/FADD chains, width + 200
 * DMUL/FMUL chains, plain width FMA chains. */
TF_API int tf_fma_peak(int width, void* out_dev, int blocks, int iters, void* stream);

/* Elements routed through the exact path since the last reset (needs
 * TF_FLAG_COUNT_EXACT on the counted calls); synchronous. */
TF_API int tf_exact_count(unsigned long long* out, int reset);

/* ---- accuracy audit (reference audit.py:207-286 run_accuracy; etalon
 * oracle.py:37-167).  Families: 0 exp, 1 expm1, 2 log, 3 log1p
 * (explog.py:44-49 FAMILIES). */
#define TF_FAM_EXP 0
#define TF_FAM_EXPM1 1
#define TF_FAM_LOG 2
#define TF_FAM_LOG1P 3
#define TF_ETALON_ORACLE 0 /* triple-double high-precision etalon (~2^-140 relative) */
#define TF_ETALON_LIB 1    /* binary64 library at x0 + x1 (binary32 audits only) */
/* audit sample states: included, excluded (non-finite / below the error floor),
 * etalon domain error, zero reference (absolute fallback) */
#define TF_AUDIT_INCLUDED 0
#define TF_AUDIT_FLOOR 1
#define TF_AUDIT_DOMAIN 2
#define TF_AUDIT_ABSOLUTE 3

/* Per-sample relative error of the results (z0, z1) of a `family` function at
 * the arguments (x0, x1), all device arrays of the lane type of `width`;
 * err[] (double) and state[] (TF_AUDIT_*) are device outputs. */
TF_API int tf_audit_errors(int family, int width, int etalon_kind, const void* x0, const void* x1,
                           const void* z0, const void* z1, int64_t n, double* err,
                           unsigned char* state, void* stream);

/* The triple-double etalon itself at x0 + x1 (binary64 device arrays):
 * value = (m[i] + m[n+i] + m[2n+i]) * 2^k[i]; NaN words outside the domain. */
TF_API int tf_etalon(int family, const double* x0, const double* x1, int64_t n, double* m,
                     int* k, void* stream);

/* run_bench's checksum (audit.py:344-349): XOR over i of the binary64 bit
 * pattern of (double) z0[i], written to *out (device). */
TF_API int tf_checksum(int width, const void* z0, int64_t n, unsigned long long* out,
                       void* stream);

/* ---- element-wise EFTs and twofold arithmetic over device arrays
 * (reference eft.py:77-237 binary64, eft32.py:36-214 binary32), bit-exact
 * including the _special non-finite policy.  Operands: a = (a0, a1),
 * b = (b0, b1); scalar ops read a0 (and b0); results (z0, z1) = (value, error)
 * or (hi, lo) for split.  backend: 0 = "fma" residual, 1 = "dv" (Dekker /
 * Veltkamp, fma_sim remainders); it only matters for the ops marked [b]. */
#define TF_OP_FAST_TWO_SUM 0 /* fast_two_sum(a0, b0)   eft.py:77-82   */
#define TF_OP_TWO_SUM 1      /* two_sum(a0, b0)        eft.py:85-92   */
#define TF_OP_TWO_DIFF 2     /* two_diff(a0, b0)       eft.py:95-104  */
#define TF_OP_TWO_PROD 3     /* two_prod_*(a0, b0) [b] eft.py:131-149 */
#define TF_OP_SPLIT 4        /* split(a0) -> (hi, lo)  eft.py:115-128 */
#define TF_OP_RENORM_FAST 5  /* renorm_fast(a)         eft.py:163-165 */
#define TF_OP_RENORM 6       /* renorm(a)              eft.py:168-171 */
#define TF_OP_T_ADD 7        /* t_add(a, b)            eft.py:182-189 */
#define TF_OP_T_ADD_D 8      /* t_add_d(a, b0)         eft.py:192-199 */
#define TF_OP_T_MUL 9        /* t_mul(a, b) [b]        eft.py:207-212 */
#define TF_OP_T_MUL_D 10     /* t_mul_d(a, b0) [b]     eft.py:214-219 */
#define TF_OP_T_DIV 11       /* t_div(a, b) [b]        eft.py:221-226 */
#define TF_OP_T_SQRT 12      /* t_sqrt(a) [b]          eft.py:228-235 */
#define TF_OP_COUNT 13

TF_API int tf_eft(int op, int width, int backend, const void* a0, const void* a1, const void* b0,
                  const void* b1, void* z0, void* z1, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TWOFOLD_B200_H */
