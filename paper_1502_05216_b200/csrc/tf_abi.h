// tf_abi.h -- host-side helpers shared by the translation units of
// libtwofold_b200.so (error string, CUDA status, SM count).
#pragma once
#include "../../include/twofold_b200.h"

namespace tfabi {
extern thread_local char g_err[512];
extern bool g_const_ready[64];
int fail(int code, const char* fmt, const char* detail = "");
int cuda_check(const char* what);
int device_sms();
// tiny launch (n <= 32) of HOST operands x0 / x1 (passed by value) that stores seq to
// *done (mapped host memory) after its results z0 / z1 (mapped too)
int tiny_eval(int fn, int width, const void* x0, const void* x1, void* z0, void* z1, int64_t n,
              void* stream, unsigned* done, unsigned seq);
}  // namespace tfabi
