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
}  // namespace tfabi
