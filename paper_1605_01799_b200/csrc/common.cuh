// common.cuh — host-side helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <string>

namespace hopf {
extern thread_local std::string g_last_error;
extern thread_local int32_t g_launches;
extern thread_local const char *g_last_kernel;
int set_error(int code, const char *fmt, ...);
int check_launch(const char *what);
int num_sms();
}  // namespace hopf
