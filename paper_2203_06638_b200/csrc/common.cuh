// common.cuh — internal helpers shared by the library's translation units
// (lpp_b200.cu: kernels + ABI; updater.cu: native updater loop + sampling).
#pragma once

#include "../../include/lpp_b200.h"

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>

// last-error string (thread-local) behind lpp_last_error(); returns code
__attribute__((visibility("hidden"))) int lpp_set_err(int code, const char* fmt, ...);
// one successful kernel launch of this library (lpp_launch_count)
__attribute__((visibility("hidden"))) void lpp_count_launch();

#define set_err lpp_set_err

#define CUDA_TRY(expr)                                                      \
  do {                                                                      \
    cudaError_t e_ = (expr);                                                \
    if (e_ != cudaSuccess)                                                  \
      return set_err(LPP_E_CUDA, "%s failed: %s", #expr,                    \
                     cudaGetErrorString(e_));                               \
  } while (0)

#define LAUNCH_CHECK(name)                                                  \
  do {                                                                      \
    cudaError_t e_ = cudaGetLastError();                                    \
    if (e_ != cudaSuccess)                                                  \
      return set_err(LPP_E_CUDA, "%s launch failed: %s", name,              \
                     cudaGetErrorString(e_));                               \
    lpp_count_launch();                                                     \
  } while (0)
