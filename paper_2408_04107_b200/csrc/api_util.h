// api_util.h — error reporting shared by the C-ABI translation units.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "zdc.h"

namespace zdc {
void set_error(const char* fmt, ...);
zdc_status fail(zdc_status s, const char* fmt, ...);
// byte ranges [a, a + na) and [b, b + nb) overlap (the x / y alias check of every entry point)
inline bool ranges_overlap(const void* a, long long na, const void* b, long long nb) {
  const char* pa = static_cast<const char*>(a);
  const char* pb = static_cast<const char*>(b);
  return pa < pb + nb && pb < pa + na;
}
}  // namespace zdc

#define ZDC_CUDA_TRY(expr)                                                                   \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return ::zdc::fail(ZDC_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                         __LINE__);                                                          \
  } while (0)
