// knobs.h — A/B and diagnostic switches of the kernel launchers.
//
// A release build (the default) compiles every knob to its default: the product library reads no
// environment variables and holds no hidden process-global configuration.  A diagnostic build
// (ZDC_BUILD_VARIANT=debug ZDC_BUILD_DEFS=-DZDC_DEBUG_KNOBS, loaded with ZDC_LIB_PATH) reads
// ZDC_<NAME> once per call site, for same-box A/B runs of kernel variants (profiles/*/NOTES.md)
// and the fused-kernel timeline trace (tools/trace_fused.py).
#pragma once
#include <cstdlib>

namespace zdc {

inline int knob(const char* name, int def) {
#ifdef ZDC_DEBUG_KNOBS
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : def;
#else
  (void)name;
  return def;
#endif
}

}  // namespace zdc
