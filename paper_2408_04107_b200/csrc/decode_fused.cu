// decode_fused.cu — host dispatch of the fused decode layer-step (kernel: decode_fused.cuh)
#include "kernels.h"

#include <cstdlib>

namespace zdc {

cudaError_t launch_fused_b1(const DecFusedArgs& a, int RK, int G, cudaStream_t s);
cudaError_t launch_fused_b2(const DecFusedArgs& a, int RK, int G, cudaStream_t s);
cudaError_t launch_fused_b4(const DecFusedArgs& a, int RK, int G, cudaStream_t s);
cudaError_t launch_fused_b8(const DecFusedArgs& a, int RK, int G, cudaStream_t s);

int decode_fused_splits(int B, int Nkv) {
  static const int forced = knob("ZDC_FUSED_SPLITS", 0);  // A/B override (capped like the default)
  if (forced > 0) return forced > 128 ? 128 : forced;
  int s = num_sms() / (B * Nkv);
  if (s > 128) s = 128;
  return s < 1 ? 1 : s;
}

bool decode_fused_supported(int B, int RK, int G) {
  return B >= 1 && B <= 8 && (RK == 16 || RK == 32 || RK == 64 || RK == 96 || RK == 128) &&
         (G == 1 || G == 2 || G == 4 || G == 8);
}

unsigned long long* fused_trace_buffer() {
  static unsigned long long* buf = nullptr;
  static bool init = false;
  if (!init) {
    init = true;
    if (knob("ZDC_FUSED_TRACE", 0) && cudaMalloc(&buf, 1024 * 16 * 8) != cudaSuccess) buf = nullptr;
    if (buf) cudaMemset(buf, 0, 1024 * 16 * 8);
  }
  return buf;
}

cudaError_t launch_decode_fused(const DecFusedArgs& a, int RK, cudaStream_t s) {
  const int G = a.Nh / a.Nkv;
  if (!decode_fused_supported(a.B, RK, G) || a.d % 8 != 0 || a.ko_p % 8 != 0) return cudaErrorNotSupported;
  if (a.B == 1) return launch_fused_b1(a, RK, G, s);
  if (a.B == 2) return launch_fused_b2(a, RK, G, s);
  if (a.B <= 4) return launch_fused_b4(a, RK, G, s);
  return launch_fused_b8(a, RK, G, s);
}

}  // namespace zdc

extern "C" int zdc_trace_read(unsigned long long* out, int n) {
  unsigned long long* b = zdc::fused_trace_buffer();
  if (!b || !out || n <= 0) return 0;
  if (n > 1024 * 16) n = 1024 * 16;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (cudaMemcpy(out, b, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return n;
}
