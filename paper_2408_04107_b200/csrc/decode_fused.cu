// decode_fused.cu — host dispatch of the fused decode layer-step (kernel: decode_fused.cuh)
#include "kernels.h"

#include <algorithm>
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

// trace ring: kTraceLaunches launches x 1024 CTAs x 32 stamps; fused_trace_buffer() hands out the
// next launch's slice (diagnostic builds only: ZDC_FUSED_TRACE)
static constexpr int kTraceLaunches = 16;
static unsigned long long* trace_base() {
  static unsigned long long* buf = nullptr;
  static bool init = false;
  if (!init) {
    init = true;
    const size_t bytes = static_cast<size_t>(kTraceLaunches) * 1024 * 32 * 8;
    if (knob("ZDC_FUSED_TRACE", 0) && cudaMalloc(&buf, bytes) != cudaSuccess) buf = nullptr;
    if (buf) cudaMemset(buf, 0, bytes);
  }
  return buf;
}
static int g_trace_next = 0;

unsigned long long* fused_trace_buffer() {
  unsigned long long* b = trace_base();
  if (!b) return nullptr;
  unsigned long long* r = b + static_cast<size_t>(g_trace_next % kTraceLaunches) * 1024 * 32;
  ++g_trace_next;
  return r;
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

// copies the trace ring: [kTraceLaunches][1024][32] ns, oldest launch first (n entries at most)
extern "C" int zdc_trace_read(unsigned long long* out, int n) {
  unsigned long long* b = zdc::trace_base();
  if (!b || !out || n <= 0) return 0;
  const int per = 1024 * 32, tot = zdc::kTraceLaunches * per;
  if (n > tot) n = tot;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  const int first = zdc::g_trace_next % zdc::kTraceLaunches;  // oldest slice
  int done = 0;
  for (int i = 0; i < zdc::kTraceLaunches && done < n; ++i) {
    const int sl = (first + i) % zdc::kTraceLaunches, m = std::min(per, n - done);
    if (cudaMemcpy(out + done, b + static_cast<size_t>(sl) * per, static_cast<size_t>(m) * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
      return -1;
    done += m;
  }
  return done;
}
