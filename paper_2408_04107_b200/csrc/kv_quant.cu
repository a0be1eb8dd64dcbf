// kv_quant.cu — NEXT-4: the FP8 compressed cache of GEAR-ZDC (P:1642 DEL: "quantizes
// each matrix element of the compressed data after ZDC compression and dequantizes them before ZDC
// decompression").  Reading c23: one scale per cached row (token, KV head) of r values,
// scale = max|x| / 448 in f32 (1 for an all-zero row), code = E4M3(x / scale) with round-to-
// nearest-even and saturation; the row is stored as r codes, the f32 scale and 12 pad bytes so
// every row stays 16-byte aligned for the decode kernel's bulk copies.  One warp per row.
#include <cuda_fp8.h>

#include "common.cuh"
#include "kernels.h"

namespace zdc {

__global__ void __launch_bounds__(256) quantize_kv_kernel(const uint16_t* __restrict__ src, int64_t src_bg,
                                                          uint8_t* __restrict__ dst, int S_cap, int n_bg, int t0, int T,
                                                          int w, const int* __restrict__ pos_ptr) {
  const int lane = threadIdx.x & 31;
  const int64_t nrows = static_cast<int64_t>(n_bg) * T;
  const int base = pos_ptr ? min(*pos_ptr, S_cap - 1) : 0;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < nrows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int bg = static_cast<int>(r / T), t = t0 + static_cast<int>(r % T);
    const uint16_t* x = src + (static_cast<int64_t>(bg) * src_bg + t) * w;
    float v[4];
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = lane + 32 * i;
      v[i] = c < w ? __uint_as_float(static_cast<uint32_t>(x[c]) << 16) : 0.f;
      amax = fmaxf(amax, fabsf(v[i]));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    const float scale = amax > 0.f ? amax / 448.0f : 1.0f;
    uint8_t* row = dst + (static_cast<int64_t>(bg) * S_cap + base + (t - t0) + (pos_ptr ? 0 : t0)) * (w + 16);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = lane + 32 * i;
      if (c < w) row[c] = __nv_cvt_float_to_fp8(v[i] / scale, __NV_SATFINITE, __NV_E4M3);
    }
    if (lane == 0) {
      *reinterpret_cast<float*>(row + w) = scale;
      *reinterpret_cast<uint32_t*>(row + w + 4) = 0u;
      *reinterpret_cast<uint2*>(row + w + 8) = make_uint2(0u, 0u);
    }
  }
}

cudaError_t launch_quantize_kv(const uint16_t* src, int64_t src_bg, uint8_t* dst, int S_cap, int n_bg, int t0, int T,
                               int w, const int* pos_ptr, cudaStream_t s) {
  if (w > 128 || w % 16 != 0) return cudaErrorInvalidValue;
  const int64_t warps = static_cast<int64_t>(n_bg) * T;
  int64_t blocks = (warps + 7) / 8;
  if (blocks > 16 * num_sms()) blocks = 16 * num_sms();
  if (blocks < 1) blocks = 1;
  quantize_kv_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(src, src_bg, dst, S_cap, n_bg, t0, T, w, pos_ptr);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace zdc
