// sp_ulysses.cu — re-layout kernels of the paper's own SP dataflow (§5.3,
// Fig. bkg:fig:all2all): "each sequence partition undergoes linear projection
// to form Q, K, and V tensors.  Subsequently, the four GPUs execute an all-to-all operation to
// gather tokens along the sequence dimension and distribute heads ... The resulting tensors undergo
// a second all-to-all operation to gather heads and sequence partitions".  With ZDC the Q'/K'/V'
// that cross the network are the compressed (rank-r) ones.
//
// The a1 GEMM epilogue (mode 2) already writes the first all-to-all's send slabs; these kernels
// place what arrives in the layouts the attention and a5 kernels read.  Pure data movement in
// 16-byte units (8 bf16), coalesced along the columns.
#include "common.cuh"
#include "kernels.h"

namespace zdc {

__device__ __forceinline__ int uly_position(int S, int P, int q, int layout, int t) {
  const int n = S / P;
  if (layout == 0) return q * n + t;
  const int c = S / (2 * P);
  return t < c ? q * c + t : (2 * P - 1 - q) * c + (t - c);
}

__global__ void uly_unpack_qkv_kernel(const uint4* __restrict__ recv, int P, int B, int n_local, int S, int layout,
                                      int hq, int kq, int vq, int rk, int rv, uint16_t* __restrict__ q,
                                      uint16_t* __restrict__ kc, uint16_t* __restrict__ vc, int S_cap) {
  const int cols = hq + kq + vq, c8 = cols / 8;
  const int64_t total = static_cast<int64_t>(P) * B * n_local * c8;
  const int gk = kq / rk;  // this rank's KV groups
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int u = static_cast<int>(i % c8);
    const int64_t row = i / c8;  // (src, b, t)
    const int t = static_cast<int>(row % n_local);
    const int b = static_cast<int>((row / n_local) % B);
    const int src = static_cast<int>(row / (static_cast<int64_t>(n_local) * B));
    const int pos = uly_position(S, P, src, layout, t);
    const uint4 val = recv[i];
    const int c = u * 8;
    uint16_t* dst;
    if (c < hq) {
      dst = q + (static_cast<int64_t>(b) * S + pos) * hq + c;
    } else if (c < hq + kq) {
      const int cc = c - hq, g = cc / rk, e = cc - g * rk;
      dst = kc + ((static_cast<int64_t>(b) * gk + g) * S_cap + pos) * rk + e;
    } else {
      const int cc = c - hq - kq, g = cc / rv, e = cc - g * rv;
      dst = vc + ((static_cast<int64_t>(b) * gk + g) * S_cap + pos) * rv + e;
    }
    *reinterpret_cast<uint4*>(dst) = val;
  }
}

__global__ void uly_pack_o_kernel(const uint4* __restrict__ o, int P, int B, int n_local, int S, int layout, int ho,
                                  uint4* __restrict__ send) {
  const int c8 = ho / 8;
  const int64_t total = static_cast<int64_t>(P) * B * n_local * c8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int u = static_cast<int>(i % c8);
    const int64_t row = i / c8;  // (dst, b, t)
    const int t = static_cast<int>(row % n_local);
    const int b = static_cast<int>((row / n_local) % B);
    const int dst = static_cast<int>(row / (static_cast<int64_t>(n_local) * B));
    const int pos = uly_position(S, P, dst, layout, t);
    send[i] = o[(static_cast<int64_t>(b) * S + pos) * c8 + u];
  }
}

__global__ void uly_unpack_o_kernel(const uint4* __restrict__ recv, int P, int B, int n_local, int ho,
                                    uint4* __restrict__ o, int ko_p) {
  const int k8 = ko_p / 8, c8 = ho / 8;
  const int64_t total = static_cast<int64_t>(B) * n_local * k8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int u = static_cast<int>(i % k8);
    const int64_t m = i / k8;  // local row b * n_local + t
    const int src = u / c8, cu = u - src * c8;
    o[i] = src < P ? recv[(static_cast<int64_t>(src) * B * n_local + m) * c8 + cu] : make_uint4(0, 0, 0, 0);
  }
}

static int uly_grid(int64_t units) {
  const int64_t g = (units + 255) / 256;
  const int cap = 8 * num_sms();
  return static_cast<int>(g < cap ? (g > 0 ? g : 1) : cap);
}

cudaError_t launch_ulysses_unpack_qkv(const uint16_t* recv, int P, int B, int n_local, int S, int layout, int hq, int kq,
                                      int vq, int rk, int rv, uint16_t* q, uint16_t* kc, uint16_t* vc, int S_cap,
                                      cudaStream_t s) {
  if ((hq | kq | vq | rk | rv) % 8 != 0) return cudaErrorInvalidValue;
  const int64_t units = static_cast<int64_t>(P) * B * n_local * ((hq + kq + vq) / 8);
  uly_unpack_qkv_kernel<<<uly_grid(units), 256, 0, s>>>(reinterpret_cast<const uint4*>(recv), P, B, n_local, S, layout,
                                                        hq, kq, vq, rk, rv, q, kc, vc, S_cap);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_ulysses_pack_o(const uint16_t* o, int P, int B, int n_local, int S, int layout, int ho,
                                  uint16_t* send, cudaStream_t s) {
  if (ho % 8 != 0) return cudaErrorInvalidValue;
  const int64_t units = static_cast<int64_t>(P) * B * n_local * (ho / 8);
  uly_pack_o_kernel<<<uly_grid(units), 256, 0, s>>>(reinterpret_cast<const uint4*>(o), P, B, n_local, S, layout, ho,
                                                    reinterpret_cast<uint4*>(send));
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_ulysses_unpack_o(const uint16_t* recv, int P, int B, int n_local, int ho, uint16_t* o, int ko_p,
                                    cudaStream_t s) {
  if (ho % 8 != 0 || ko_p % 8 != 0 || P * ho > ko_p) return cudaErrorInvalidValue;
  const int64_t units = static_cast<int64_t>(B) * n_local * (ko_p / 8);
  uly_unpack_o_kernel<<<uly_grid(units), 256, 0, s>>>(reinterpret_cast<const uint4*>(recv), P, B, n_local, ho,
                                                      reinterpret_cast<uint4*>(o), ko_p);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace zdc
