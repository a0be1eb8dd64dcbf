// decode_cluster.cu — host dispatch of the cluster decode layer-step (kernel: decode_cluster.cuh):
// cluster-size choice, W_O tensor maps, batch-width dispatch.
#include "kernels.h"

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

namespace zdc {

cudaError_t cluster_dispatch_b1(const DecClusterArgs& a, int* cap, int C, int RK, int G, cudaStream_t s);
cudaError_t cluster_dispatch_b2(const DecClusterArgs& a, int* cap, int C, int RK, int G, cudaStream_t s);
cudaError_t cluster_dispatch_b4(const DecClusterArgs& a, int* cap, int C, int RK, int G, cudaStream_t s);
cudaError_t cluster_dispatch_b8(const DecClusterArgs& a, int* cap, int C, int RK, int G, cudaStream_t s);

static int nb_of(int B) { return B == 1 ? 1 : B == 2 ? 2 : B <= 4 ? 4 : 8; }

static cudaError_t dispatch(const DecClusterArgs& a, int* cap, int C, int RK, int G, cudaStream_t s) {
  switch (nb_of(a.B)) {
    case 1: return cluster_dispatch_b1(a, cap, C, RK, G, s);
    case 2: return cluster_dispatch_b2(a, cap, C, RK, G, s);
    case 4: return cluster_dispatch_b4(a, cap, C, RK, G, s);
    default: return cluster_dispatch_b8(a, cap, C, RK, G, s);
  }
}

bool decode_cluster_layer_ok(int RK, int G) {
  return (RK == 16 || RK == 32 || RK == 64 || RK == 128) && (G == 1 || G == 2 || G == 4 || G == 8) && G * RK <= 256;
}

bool decode_cluster_supported(int B, int RK, int G) { return B >= 1 && B <= 8 && decode_cluster_layer_ok(RK, G); }

int decode_cluster_size(int B, int RK, int G, int Nkv, int d) {
  if (!decode_cluster_supported(B, RK, G) || Nkv < 1) return 0;
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int, int>, int> cap;  // (NB, RK, G, C, Nkv, d) -> resident clusters
  const int forced = knob("ZDC_DEC_CLUSTER_C", 0);
  std::lock_guard<std::mutex> lk(mu);
  for (int C = 8; C >= 1; C >>= 1) {
    if (forced > 0 && C != forced) continue;
    if (d % (64 * C) != 0) continue;
    const auto key = std::make_tuple(nb_of(B), RK, G, C, Nkv, d);
    auto it = cap.find(key);
    if (it == cap.end()) {
      DecClusterArgs a;
      a.B = B;
      a.d = d;
      a.Nkv = Nkv;
      int n = 0;
      if (dispatch(a, &n, C, RK, G, nullptr) != cudaSuccess) n = 0;
      it = cap.emplace(key, n).first;
    }
    if (it->second >= Nkv) return C;
  }
  return 0;
}

bool cluster_wo_tmap(CUtensorMap* tw, const uint16_t* wod, int Nkv, int d, int K3, int KB3) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int, int>, CUtensorMap> cw;
  std::lock_guard<std::mutex> lk(mu);
  const auto kw = std::make_tuple(static_cast<const void*>(wod), Nkv, d, K3, KB3);
  auto iw = cw.find(kw);
  if (iw == cw.end()) {
    CUtensorMap m;
    if (!make_tmap_2d(&m, wod, static_cast<uint64_t>(K3), static_cast<uint64_t>(Nkv) * d, static_cast<uint64_t>(K3) * 2,
                      static_cast<uint32_t>(KB3), 128, KB3 * 2))
      return false;
    iw = cw.emplace(kw, m).first;
  }
  *tw = iw->second;
  return true;
}

// element (i, k) of tile (g, kb): row i of the group's (Q'_g | K'_g | V'_g) rows, column kb*64 + k,
// at byte i*128 + k*2 with the 16-byte unit XOR (i & 7) (SW128 K-major image)
__global__ void pack_qkv_decode_kernel(const uint16_t* __restrict__ wqkv_t, uint16_t* __restrict__ wqd, int d, int nq,
                                       int nk, int Nkv, int G, int RK) {
  const int NV1 = (G + 2) * RK, nkb = d / 64;
  const int64_t total = static_cast<int64_t>(Nkv) * nkb * NV1 * 64;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(e % 64);
    const int64_t t = e / 64;
    const int i = static_cast<int>(t % NV1);
    const int64_t gk = t / NV1;
    const int kb = static_cast<int>(gk % nkb), g = static_cast<int>(gk / nkb);
    const int row = i < G * RK ? g * G * RK + i : i < (G + 1) * RK ? nq + g * RK + (i - G * RK)
                                                                   : nq + nk + g * RK + (i - (G + 1) * RK);
    const int unit = (k >> 3) ^ (i & 7);
    wqd[gk * NV1 * 64 + i * 64 + unit * 8 + (k & 7)] = wqkv_t[static_cast<int64_t>(row) * d + kb * 64 + k];
  }
}

cudaError_t launch_pack_qkv_decode(const uint16_t* wqkv_t, uint16_t* wqd, int d, int nq, int nk, int Nkv, int G,
                                   int RK, cudaStream_t s) {
  pack_qkv_decode_kernel<<<4 * num_sms(), 256, 0, s>>>(wqkv_t, wqd, d, nq, nk, Nkv, G, RK);
  return cudaGetLastError();
}

__global__ void pack_wo_decode_kernel(const uint16_t* __restrict__ wo_t, uint16_t* __restrict__ wod, int d, int ko_p,
                                      int Nkv, int K3) {
  const int64_t total = static_cast<int64_t>(Nkv) * d * K3;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i % K3);
    const int64_t gn = i / K3;
    const int n = static_cast<int>(gn % d), g = static_cast<int>(gn / d);
    wod[i] = wo_t[static_cast<int64_t>(n) * ko_p + g * K3 + j];
  }
}

cudaError_t launch_pack_wo_decode(const uint16_t* wo_t, uint16_t* wod, int d, int ko_p, int Nkv, int K3,
                                  cudaStream_t s) {
  pack_wo_decode_kernel<<<4 * num_sms(), 256, 0, s>>>(wo_t, wod, d, ko_p, Nkv, K3);
  return cudaGetLastError();
}

cudaError_t launch_decode_cluster(const DecClusterArgs& a, int RK, cudaStream_t s) {
  const int G = a.Nh / a.Nkv;
  if (!decode_cluster_supported(a.B, RK, G) || a.C < 1 || !a.wod || !a.wqd || a.d % (64 * a.C) != 0)
    return cudaErrorNotSupported;
  return dispatch(a, nullptr, a.C, RK, G, s);
}

}  // namespace zdc
