// decode_cluster_b4.cu — instances of the cluster decode kernel for batch widths NB = 4
#include "decode_cluster.cuh"

namespace zdc {
cudaError_t cluster_dispatch_b4(const DecClusterArgs& a, int* cap, int C, int RK, int G, cudaStream_t s) {
  return dispatch_cluster_r<4>(a, cap, C, RK, G, s);
}
}  // namespace zdc
