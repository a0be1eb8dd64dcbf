// decode_cluster_b1.cu — instances of the cluster decode kernel for batch widths NB = 1
#include "decode_cluster.cuh"

namespace zdc {
cudaError_t cluster_dispatch_b1(const DecClusterArgs& a, int* cap, int C, int RK, int G, cudaStream_t s) {
  return dispatch_cluster_r<1>(a, cap, C, RK, G, s);
}
}  // namespace zdc
