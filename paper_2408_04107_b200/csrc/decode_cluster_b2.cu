// decode_cluster_b2.cu — instances of the cluster decode kernel for batch widths NB = 2
#include "decode_cluster.cuh"

namespace zdc {
cudaError_t cluster_dispatch_b2(const DecClusterArgs& a, int* cap, int C, int RK, int G, cudaStream_t s) {
  return dispatch_cluster_r<2>(a, cap, C, RK, G, s);
}
}  // namespace zdc
