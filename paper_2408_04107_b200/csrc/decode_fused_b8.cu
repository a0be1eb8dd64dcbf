// decode_fused_b8.cu — instantiations of the fused decode layer-step for 8 input rows (B <= 8)
// (split per batch size so the 80 template instances compile in parallel)
#include "decode_fused.cuh"

namespace zdc {
cudaError_t launch_fused_b8(const DecFusedArgs& a, int RK, int G, cudaStream_t s) {
  return launch_fused_r<8>(a, RK, G, s);
}
}  // namespace zdc
