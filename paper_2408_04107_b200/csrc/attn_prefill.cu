// attn_prefill.cu — placeholder until the tcgen05 prefill attention lands.
#include "kernels.h"
namespace zdc {
cudaError_t launch_prefill_attention(const PrefillAttnArgs&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace zdc
