// attn_prefill.cu — a3 for prompt processing: dispatch of the causal attention kernels at head
// dimension r, run directly on the compressed Q'/K'/V' (Lemma 2: Q'(K')^T ~ QK^T needs
// no decompression; the V' decompression happens inside a5).  Eqs. 2-3
// with the ORIGINAL scale 1/sqrt(d_h) (reading c2), and the log of each row's softmax denominator
// (LSE) written out in f32 — the "reused softmax denominators" of P:1442 that a4 ranks.
//
//   r <= 96           attn_prefill4.cu  persistent, two query tiles per work item, P in TMEM (r <= 64)
//   r in {112, 128}   attn_prefill3.cu  one 128-row query tile per CTA
// Both run the two contractions on tcgen05 (S = Q'K'^T and O += P V' with TMEM accumulators, TMA
// operands) and accept the SP gather-buffer key addressing (kv_mode 1, comm.cpp).
// (The round-1 kernels v1 / v2 that these superseded were removed in round 2.)
#include "common.cuh"
#include "kernels.h"

namespace zdc {

cudaError_t launch_prefill_attention(const PrefillAttnArgs& a, cudaStream_t stream) {
  if (a.rk != a.rv) return cudaErrorInvalidValue;
  if (prefill_attention_v4_supported(a.rk)) return launch_prefill_attention_v4(a, stream);
  return launch_prefill_attention_v3(a, stream);
}

}  // namespace zdc
