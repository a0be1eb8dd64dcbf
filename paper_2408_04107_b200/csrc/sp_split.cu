// sp_split.cu — NEXT-2: the token-level rank split of §5.2 under sequence
// parallelism.  Importance (the reused softmax denominators, summed over all N_h heads)
// is computed by each rank for ITS query rows; the top-g selection is over the WHOLE sequence
// ("the tokens in layer l are then sorted in descending order, and g^l proportion of tokens from
// the top are classified as important"), so the ranks all-gather their scores (B S/P floats each)
// and every rank runs the same deterministic selection (select.cu) on the same [B][S] vector:
// identical classes and tau everywhere, bit-exact with a single-GPU prefill.  Unimportant rows of
// the compressed K'/V' are then truncated to r^u (zero-filled) in the gather buffer.
#include "common.cuh"
#include "kernels.h"

namespace zdc {

__global__ void sp_importance_kernel(const float* __restrict__ lse, int n_local, int Nh, int B, int mode, int S, int P,
                                     int p, int layout, float* __restrict__ out) {
  const int b = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_local) return;
  const int pos = sp_global_pos(S, P, p, layout, t);
  // the same arithmetic as importance_kernel (select.cu), per token
  const float adj = mode == 1 ? logf(static_cast<float>(pos) + 1.0f) : 0.f;
  float m = -INFINITY;
  for (int h = 0; h < Nh; ++h) m = fmaxf(m, lse[(static_cast<int64_t>(b) * Nh + h) * n_local + t] - adj);
  float s = 0.f;
  for (int h = 0; h < Nh; ++h) s += expf(lse[(static_cast<int64_t>(b) * Nh + h) * n_local + t] - adj - m);
  out[static_cast<int64_t>(b) * n_local + t] = m + logf(s);
}

__global__ void sp_scores_global_kernel(const float* __restrict__ slots, int P, int B, int n_local, int S, int layout,
                                        float* __restrict__ scores, int64_t ld) {
  const int64_t total = static_cast<int64_t>(P) * B * n_local;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(i % n_local);
    const int b = static_cast<int>((i / n_local) % B);
    const int q = static_cast<int>(i / (static_cast<int64_t>(n_local) * B));
    scores[b * ld + sp_global_pos(S, P, q, layout, t)] = slots[i];
  }
}

__global__ void sp_truncate_kernel(uint16_t* __restrict__ gbuf, int q0, int q1, int P, int layout, int S, int B,
                                   int Nkv, int n_local, int w, int r_u, const uint8_t* __restrict__ cls,
                                   int64_t ld_cls) {
  const int64_t slot_rows = static_cast<int64_t>(B) * Nkv * n_local;
  const int64_t total = static_cast<int64_t>(q1 - q0) * 2 * slot_rows;  // rows of K and V of the slots
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i % slot_rows;        // (b, g, t) within K or V of the slot
    const int64_t qk = i / slot_rows;       // (slot - q0) * 2 + {0 K, 1 V}
    const int q = q0 + static_cast<int>(qk / 2);
    const int t = static_cast<int>(r % n_local);
    const int b = static_cast<int>(r / (static_cast<int64_t>(Nkv) * n_local));
    if (cls[b * ld_cls + sp_global_pos(S, P, q, layout, t)]) continue;
    uint16_t* row = gbuf + (static_cast<int64_t>(q) * 2 * slot_rows + (qk & 1) * slot_rows + r) * w;
    for (int c = r_u; c < w; ++c) row[c] = 0;
  }
}

// ---- SP decode (NEXT-2): this rank's attention over ITS keys (its prompt slot + the decode tokens
// it owns) gives O'_p (bf16, normalised over those keys) and LSE_p; the ranks all-gather
// {O'_p, LSE_p} and merge them like the key splits of one GPU: O' = sum_p w_p O'_p / sum_p w_p,
// w_p = exp(LSE_p - max_p LSE_p), LSE = max + log sum_p w_p.
__global__ void sp_decode_pack_kernel(const uint16_t* __restrict__ o, int64_t ldo, const float* __restrict__ lse, int B,
                                      int Nh, int rv, float* __restrict__ slot) {
  const int64_t total = static_cast<int64_t>(B) * Nh * (rv + 1);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % (rv + 1));
    const int64_t bh = i / (rv + 1);
    const int b = static_cast<int>(bh / Nh), h = static_cast<int>(bh % Nh);
    slot[i] = c < rv ? __uint_as_float(static_cast<uint32_t>(o[b * ldo + h * rv + c]) << 16) : lse[bh];
  }
}

__global__ void sp_decode_merge_kernel(const float* __restrict__ slots, int P, int B, int Nh, int rv,
                                       uint16_t* __restrict__ o, int64_t ldo, float* __restrict__ lse) {
  const int64_t per = static_cast<int64_t>(B) * Nh * (rv + 1);
  const int64_t total = static_cast<int64_t>(B) * Nh * rv;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % rv);
    const int64_t bh = i / rv;
    float M = -INFINITY;
    for (int q = 0; q < P; ++q) M = fmaxf(M, slots[q * per + bh * (rv + 1) + rv]);
    float W = 0.f, O = 0.f;
    for (int q = 0; q < P; ++q) {
      const float* e = slots + q * per + bh * (rv + 1);
      const float w = e[rv] == -INFINITY ? 0.f : expf(e[rv] - M);
      W += w;
      O = fmaf(w, e[c], O);
    }
    const int b = static_cast<int>(bh / Nh), h = static_cast<int>(bh % Nh);
    o[b * ldo + h * rv + c] = f32_to_bf16_bits(O / W);
    if (c == 0 && lse) lse[bh] = M + logf(W);
  }
}

static int sp_grid(int64_t n) {
  const int64_t g = (n + 255) / 256;
  const int cap = 8 * num_sms();
  return static_cast<int>(g < 1 ? 1 : (g < cap ? g : cap));
}

cudaError_t launch_sp_importance(const float* lse, int n_local, int Nh, int B, int mode, int S, int P, int p,
                                 int layout, float* out, cudaStream_t s) {
  dim3 grid((n_local + 127) / 128, B);
  sp_importance_kernel<<<grid, 128, 0, s>>>(lse, n_local, Nh, B, mode, S, P, p, layout, out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_sp_scores_global(const float* slots, int P, int B, int n_local, int S, int layout, float* scores,
                                    int64_t ld, cudaStream_t s) {
  sp_scores_global_kernel<<<sp_grid(static_cast<int64_t>(P) * B * n_local), 256, 0, s>>>(slots, P, B, n_local, S,
                                                                                         layout, scores, ld);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_sp_truncate(uint16_t* gbuf, int q0, int q1, int P, int layout, int S, int B, int Nkv, int n_local,
                               int w, int r_u, const uint8_t* cls, int64_t ld_cls, cudaStream_t s) {
  const int64_t rows = static_cast<int64_t>(q1 - q0) * 2 * B * Nkv * n_local;
  sp_truncate_kernel<<<sp_grid(rows), 256, 0, s>>>(gbuf, q0, q1, P, layout, S, B, Nkv, n_local, w, r_u, cls, ld_cls);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_sp_decode_pack(const uint16_t* o, int64_t ldo, const float* lse, int B, int Nh, int rv, float* slot,
                                  cudaStream_t s) {
  sp_decode_pack_kernel<<<sp_grid(static_cast<int64_t>(B) * Nh * (rv + 1)), 256, 0, s>>>(o, ldo, lse, B, Nh, rv, slot);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_sp_decode_merge(const float* slots, int P, int B, int Nh, int rv, uint16_t* o, int64_t ldo,
                                   float* lse, cudaStream_t s) {
  sp_decode_merge_kernel<<<sp_grid(static_cast<int64_t>(B) * Nh * rv), 256, 0, s>>>(slots, P, B, Nh, rv, o, ldo, lse);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace zdc
