// select.cu — a4 (token importance + rank selection) and the class-aware KV packing of a2 for
// the layer-token hybrid compression of §5.2:
//   importance_kernel   score_t = log sum_h exp(LSE_{h,t}): the reused softmax denominators
//                       sum_h sum_{k<=t} exp(s_k^h) of P:1442 in the log domain (reading c9),
//                       fixed head order; mode 1 subtracts log(t+1) per head (reading c10).
//   select_kernel       "sorted in descending order, g^l proportion of tokens from the top are
//                       classified as important": deterministic radix select of the
//                       k-th largest 64-bit key (score desc, index asc), k = ceil(g S) in integer
//                       basis points (reading c11); tau = the k-th score (reading c12).
//   truncate_kernel     non-representative layers: unimportant rows lose dims >= r^u before
//                       attention (zero-fill, P:774-776 DEL).
//   rank_kernel         stable class-aware compaction indices: __ballot_sync + __popc warp scan,
//                       block scan of the warp totals.
//   pack_kernel         coalesced 16-byte copy of every staged K'/V' row into pool_I (width r^i)
//                       or pool_U (width r^u, truncated) at its compacted index.
//   append / classify   the decode-step versions (one new token per sequence).
#include "common.cuh"
#include "kernels.h"

namespace zdc {


// ------------------------------------------------------------------ importance
__global__ void importance_kernel(const float* __restrict__ lse, int T, int Nh, int B, int t0, int mode,
                                  float* __restrict__ scores, int64_t ld_scores, float* __restrict__ out_copy,
                                  int64_t ld_copy, const int* __restrict__ pos_ptr) {
  const int b = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int pos = (pos_ptr ? *pos_ptr : t0) + t;  // position of the token (decode: the new token)
  const float adj = mode == 1 ? logf(static_cast<float>(pos) + 1.0f) : 0.f;
  float m = -INFINITY;
  for (int h = 0; h < Nh; ++h) m = fmaxf(m, lse[(static_cast<int64_t>(b) * Nh + h) * T + t] - adj);
  float s = 0.f;
  for (int h = 0; h < Nh; ++h) s += expf(lse[(static_cast<int64_t>(b) * Nh + h) * T + t] - adj - m);
  const float score = m + logf(s);
  scores[b * ld_scores + pos] = score;
  if (out_copy) out_copy[b * ld_copy + pos] = score;
}

// ------------------------------------------------------------------ selection (radix select)
__device__ __forceinline__ uint64_t order_key(float score, int t) {
  uint32_t u = __float_as_uint(score);
  if (u == 0x80000000u) u = 0;                         // -0.0 == +0.0 (reading c11)
  const uint32_t ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // monotone in the float value
  return (static_cast<uint64_t>(ord) << 32) | static_cast<uint64_t>(0xFFFFFFFFu - static_cast<uint32_t>(t));
}

// One CTA of 1024 threads per sequence.  Important = the k largest keys.
__global__ void __launch_bounds__(1024) select_kernel(const float* __restrict__ scores, int64_t ld, int S, int g_bp,
                                                      uint8_t* __restrict__ cls, float* __restrict__ tau,
                                                      int* __restrict__ nan_flag) {
  const int b = blockIdx.x;
  const float* sc = scores + b * ld;
  // a NaN score has no place in the order (the oracle raises, reading c11): flag it for the host
  if (nan_flag)
    for (int t = threadIdx.x; t < S; t += blockDim.x)
      if (isnan(sc[t])) *nan_flag = 1;
  const int k = static_cast<int>((static_cast<int64_t>(g_bp) * S + 9999) / 10000);
  __shared__ uint32_t hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int s_k;
  __shared__ float s_tau;
  if (k <= 0 || k >= S) {
    for (int t = threadIdx.x; t < S; t += blockDim.x) cls[b * ld + t] = k >= S ? 1 : 0;
    if (threadIdx.x == 0) tau[b] = k >= S ? -INFINITY : INFINITY;
    return;
  }
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_k = k;
  }
  __syncthreads();
  // MSB-first: at pass p the top 8p bits of the k-th largest key are known (s_prefix)
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    const uint64_t hi_mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    for (int t = threadIdx.x; t < S; t += blockDim.x) {
      const uint64_t key = order_key(sc[t], t);
      if ((key & hi_mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int rem = s_k;
      int digit = 255;
      for (; digit > 0; --digit) {
        if (static_cast<int>(hist[digit]) >= rem) break;
        rem -= hist[digit];
      }
      s_prefix = prefix | (static_cast<uint64_t>(digit) << shift);
      s_k = rem;
    }
    __syncthreads();
  }
  const uint64_t kth = s_prefix;  // the exact k-th largest key (keys are unique)
  for (int t = threadIdx.x; t < S; t += blockDim.x) {
    const uint64_t key = order_key(sc[t], t);
    cls[b * ld + t] = key >= kth ? 1 : 0;
    if (key == kth) s_tau = sc[t];
  }
  __syncthreads();
  if (threadIdx.x == 0) tau[b] = s_tau;
}

// ------------------------------------------------------------------ prefill: truncate / rank / pack
// Zero dims [r_u, width) of unimportant rows of a staged [B][Nkv][S_cap][width] buffer.
__global__ void truncate_kernel(uint16_t* __restrict__ kv, int width, int r_u, int B, int Nkv, int S, int S_cap,
                                const uint8_t* __restrict__ cls, int64_t ld_cls) {
  const int64_t total = static_cast<int64_t>(B) * Nkv * S;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(i % S);
    const int64_t bg = i / S;
    const int b = static_cast<int>(bg / Nkv);
    if (cls[b * ld_cls + t]) continue;
    uint16_t* row = kv + (bg * S_cap + t) * width;
    for (int c = r_u; c < width; ++c) row[c] = 0;
  }
}

// Per sequence: didx[t] = compacted index of token t in its pool (important: >= 0 index into
// pool_I, unimportant: -(index into pool_U) - 1); pos_I / pos_U record the positions; n_I / n_U.
__global__ void __launch_bounds__(1024) rank_kernel(const uint8_t* __restrict__ cls, int64_t ld_cls, int S,
                                                    int* __restrict__ didx, int64_t ld_didx, int* __restrict__ pos_i,
                                                    int* __restrict__ pos_u, int64_t ld_pos, int* __restrict__ n_i,
                                                    int* __restrict__ n_u) {
  const int b = blockIdx.x;
  __shared__ int warp_tot[32];
  __shared__ int base_i;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) base_i = 0;
  __syncthreads();
  for (int t0 = 0; t0 < S; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    const bool imp = t < S && cls[b * ld_cls + t];
    const unsigned bal = __ballot_sync(0xffffffffu, imp);
    const int in_warp = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 32 warp totals
      const int v = warp_tot[lane];
      int incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += n;
      }
      warp_tot[lane] = incl - v;
    }
    __syncthreads();
    const int rank_i = base_i + warp_tot[warp] + in_warp;  // important tokens before t
    if (t < S) {
      if (imp) {
        didx[b * ld_didx + t] = rank_i;
        pos_i[b * ld_pos + rank_i] = t;
      } else {
        const int rank_u = t - rank_i;
        didx[b * ld_didx + t] = -rank_u - 1;
        pos_u[b * ld_pos + rank_u] = t;
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base_i = rank_i + (imp ? 1 : 0);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    n_i[b] = base_i;
    n_u[b] = S - base_i;
  }
}

// Copy staged rows into the pools, 16 bytes per thread, consecutive threads on consecutive
// units of a row (coalesced reads and writes).  Unimportant rows keep units < ceil(r_u/8) with
// dims >= r_u zeroed (padding).
__global__ void pack_kernel(const uint16_t* __restrict__ src, int w, uint16_t* __restrict__ pool_i,
                            uint16_t* __restrict__ pool_u, int wu, int r_u, int B, int Nkv, int S, int S_cap,
                            const int* __restrict__ didx, int64_t ld_didx) {
  const int units = w / 8;
  const int64_t total = static_cast<int64_t>(B) * Nkv * S * units;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int u = static_cast<int>(i % units);
    const int64_t row = i / units;  // (b*Nkv + g)*S + t
    const int t = static_cast<int>(row % S);
    const int64_t bg = row / S;
    const int b = static_cast<int>(bg / Nkv);
    const int di = didx[b * ld_didx + t];
    const uint4 val = *reinterpret_cast<const uint4*>(src + (bg * S_cap + t) * w + u * 8);
    if (di >= 0) {
      *reinterpret_cast<uint4*>(pool_i + (bg * S_cap + di) * w + u * 8) = val;
    } else if (u * 8 < wu) {
      uint4 v = val;
      uint16_t* e = reinterpret_cast<uint16_t*>(&v);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (u * 8 + q >= r_u) e[q] = 0;
      *reinterpret_cast<uint4*>(pool_u + (bg * S_cap + (-di - 1)) * wu + u * 8) = v;
    }
  }
}

// ------------------------------------------------------------------ decode: append / classify
// One block per sequence.  The new token (position *len_ptr) goes to pool_I (representative
// layer: always, it attends at r^i first) or, at a non-representative layer, to the pool of the
// class its representative assigned (truncated before attention).
__global__ void append_kernel(const uint16_t* __restrict__ knew, const uint16_t* __restrict__ vnew, int w, int Nkv,
                              uint16_t* __restrict__ ki, uint16_t* __restrict__ vi, uint16_t* __restrict__ ku,
                              uint16_t* __restrict__ vu, int wu, int r_u, int S_cap, int* __restrict__ n_i,
                              int* __restrict__ n_u, int* __restrict__ pos_i, int* __restrict__ pos_u, int64_t ld_pos,
                              const int* __restrict__ len_ptr, const uint8_t* __restrict__ rep_cls, int64_t ld_cls,
                              int is_rep) {
  pdl_wait();     // knew / vnew come from the a1 projection (a programmatic launch waits for it)
  pdl_trigger();  // the attention may start its prologue
  const int b = blockIdx.x;
  const int t = *len_ptr;
  if (t >= S_cap) return;  // cache full (graph replays past max_seq): the a5 length advance flags it
  const bool imp = is_rep || rep_cls[b * ld_cls + t];
  const int idx = imp ? n_i[b] : n_u[b];
  __syncthreads();
  const int units = w / 8;
  for (int i = threadIdx.x; i < 2 * Nkv * units; i += blockDim.x) {
    const int which = i / (Nkv * units);  // 0 = K, 1 = V
    const int rem = i - which * Nkv * units;
    const int g = rem / units, u = rem - g * units;
    const uint16_t* src = (which ? vnew : knew) + (static_cast<int64_t>(b) * Nkv + g) * w + u * 8;
    const int64_t row = (static_cast<int64_t>(b) * Nkv + g) * S_cap + idx;
    uint4 val = *reinterpret_cast<const uint4*>(src);
    if (imp) {
      *reinterpret_cast<uint4*>((which ? vi : ki) + row * w + u * 8) = val;
    } else if (u * 8 < wu) {
      uint16_t* e = reinterpret_cast<uint16_t*>(&val);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (u * 8 + q >= r_u) e[q] = 0;
      *reinterpret_cast<uint4*>((which ? vu : ku) + row * wu + u * 8) = val;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (imp) {
      pos_i[b * ld_pos + idx] = t;
      n_i[b] = idx + 1;
    } else {
      pos_u[b * ld_pos + idx] = t;
      n_u[b] = idx + 1;
    }
  }
}

// Representative layer, after the new token attended at r^i: score it (same formula as the
// prompt tokens), classify it against tau (strict >, reading c12) and, if unimportant, move its
// row from the end of pool_I to the end of pool_U (truncated).  One block per sequence.
__global__ void classify_kernel(const float* __restrict__ lse, int Nh, int mode, const float* __restrict__ tau,
                                float* __restrict__ scores, uint8_t* __restrict__ cls, int64_t ld,
                                float* __restrict__ out_copy, int64_t ld_copy, int w, int Nkv, uint16_t* __restrict__ ki,
                                uint16_t* __restrict__ vi, uint16_t* __restrict__ ku, uint16_t* __restrict__ vu,
                                int wu, int r_u, int S_cap, int* __restrict__ n_i, int* __restrict__ n_u,
                                int* __restrict__ pos_i, int* __restrict__ pos_u, const int* __restrict__ len_ptr) {
  pdl_wait();     // the LSE of the attention
  pdl_trigger();
  const int b = blockIdx.x;
  const int t = *len_ptr;
  if (t >= S_cap) return;  // cache full: nothing was appended
  __shared__ int s_imp;
  if (threadIdx.x == 0) {
    const float adj = mode == 1 ? logf(static_cast<float>(t) + 1.0f) : 0.f;
    float m = -INFINITY;
    for (int h = 0; h < Nh; ++h) m = fmaxf(m, lse[b * Nh + h] - adj);
    float s = 0.f;
    for (int h = 0; h < Nh; ++h) s += expf(lse[b * Nh + h] - adj - m);
    const float score = m + logf(s);
    scores[b * ld + t] = score;
    if (out_copy) out_copy[b * ld_copy + t] = score;
    const int imp = score > tau[b] ? 1 : 0;
    cls[b * ld + t] = static_cast<uint8_t>(imp);
    s_imp = imp;
  }
  __syncthreads();
  if (s_imp) return;
  const int src_idx = n_i[b] - 1;  // the new token is the last row of pool_I
  const int dst_idx = n_u[b];
  const int units = wu / 8;
  for (int i = threadIdx.x; i < 2 * Nkv * units; i += blockDim.x) {
    const int which = i / (Nkv * units);
    const int rem = i - which * Nkv * units;
    const int g = rem / units, u = rem - g * units;
    const int64_t bg = static_cast<int64_t>(b) * Nkv + g;
    uint4 val = *reinterpret_cast<const uint4*>((which ? vi : ki) + (bg * S_cap + src_idx) * w + u * 8);
    uint16_t* e = reinterpret_cast<uint16_t*>(&val);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (u * 8 + q >= r_u) e[q] = 0;
    *reinterpret_cast<uint4*>((which ? vu : ku) + (bg * S_cap + dst_idx) * wu + u * 8) = val;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    pos_u[b * ld + dst_idx] = t;
    n_i[b] = src_idx;
    n_u[b] = dst_idx + 1;
  }
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_importance(const float* lse, int T, int Nh, int B, int t0, int mode, float* scores, int64_t ld,
                              float* out_copy, int64_t ld_copy, const int* pos_ptr, cudaStream_t s) {
  dim3 grid((T + 127) / 128, B);
  importance_kernel<<<grid, 128, 0, s>>>(lse, T, Nh, B, t0, mode, scores, ld, out_copy, ld_copy, pos_ptr);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_select(const float* scores, int64_t ld, int S, int g_bp, int B, uint8_t* cls, float* tau,
                          cudaStream_t s, int* nan_flag) {
  select_kernel<<<B, 1024, 0, s>>>(scores, ld, S, g_bp, cls, tau, nan_flag);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_truncate(uint16_t* kv, int width, int r_u, int B, int Nkv, int S, int S_cap, const uint8_t* cls,
                            int64_t ld_cls, cudaStream_t s) {
  truncate_kernel<<<2 * num_sms(), 256, 0, s>>>(kv, width, r_u, B, Nkv, S, S_cap, cls, ld_cls);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_rank(const uint8_t* cls, int64_t ld_cls, int S, int B, int* didx, int64_t ld_didx, int* pos_i,
                        int* pos_u, int64_t ld_pos, int* n_i, int* n_u, cudaStream_t s) {
  rank_kernel<<<B, 1024, 0, s>>>(cls, ld_cls, S, didx, ld_didx, pos_i, pos_u, ld_pos, n_i, n_u);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_pack(const uint16_t* src, int w, uint16_t* pool_i, uint16_t* pool_u, int wu, int r_u, int B, int Nkv,
                        int S, int S_cap, const int* didx, int64_t ld_didx, cudaStream_t s) {
  pack_kernel<<<4 * num_sms(), 256, 0, s>>>(src, w, pool_i, pool_u, wu, r_u, B, Nkv, S, S_cap, didx, ld_didx);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_append(const uint16_t* knew, const uint16_t* vnew, int w, int Nkv, uint16_t* ki, uint16_t* vi,
                          uint16_t* ku, uint16_t* vu, int wu, int r_u, int S_cap, int* n_i, int* n_u, int* pos_i,
                          int* pos_u, int64_t ld_pos, const int* len_ptr, const uint8_t* rep_cls, int64_t ld_cls,
                          int is_rep, int B, cudaStream_t s) {
  cudaError_t e = launch_k(append_kernel, dim3(B), dim3(256), 0, s, g_pdl, knew, vnew, w, Nkv, ki, vi, ku, vu, wu, r_u,
                           S_cap, n_i, n_u, pos_i, pos_u, ld_pos, len_ptr, rep_cls, ld_cls, is_rep);
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_classify(const float* lse, int Nh, int mode, const float* tau, float* scores, uint8_t* cls,
                            int64_t ld, float* out_copy, int64_t ld_copy, int w, int Nkv, uint16_t* ki, uint16_t* vi,
                            uint16_t* ku, uint16_t* vu, int wu, int r_u, int S_cap, int* n_i, int* n_u, int* pos_i,
                            int* pos_u, const int* len_ptr, int B, cudaStream_t s) {
  cudaError_t e = launch_k(classify_kernel, dim3(B), dim3(256), 0, s, g_pdl, lse, Nh, mode, tau, scores, cls, ld,
                           out_copy, ld_copy, w, Nkv, ki, vi, ku, vu, wu, r_u, S_cap, n_i, n_u, pos_i, pos_u, len_ptr);
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

__global__ void evict_last_kernel(const uint8_t* __restrict__ cls, int64_t ld_cls, int* __restrict__ n_i,
                                  int* __restrict__ n_u, int* __restrict__ pos_u, int64_t ld_pos,
                                  const int* __restrict__ len_ptr, int S_cap) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x;
  const int t = *len_ptr;
  if (threadIdx.x != 0 || t >= S_cap || cls[b * ld_cls + t]) return;
  const int dst = n_u[b];
  pos_u[b * ld_pos + dst] = t;  // recorded as evicted (no row is kept)
  n_i[b] = n_i[b] - 1;
  n_u[b] = dst + 1;
}

cudaError_t launch_evict_last(const uint8_t* cls, int64_t ld_cls, int* n_i, int* n_u, int* pos_u, int64_t ld_pos,
                              const int* len_ptr, int S_cap, int B, cudaStream_t s) {
  cudaError_t e = launch_k(evict_last_kernel, dim3(B), dim3(32), 0, s, g_pdl, cls, ld_cls, n_i, n_u, pos_u, ld_pos,
                           len_ptr, S_cap);
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace zdc
