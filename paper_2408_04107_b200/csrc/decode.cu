// decode.cu — token-generation kernels ("Q^h is obtained from the input token, while K^h
// and V^h of all previous tokens are retrieved from the KVC"), HBM-bound:
//   gemv_kernel            a1 / a5 for B <= 8 rows: every folded weight byte is read once,
//                          16-byte non-allocating loads, x staged in shared memory; the a1
//                          epilogue writes K'/V' of the new token straight into the cache (a2).
//   decode_attn_partial    a3: split-K over the context ("flash decoding"); one CTA per
//                          (chunk, KV head, sequence); the G = N_h/N_kv query heads of a KV
//                          group share each K'/V' row load (GQA, reading c4).
//                          The last CTA of each (sequence, KV head) LSE-merges the chunks -> O' (bf16)
//                          and the row LSE (f32) (no separate combine launch).
//   pack_weights_kernel    load-time truncation + zero padding + transposition of the folded
//                          weights; never on the hot path.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace zdc {

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// one bf16 output element (m, n) through the same destination map as the GEMM epilogue
__device__ __forceinline__ void store_scalar(const Epilogue& e, int m, int n, uint16_t val) {
  uint16_t* dst;
  if (e.mode == 0) {
    dst = e.d + static_cast<int64_t>(m) * e.ldd + n;
  } else {
    const QkvDest& q = e.qkv;
    if (n < q.nq) {
      dst = q.q + static_cast<int64_t>(m) * q.ldq + n;
    } else {
      const int b = m / q.S, t = m - b * q.S;
      const int pos = q.posmap ? q.posmap[t] : (q.pos_ptr ? min(*q.pos_ptr, q.pos_cap - 1) : q.pos0) + t;
      if (n < q.nq + q.nk) {
        const int nn = n - q.nq, g = nn / q.rk, c = nn - g * q.rk;
        dst = q.k + b * q.kb + g * q.kg + static_cast<int64_t>(pos) * q.rk + c;
      } else {
        const int nn = n - q.nq - q.nk, g = nn / q.rv, c = nn - g * q.rv;
        dst = q.v + b * q.vb + g * q.vg + static_cast<int64_t>(pos) * q.rv + c;
      }
    }
  }
  *dst = val;
}


// ------------------------------------------------------------------ skinny projection
// pdl_mode bit 0: trigger the dependent launch only after this kernel's own wait (bounds the
// look-ahead to one kernel); otherwise trigger at entry.  Weight rows are bulk-prefetched into L2
// before the wait: they do not depend on the predecessor, so with PDL their HBM stream overlaps
// the previous kernels of the decode step.
template <int NB>
__global__ void __launch_bounds__(256) gemv_kernel(const uint16_t* __restrict__ W, const uint16_t* __restrict__ x,
                                                   int64_t ldx, int N, int K, const Epilogue epi, int pdl_mode) {
  extern __shared__ uint4 xs[];  // [NB][K/8] bf16 units
  const int kc = K >> 3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!(pdl_mode & 1)) pdl_trigger();
  if (lane == 0)
    for (int n = blockIdx.x * 8 + warp; n < N; n += gridDim.x * 8)
      l2_prefetch(W + static_cast<int64_t>(n) * K, static_cast<uint32_t>(K) * 2u);
  pdl_wait();
  if (pdl_mode & 1) pdl_trigger();
  if (epi.len_inc && blockIdx.x == 0 && threadIdx.x == 0) advance_len(epi);
  for (int i = threadIdx.x; i < NB * kc; i += blockDim.x) {
    const int b = i / kc, c = i - b * kc;
    xs[i] = *reinterpret_cast<const uint4*>(x + b * ldx + c * 8);
  }
  __syncthreads();
  constexpr int U = 16;
  for (int n = blockIdx.x * 8 + warp; n < N; n += gridDim.x * 8) {
    const uint4* w = reinterpret_cast<const uint4*>(W + static_cast<int64_t>(n) * K);
    float acc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[b] = 0.f;
    for (int c0 = lane; c0 < kc; c0 += 32 * U) {
      uint4 wv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        wv[u] = c < kc ? ldg_stream(w + c) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        if (c < kc) {
#pragma unroll
          for (int b = 0; b < NB; ++b) acc[b] += dot8(wv[u], xs[b * kc + c]);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], off);
    }
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < NB; ++b) store_scalar(epi, b, n, f32_to_bf16_bits(acc[b]));
    }
  }
}

// TMA-staged version (the one launched): one CTA per SM owns a contiguous block of weight rows.
// Warp 8 keeps a ring of row slots in shared memory full with cp.async.bulk copies; the first
// `slots` rows are issued BEFORE the PDL wait (weights do not depend on the predecessor), so they
// stream in while the previous decode kernels run.  Warps 0-7 wait for the predecessor, stage x,
// and reduce one row per warp from shared memory.
template <int NB>
__global__ void __launch_bounds__(288, 1)
    gemv_ring_kernel(const uint16_t* __restrict__ W, const uint16_t* __restrict__ x, int64_t ldx, int N, int K,
                     const Epilogue epi, int pdl_mode, int slots) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int row_bytes = K * 2;
  const int kc = K >> 3;
  uint8_t* ring = smem_raw;
  uint4* xs = reinterpret_cast<uint4*>(smem_raw + static_cast<size_t>(slots) * row_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + static_cast<size_t>(slots) * row_bytes +
                                               static_cast<size_t>(NB) * row_bytes);
  uint64_t* empty = full + slots;
  const int per = (N + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per;
  const int nrows = max(0, min(N, r0 + per) - r0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 256) {
    for (int s = 0; s < slots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (!(pdl_mode & 1)) pdl_trigger();
  // Row i is reduced by warp i % 8; warp w owns the slots [w*spw, (w+1)*spw) and uses them in order,
  // so every mbarrier wait is for the phase right after the one last observed (a shared ring let a
  // warp wait two phases ahead, where the parity test aliases: profiles/r01/NOTES.md).
  const int spw = slots / 8;
  if (warp == 8) {
    // ---- producer: weight rows HBM -> smem ring (independent of the predecessor: no wait)
    if (lane == 0) {
      if (pdl_mode & 2) pdl_wait();  // debug knob: issue the copies only after the dependency
      for (int i = 0; i < nrows; ++i) {
        const int k = i >> 3;
        const int s = (i & 7) * spw + k % spw;
        if (k >= spw) mbar_wait(&empty[s], ((k / spw) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], row_bytes);
        bulk_g2s(ring + static_cast<size_t>(s) * row_bytes, W + static_cast<int64_t>(r0 + i) * K, row_bytes,
                 &full[s]);
      }
    }
    return;
  }
  // ---- consumers
  pdl_wait();
  if (pdl_mode & 1) pdl_trigger();
  if (epi.len_inc && blockIdx.x == 0 && threadIdx.x == 0) advance_len(epi);
  for (int i = threadIdx.x; i < NB * kc; i += 256) {
    const int b = i / kc, c = i - b * kc;
    xs[i] = *reinterpret_cast<const uint4*>(x + b * ldx + c * 8);
  }
  asm volatile("bar.sync 1, 256;" ::: "memory");
  for (int i = warp; i < nrows; i += 8) {
    const int k = i >> 3;
    const int s = warp * spw + k % spw;
    mbar_wait(&full[s], (k / spw) & 1);
    const uint4* w = reinterpret_cast<const uint4*>(ring + static_cast<size_t>(s) * row_bytes);
    float acc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[b] = 0.f;
#pragma unroll 4
    for (int c = lane; c < kc; c += 32) {
      const uint4 wv = w[c];
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[b] += dot8(wv, xs[b * kc + c]);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], off);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&empty[s]);
#pragma unroll
      for (int b = 0; b < NB; ++b) store_scalar(epi, b, r0 + i, f32_to_bf16_bits(acc[b]));
    }
  }
}

// ring bytes per CTA (tunable with ZDC_GEMV_RING_KB); 96 KB leaves room for the next kernel's CTAs
static const int kGemvRingBytes = knob("ZDC_GEMV_RING_KB", 128) * 1024;
// CTAs per SM for the projection GEMV (tunable with ZDC_GEMV_CTAS)
static const int kGemvCtasPerSm = knob("ZDC_GEMV_CTAS", 1);

template <int NB>
static cudaError_t launch_gemv_nb(const uint16_t* W, const uint16_t* x, int64_t ldx, int N, int K, const Epilogue& epi,
                                  cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(gemv_ring_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int blocks = (N + 7) / 8;
  if (blocks > num_sms() * kGemvCtasPerSm) blocks = num_sms() * kGemvCtasPerSm;
  const int per = (N + blocks - 1) / blocks;
  int spw = kGemvRingBytes / (8 * K * 2);  // slots per consumer warp
  if (spw > (per + 7) / 8) spw = (per + 7) / 8;
  if (spw < 1) spw = 1;
  const int slots = 8 * spw;
  const size_t smem = static_cast<size_t>(slots) * K * 2 + static_cast<size_t>(NB) * K * 2 + 16 * slots + 16;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  // the a1 projection (writes the staging read by attention) bounds the look-ahead
  const int mode = (epi.mode == 1 ? 1 : 0) | (knob("ZDC_GEMV_NO_PREWAIT", 0) ? 2 : 0);
  prof_mark(stream, true, g_prof_class);
  cudaError_t e = launch_k(gemv_ring_kernel<NB>, dim3(blocks), dim3(288), smem, stream, g_pdl && (g_pdl_mask & 1), W,
                           x, ldx, N, K, epi,
                           mode, slots);
  prof_mark(stream, false, g_prof_class);
  ++g_launches;
  return e;
}

bool gemv_supported(int B, int K) {
  // at least one K-row slot per consumer warp plus the B input rows must fit in shared memory
  return B >= 1 && B <= 8 && K % 8 == 0 &&
         static_cast<size_t>(8) * K * 2 + static_cast<size_t>(B) * K * 2 + 16 * 8 + 16 <= 227 * 1024;
}

cudaError_t launch_gemv(const uint16_t* W, const uint16_t* x, int64_t ldx, int B, int N, int K, const Epilogue& epi,
                        cudaStream_t stream) {
  if (K % 8 != 0) return cudaErrorInvalidValue;
  switch (B) {
    case 1: return launch_gemv_nb<1>(W, x, ldx, N, K, epi, stream);
    case 2: return launch_gemv_nb<2>(W, x, ldx, N, K, epi, stream);
    case 3: return launch_gemv_nb<3>(W, x, ldx, N, K, epi, stream);
    case 4: return launch_gemv_nb<4>(W, x, ldx, N, K, epi, stream);
    case 5: return launch_gemv_nb<5>(W, x, ldx, N, K, epi, stream);
    case 6: return launch_gemv_nb<6>(W, x, ldx, N, K, epi, stream);
    case 7: return launch_gemv_nb<7>(W, x, ldx, N, K, epi, stream);
    case 8: return launch_gemv_nb<8>(W, x, ldx, N, K, epi, stream);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------ decode attention
static constexpr int kMaxChunk = 512;
static constexpr float kLog2e = 1.4426950408889634f;

__host__ __device__ constexpr int pow2_at_least(int x) { return x <= 1 ? 1 : x <= 2 ? 2 : x <= 4 ? 4 : x <= 8 ? 8 : 16; }

// One CTA per (chunk, KV head, sequence) of ONE pool (pool 0 = important / uniform rows at
// width RK/RV, pool 1 = unimportant rows at their truncated width; the query is used at the
// pool's width, which is exact because the truncated dims of pool-1 keys are zero, P:776 DEL).
// Writes an unnormalised partial (o[0..RVO), m, l) to slot `slot0 + chunk`; o[c] = 0 for c >= RV.
template <int RK, int RV, int G>
__global__ void __launch_bounds__(128) decode_attn_partial(const DecodeAttnArgs a, const uint16_t* __restrict__ kp,
                                                           const uint16_t* __restrict__ vp, int pool, int slot0,
                                                           int nslots) {
  constexpr int UK = RK / 8;                                            // 16-byte chunks per K' row
  constexpr int UV = RV / 8, UVP = pow2_at_least(UV), RPWV = 32 / UVP;  // lanes per V' row (padded)
  __shared__ float sc[G][kMaxChunk];
  __shared__ float red[4][G][RV];
  __shared__ float stat[2][4][G];
  __shared__ int s_last;
  const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (static_cast<int64_t>(b) * a.Nkv + g) * a.S_cap;
  const float scl = a.scale * kLog2e;
  // the chunk's K'/V' rows (contiguous in the cache) are staged in shared memory by two bulk copies
  extern __shared__ __align__(128) uint8_t dsm[];
  const int cmax = (a.len + a.splits - 1) / a.splits;
  uint16_t* Ks = reinterpret_cast<uint16_t*>(dsm);
  uint16_t* Vs = Ks + static_cast<size_t>(cmax) * RK;
  uint64_t* kvbar = reinterpret_cast<uint64_t*>(Vs + static_cast<size_t>(cmax) * RV);  // [0] cached, [1] rest
  pdl_trigger();
  if (threadIdx.x == 0) {
    mbar_init(&kvbar[0], 1);
    mbar_init(&kvbar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const bool uniform = a.n0_ptr == nullptr;
  int pre = 0;  // rows staged in shared memory before the dependency wait
  if (uniform && a.prefetch_before_wait) {
    // uniform cache: the length is final before the predecessor (the a1 projection) runs, so every
    // cached row of the chunk can stream in while it finishes (the new row is excluded):
    // mode 2 stages them straight into shared memory, mode 1 only into L2.
    const int len0 = a.len_ptr ? min(*a.len_ptr + 1, a.S_cap) : a.len;
    const int ch0 = (len0 + a.splits - 1) / a.splits;
    const int p0 = split * ch0;
    const int np = max(0, min(min(len0, p0 + ch0), len0 - 1) - p0);
    if (a.prefetch_before_wait == 2) {
      pre = np;
      if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&kvbar[0], static_cast<uint32_t>(np) * (RK + RV) * 2u);
        if (np > 0) {
          bulk_g2s(Ks, kp + (row0 + p0) * RK, static_cast<uint32_t>(np) * RK * 2u, &kvbar[0]);
          bulk_g2s(Vs, vp + (row0 + p0) * RV, static_cast<uint32_t>(np) * RV * 2u, &kvbar[0]);
        }
      }
    } else if (threadIdx.x == 0 && np > 0) {
      l2_prefetch(kp + (row0 + p0) * RK, static_cast<uint32_t>(np) * RK * 2u);
      l2_prefetch(vp + (row0 + p0) * RV, static_cast<uint32_t>(np) * RV * 2u);
    }
  }
  if (threadIdx.x == 32 && pool == 0) {
    // read-only weights of the following kernels -> L2 (this kernel's own rows were issued first)
    const int64_t ncta = static_cast<int64_t>(gridDim.x) * gridDim.y * gridDim.z;
    const int64_t cta = (static_cast<int64_t>(b) * gridDim.y + g) * gridDim.x + split;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (a.pf_bytes[i] <= 0) continue;
      const int64_t per = ((a.pf_bytes[i] + ncta - 1) / ncta + 15) & ~int64_t(15);
      const int64_t lo = cta * per, hi = min(a.pf_bytes[i], lo + per);
      for (int64_t o = lo; o < hi; o += 32768)
        l2_prefetch(static_cast<const uint8_t*>(a.pf_ptr[i]) + o, static_cast<uint32_t>(min(static_cast<int64_t>(32768), hi - o)));
    }
  }
  pdl_wait();
  int len;
  if (pool == 0)
    len = a.n0_ptr ? a.n0_ptr[b] : (a.len_ptr ? min(*a.len_ptr + 1, a.S_cap) : a.len);
  else
    len = a.n1_ptr[b];
  const int chunk = (len + a.splits - 1) / a.splits;
  const int s0 = split * chunk;
  const int s1 = min(len, s0 + chunk);
  const int n = max(0, s1 - s0);
  if (threadIdx.x == 0) {
    if (!(uniform && a.prefetch_before_wait == 2)) mbar_arrive_expect_tx(&kvbar[0], 0);
    const int rest = n - pre;
    mbar_arrive_expect_tx(&kvbar[1], static_cast<uint32_t>(max(rest, 0)) * (RK + RV) * 2u);
    if (rest > 0) {
      bulk_g2s(Ks + static_cast<size_t>(pre) * RK, kp + (row0 + s0 + pre) * RK, static_cast<uint32_t>(rest) * RK * 2u,
               &kvbar[1]);
      bulk_g2s(Vs + static_cast<size_t>(pre) * RV, vp + (row0 + s0 + pre) * RV, static_cast<uint32_t>(rest) * RV * 2u,
               &kvbar[1]);
    }
  }
  mbar_wait(&kvbar[0], 0);
  mbar_wait(&kvbar[1], 0);

  // ---- scores s = q . k * scale * log2(e): one thread per key row, all G heads of the group
  // per row.  q sits in shared memory as f32; each thread visits the 16-byte chunks of its row in
  // a rotated order ((k + j) mod UK), so the 32 rows a warp reads hit distinct banks.
  {
    __shared__ __align__(16) float qsf[G][RK];
    for (int i = threadIdx.x; i < G * UK; i += 128) {
      const int gi = i / UK, u = i - gi * UK;
      float f[8];
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(a.q + b * a.ldq + (g * G + gi) * a.rk + u * 8), f);
#pragma unroll
      for (int e = 0; e < 8; ++e) qsf[gi][u * 8 + e] = f[e];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += 128) {
      float acc[G];
#pragma unroll
      for (int gi = 0; gi < G; ++gi) acc[gi] = 0.f;
      const int rot = j % UK;
#pragma unroll
      for (int k = 0; k < UK; ++k) {
        int kc = k + rot;
        if (kc >= UK) kc -= UK;
        float kf[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(Ks + static_cast<size_t>(j) * RK + kc * 8), kf);
#pragma unroll
        for (int gi = 0; gi < G; ++gi) {
          const float4 q0 = *reinterpret_cast<const float4*>(&qsf[gi][kc * 8]);
          const float4 q1 = *reinterpret_cast<const float4*>(&qsf[gi][kc * 8 + 4]);
          acc[gi] = fmaf(q0.x, kf[0], acc[gi]);
          acc[gi] = fmaf(q0.y, kf[1], acc[gi]);
          acc[gi] = fmaf(q0.z, kf[2], acc[gi]);
          acc[gi] = fmaf(q0.w, kf[3], acc[gi]);
          acc[gi] = fmaf(q1.x, kf[4], acc[gi]);
          acc[gi] = fmaf(q1.y, kf[5], acc[gi]);
          acc[gi] = fmaf(q1.z, kf[6], acc[gi]);
          acc[gi] = fmaf(q1.w, kf[7], acc[gi]);
        }
      }
#pragma unroll
      for (int gi = 0; gi < G; ++gi) sc[gi][j] = acc[gi] * scl;
    }
  }
  __syncthreads();
  // ---- chunk max and exponentials (P rounded to bf16 before PV; l from the unrounded P)
  float mx[G], ls[G];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    float m = -INFINITY;
    for (int j = threadIdx.x; j < n; j += 128) m = fmaxf(m, sc[gi][j]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (lane == 0) stat[0][warp][gi] = m;
  }
  __syncthreads();
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    mx[gi] = fmaxf(fmaxf(stat[0][0][gi], stat[0][1][gi]), fmaxf(stat[0][2][gi], stat[0][3][gi]));
    float l = 0.f;
    for (int j = threadIdx.x; j < n; j += 128) {
      const float p = exp2f(sc[gi][j] - mx[gi]);
      l += p;
      sc[gi][j] = __bfloat162float(__float2bfloat16_rn(p));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    if (lane == 0) stat[1][warp][gi] = l;
  }
  __syncthreads();
#pragma unroll
  for (int gi = 0; gi < G; ++gi) ls[gi] = stat[1][0][gi] + stat[1][1][gi] + stat[1][2][gi] + stat[1][3][gi];
  // ---- o = sum_j p_j V'_j  (unnormalised, relative to the chunk max)
  {
    const int sub = lane / UVP, u = lane % UVP;
    const bool lane_on = sub < RPWV && u < UV;
    float acc[G][8];
#pragma unroll
    for (int gi = 0; gi < G; ++gi)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[gi][e] = 0.f;
#pragma unroll 4
    for (int jb = warp * RPWV; jb < n; jb += 4 * RPWV) {
      const int j = jb + sub;
      if (lane_on && j < n) {
        const uint4 vv = *reinterpret_cast<const uint4*>(Vs + static_cast<size_t>(j) * RV + u * 8);
        float vf[8];
        bf16x8_to_f32(vv, vf);
#pragma unroll
        for (int gi = 0; gi < G; ++gi) {
          const float p = sc[gi][j];
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[gi][e] = fmaf(p, vf[e], acc[gi][e]);
        }
      }
    }
#pragma unroll
    for (int gi = 0; gi < G; ++gi)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float v = acc[gi][e];
#pragma unroll
        for (int off = UVP; off < 32; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        acc[gi][e] = v;
      }
    if (sub == 0 && u < UV) {
#pragma unroll
      for (int gi = 0; gi < G; ++gi)
#pragma unroll
        for (int e = 0; e < 8; ++e) red[warp][gi][u * 8 + e] = acc[gi][e];
    }
  }
  __syncthreads();
  const int RVO = a.rv;
  for (int i = threadIdx.x; i < G * RVO; i += 128) {
    const int gi = i / RVO, c = i - gi * RVO;
    const int h = g * G + gi;
    float* dst = a.part + ((static_cast<int64_t>(b) * a.Nh + h) * nslots + slot0 + split) * (RVO + 2);
    dst[c] = c < RV ? red[0][gi][c] + red[1][gi][c] + red[2][gi][c] + red[3][gi][c] : 0.f;
    if (c == 0) {
      float m = -INFINITY, l = 0.f;
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
        if (gg == gi) m = mx[gg], l = ls[gg];
      dst[RVO] = n > 0 ? m : -INFINITY;
      dst[RVO + 1] = n > 0 ? l : 0.f;
    }
  }
  // ---- the last CTA of this (sequence, KV head) merges every partial (replaces a combine launch):
  // O' = sum_s o_s 2^(m_s - M) / sum_s l_s 2^(m_s - M), LSE = (M + log2 L) ln 2
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(&a.counters[b * a.Nkv + g], 1);
    s_last = prev == nslots - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  float* wts = &sc[0][0];  // reuse: [G][nslots] merge weights (nslots <= 128 <= kMaxChunk)
#pragma unroll 1
  for (int gi = 0; gi < G; ++gi) {
    const float* hp = a.part + ((static_cast<int64_t>(b) * a.Nh + g * G + gi) * nslots) * (RVO + 2);
    float m = threadIdx.x < nslots ? __ldcg(hp + threadIdx.x * (RVO + 2) + RVO) : -INFINITY;
    float mm = m;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, off));
    if (lane == 0) stat[0][warp][gi] = mm;
    __syncthreads();
    const float M = fmaxf(fmaxf(stat[0][0][gi], stat[0][1][gi]), fmaxf(stat[0][2][gi], stat[0][3][gi]));
    float wl = 0.f;
    if (threadIdx.x < nslots) {
      const float w = m == -INFINITY ? 0.f : exp2f(m - M);
      wts[gi * 128 + threadIdx.x] = w;
      wl = w * __ldcg(hp + threadIdx.x * (RVO + 2) + RVO + 1);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) wl += __shfl_xor_sync(0xffffffffu, wl, off);
    if (lane == 0) stat[1][warp][gi] = wl;
    __syncthreads();
    const float L = stat[1][0][gi] + stat[1][1][gi] + stat[1][2][gi] + stat[1][3][gi];
    const float inv = 1.f / L;
    for (int c = threadIdx.x; c < RVO; c += 128) {
      float o = 0.f;
#pragma unroll 8  // independent loads in flight (this merge sits on the decode critical path)
      for (int s2 = 0; s2 < nslots; ++s2) o = fmaf(wts[gi * 128 + s2], __ldcg(hp + s2 * (RVO + 2) + c), o);
      a.o[b * a.ldo + (g * G + gi) * RVO + c] = f32_to_bf16_bits(o * inv);
    }
    if (threadIdx.x == 0 && a.lse) a.lse[b * a.Nh + g * G + gi] = (M + log2f(L)) / kLog2e;
  }
  if (threadIdx.x == 0) a.counters[b * a.Nkv + g] = 0;
}

int decode_splits(int B, int Nkv, int len) {
  const int pairs = B * Nkv;
  int s = (2 * num_sms() + pairs - 1) / pairs;     // ~2 CTAs per SM
  // a chunk's K'/V' rows are staged in shared memory: <= 300 rows (150 KB at width 128)
  constexpr int kMaxStagedRows = 300;
  const int min_for_smem = (len + kMaxStagedRows - 1) / kMaxStagedRows;
  const int max_useful = (len + 31) / 32;            // >= 32 keys per chunk
  if (s > max_useful) s = max_useful;
  if (s < min_for_smem) s = min_for_smem;
  if (s > 64) s = 64;
  if (s < 1) s = 1;
  return s;
}

template <int RK, int G>
static void launch_partial_t(const DecodeAttnArgs& a, const uint16_t* kp, const uint16_t* vp, int pool, int slot0,
                             int nslots, cudaStream_t stream) {
  dim3 grid(a.splits, a.Nkv, a.B);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_attn_partial<RK, RK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  const int cmax = (a.len + a.splits - 1) / a.splits;
  const size_t smem = static_cast<size_t>(cmax) * (RK + RK) * 2 + 16;
  launch_k(decode_attn_partial<RK, RK, G>, grid, dim3(128), smem, stream, g_pdl && (g_pdl_mask & 2), a, kp, vp, pool,
           slot0, nslots);
}

template <int G>
static cudaError_t launch_partial_g(const DecodeAttnArgs& a, int width, const uint16_t* kp, const uint16_t* vp,
                                    int pool, int slot0, int nslots, cudaStream_t stream) {
  switch (width) {
    case 16: launch_partial_t<16, G>(a, kp, vp, pool, slot0, nslots, stream); break;
    case 32: launch_partial_t<32, G>(a, kp, vp, pool, slot0, nslots, stream); break;
    case 48: launch_partial_t<48, G>(a, kp, vp, pool, slot0, nslots, stream); break;
    case 64: launch_partial_t<64, G>(a, kp, vp, pool, slot0, nslots, stream); break;
    case 80: launch_partial_t<80, G>(a, kp, vp, pool, slot0, nslots, stream); break;
    case 96: launch_partial_t<96, G>(a, kp, vp, pool, slot0, nslots, stream); break;
    case 112: launch_partial_t<112, G>(a, kp, vp, pool, slot0, nslots, stream); break;
    case 128: launch_partial_t<128, G>(a, kp, vp, pool, slot0, nslots, stream); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

static cudaError_t launch_partial(const DecodeAttnArgs& a, int width, const uint16_t* kp, const uint16_t* vp, int pool,
                                  int slot0, int nslots, cudaStream_t stream) {
  switch (a.Nh / a.Nkv) {
    case 1: return launch_partial_g<1>(a, width, kp, vp, pool, slot0, nslots, stream);
    case 2: return launch_partial_g<2>(a, width, kp, vp, pool, slot0, nslots, stream);
    case 4: return launch_partial_g<4>(a, width, kp, vp, pool, slot0, nslots, stream);
    case 8: return launch_partial_g<8>(a, width, kp, vp, pool, slot0, nslots, stream);
    default: return cudaErrorInvalidValue;
  }
}

// v2 (decode_attn2.cu) is opt-in (ZDC_DEC_ATTN_V2=1): measured 12.3 us vs 11.3 us for v1 at the
// c2 shape in round 1 (profiles/r01/NOTES.md)
// v2 (decode_attn2.cu) is the default for the separate-kernel decode path (B > 8, token-split
// layers): 8-warp pipelined CTAs, ~30 % faster than v1 at config 3 (profiles/r01/NOTES.md);
// ZDC_DEC_ATTN_V2=0 selects v1
static const bool g_dec_attn_v2 = knob("ZDC_DEC_ATTN_V2", 1) != 0;
static bool v2_width(int w) { return w == 32 || w == 64 || w == 96 || w == 128; }

static const bool g_dec_attn_v3 = knob("ZDC_DEC_ATTN_V3", 1) != 0;
cudaError_t launch_decode_attention(const DecodeAttnArgs& a_in, cudaStream_t stream) {
  // v3 (decode_attn3.cu): the byte-balanced flat split, both pools in one launch -- for token-split
  // layers and for at least one (sequence, KV head) pair per SM; with fewer pairs (e.g. B = 1,
  // 32 heads) its warps' shares are a few tiles each and v2's per-split CTAs are faster
  // (21.2 vs 12.4 us at the c2 shape)
  if (g_dec_attn_v3 && decode3_supported(a_in) && (a_in.k1 || a_in.B * a_in.Nkv >= num_sms())) {
    const cudaError_t e3 = launch_decode_attention3(a_in, stream);
    if (e3 != cudaErrorNotSupported) return e3;
    cudaGetLastError();  // shape outside v3's shared-memory budget: v2 below
  }
  if (g_dec_attn_v2 && v2_width(a_in.rk) && (!a_in.k1 || v2_width(a_in.rk1)) && a_in.rk == a_in.rv &&
      (!a_in.k1 || a_in.rk1 == a_in.rv1) && a_in.counters) {
    // v2 (decode_attn2.cu): 8-warp CTAs, per-warp pipelined tiles; its own split count
    DecodeAttnArgs a = a_in;
    a.splits = decode2_splits(a.B, a.Nkv, a.len, a.rk, a.Nh / a.Nkv);
    const int nslots = a.splits * (a.k1 ? 2 : 1);
    if (nslots > 128) return cudaErrorInvalidValue;
    prof_mark(stream, true, kProfAttnDecode);
    cudaError_t e = launch_decode2_partial(a, a.rk, a.k, a.v, 0, 0, nslots, stream);
    if (e == cudaSuccess && a.k1) e = launch_decode2_partial(a, a.rk1, a.k1, a.v1, 1, a.splits, nslots, stream);
    prof_mark(stream, false, kProfAttnDecode);
    g_launches += a.k1 ? 2 : 1;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  const DecodeAttnArgs& a = a_in;
  // a.len bounds the rows of either pool (graph replays may see any length up to it)
  if (a.splits > 64 || (a.len + a.splits - 1) / a.splits > kMaxChunk) return cudaErrorInvalidValue;
  if (a.rk != a.rv || (a.k1 && a.rk1 != a.rv1)) return cudaErrorInvalidValue;
  const int nslots = a.splits * (a.k1 ? 2 : 1);
  if (nslots > 128 || !a.counters) return cudaErrorInvalidValue;
  prof_mark(stream, true, kProfAttnDecode);
  cudaError_t e = launch_partial(a, a.rk, a.k, a.v, 0, 0, nslots, stream);
  if (e == cudaSuccess && a.k1) e = launch_partial(a, a.rk1, a.k1, a.v1, 1, a.splits, nslots, stream);
  prof_mark(stream, false, kProfAttnDecode);
  g_launches += a.k1 ? 2 : 1;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ weight packing (load time)
// W_qkv^T [nq + nk + nv][d]: row h*rk_p + c (c < rk) = column h*dh + c of W_Q^R (zero for c >= rk),
// then K groups, then V groups (rank rv).  W_o^T [d][ko_p]: column h*rv_p + c (c < rv) = row
// h*dh + c of W_O^R; padding columns zero.
__global__ void pack_qkv_kernel(const uint16_t* __restrict__ wq, const uint16_t* __restrict__ wk,
                                const uint16_t* __restrict__ wv, uint16_t* __restrict__ out, int d, int Nh, int Nkv,
                                int dh, int rk, int rv, int rk_p, int rv_p) {
  const int64_t nq = static_cast<int64_t>(Nh) * rk_p, nk = static_cast<int64_t>(Nkv) * rk_p,
                nv = static_cast<int64_t>(Nkv) * rv_p;
  const int64_t total = (nq + nk + nv) * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = i / d;
    const int k = static_cast<int>(i - n * d);
    uint16_t val = 0;
    if (n < nq) {
      const int h = static_cast<int>(n / rk_p), c = static_cast<int>(n % rk_p);
      if (c < rk) val = wq[static_cast<int64_t>(k) * Nh * dh + h * dh + c];
    } else if (n < nq + nk) {
      const int g = static_cast<int>((n - nq) / rk_p), c = static_cast<int>((n - nq) % rk_p);
      if (c < rk) val = wk[static_cast<int64_t>(k) * Nkv * dh + g * dh + c];
    } else {
      const int g = static_cast<int>((n - nq - nk) / rv_p), c = static_cast<int>((n - nq - nk) % rv_p);
      if (c < rv) val = wv[static_cast<int64_t>(k) * Nkv * dh + g * dh + c];
    }
    out[i] = val;
  }
}

__global__ void pack_o_kernel(const uint16_t* __restrict__ wo, uint16_t* __restrict__ out, int d, int Nh, int dh,
                              int rv, int rv_p, int ko_p) {
  const int64_t total = static_cast<int64_t>(d) * ko_p;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i / ko_p);
    const int col = static_cast<int>(i - static_cast<int64_t>(j) * ko_p);
    const int h = col / rv_p, c = col - h * rv_p;
    uint16_t val = 0;
    if (h < Nh && c < rv) val = wo[static_cast<int64_t>(h * dh + c) * d + j];
    out[i] = val;
  }
}

cudaError_t launch_pack_weights_bf16(const uint16_t* wq, const uint16_t* wk, const uint16_t* wv, const uint16_t* wo,
                                     uint16_t* wqkv_t, uint16_t* wo_t, int d, int Nh, int Nkv, int dh, int rk, int rv,
                                     int rk_p, int rv_p, int ko_p, cudaStream_t stream) {
  pack_qkv_kernel<<<4 * num_sms(), 256, 0, stream>>>(wq, wk, wv, wqkv_t, d, Nh, Nkv, dh, rk, rv, rk_p, rv_p);
  pack_o_kernel<<<4 * num_sms(), 256, 0, stream>>>(wo, wo_t, d, Nh, dh, rv, rv_p, ko_p);
  return cudaGetLastError();
}

}  // namespace zdc
