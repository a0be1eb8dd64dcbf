// decode_attn2.cu — a3 for token generation, v2 (the default): split-K "flash decoding" over the
// compressed cache, restructured after the round-1 measurement (v1: 24% of HBM, one long serial
// chain of phases per CTA):
//   * one CTA (kNW = 4 warps) per (split, KV head, sequence), as many splits as fill ONE wave of
//     the occupancy-limited CTA slots; each warp streams its own slice of rows in
//     32-row tiles through a private 2-stage shared-memory ring filled by cp.async.bulk (per-warp
//     mbarriers: no block-wide syncs in the main loop), so load and compute overlap per warp;
//   * lane j scores row j of the tile for all G query heads of the KV group (GQA, reading c4);
//     online softmax per warp (running max / sum), P rounded to bf16 before PV;
//   * PV: each lane owns RV/32 output columns, p_j broadcast by shuffle;
//   * the 8 warp partials merge in shared memory, the CTA writes one partial, and the last CTA of
//     the (sequence, KV head) LSE-merges the splits (O' bf16 + LSE f32).
// Same arguments and partial layout as v1 (decode.cu), so both pools of the token split work.
#include <cuda_fp8.h>

#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace zdc {

static constexpr float kLog2eD = 1.4426950408889634f;
static constexpr int kNW = 4;  // warps per CTA

__device__ __forceinline__ void bf16x8_f32(uint4 v, float (&f)[8]) {
  f[0] = __uint_as_float(v.x << 16);
  f[1] = __uint_as_float(v.x & 0xFFFF0000u);
  f[2] = __uint_as_float(v.y << 16);
  f[3] = __uint_as_float(v.y & 0xFFFF0000u);
  f[4] = __uint_as_float(v.z << 16);
  f[5] = __uint_as_float(v.z & 0xFFFF0000u);
  f[6] = __uint_as_float(v.w << 16);
  f[7] = __uint_as_float(v.w & 0xFFFF0000u);
}

template <int RK, int RV>
struct DA2 {
  static constexpr int TR = 32;                 // rows per tile (lane j <-> row j)
  static constexpr int UK = RK / 8;             // 16-byte units per K' row
  static constexpr int CPL = RV / 32 > 0 ? RV / 32 : 1;  // output columns per lane (RV >= 32)
  static constexpr uint32_t KT = TR * RK * 2, VT = TR * RV * 2;  // bytes of one K / V tile
  static constexpr uint32_t STAGE = KT + VT;
  static constexpr int NST = RK <= 96 ? 2 : 1;                    // ring stages per warp
  static constexpr uint32_t WARP_BYTES = NST * STAGE;
};

template <int RK, int RV, int G>
__global__ void __launch_bounds__(kNW * 32)
    decode_attn2_kernel(const DecodeAttnArgs a, const uint16_t* __restrict__ kp, const uint16_t* __restrict__ vp,
                        int pool, int slot0, int nslots) {
  using C = DA2<RK, RV>;
  static_assert(RV % 32 == 0 || RV == 16, "RV must be a multiple of 32 (or 16)");
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ __align__(16) float qsf[G][RK];
  __shared__ float wm[kNW][G], wl[kNW][G];
  __shared__ float wo[kNW][G][RV];
  __shared__ uint64_t bars[kNW][2];
  __shared__ int s_last;
  const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (static_cast<int64_t>(b) * a.Nkv + g) * a.S_cap;
  const float scl = a.scale * kLog2eD;
  uint8_t* ring = dsm + warp * C::WARP_BYTES;
  uint64_t* wbar = bars[warp];
  if (lane == 0) {
    mbar_init(&wbar[0], 1);
    mbar_init(&wbar[1], 1);
    fence_barrier_init();
  }
  __syncwarp();
  pdl_trigger();

  // rows of this CTA and of this warp (computed from the length; the uniform length is final
  // before the predecessor runs, so tiles below the new row can be issued before the wait)
  auto ranges = [&](int len, int& w0, int& w1) {
    const int chunk = (len + a.splits - 1) / a.splits;
    const int c0 = split * chunk, c1 = min(len, c0 + chunk);
    const int per = (max(0, c1 - c0) + kNW - 1) / kNW;
    w0 = c0 + warp * per;
    w1 = min(c1, w0 + per);
    if (w1 < w0) w1 = w0;
  };
  // tile t of this warp -> ring stage: rows [r0, min(r0 + TR, w1)) only (never past the range)
  auto issue = [&](int t, int w0, int w1, int stage) {
    const int r0 = w0 + t * C::TR;
    const uint32_t nr = static_cast<uint32_t>(min(C::TR, w1 - r0));
    mbar_arrive_expect_tx(&wbar[stage], nr * (RK + RV) * 2u);
    bulk_g2s(ring + stage * C::STAGE, kp + (row0 + r0) * RK, nr * RK * 2u, &wbar[stage]);
    bulk_g2s(ring + stage * C::STAGE + C::KT, vp + (row0 + r0) * RV, nr * RV * 2u, &wbar[stage]);
  };
  const bool uniform = a.n0_ptr == nullptr;
  int pre_tiles = 0;
  if (uniform && a.prefetch_before_wait) {
    const int len0 = a.len_ptr ? min(*a.len_ptr + 1, a.S_cap) : a.len;
    int w0, w1;
    ranges(len0, w0, w1);
    const int ntile = (w1 - w0 + C::TR - 1) / C::TR;
    // tiles that end before the new row (position len0 - 1) do not depend on the predecessor
    for (int t = 0; t < min(ntile, C::NST); ++t)
      if (w0 + (t + 1) * C::TR <= min(w1, len0 - 1)) pre_tiles = t + 1;
    if (lane == 0)
      for (int t = 0; t < pre_tiles; ++t) issue(t, w0, w1, t);
  }
  pdl_wait();
  int len;
  if (pool == 0)
    len = a.n0_ptr ? a.n0_ptr[b] : (a.len_ptr ? min(*a.len_ptr + 1, a.S_cap) : a.len);
  else
    len = a.n1_ptr[b];
  int w0, w1;
  ranges(len, w0, w1);
  const int ntile = (w1 - w0 + C::TR - 1) / C::TR;
  if (lane == 0)
    for (int t = pre_tiles; t < min(ntile, C::NST); ++t) issue(t, w0, w1, t);
  // q of the G heads of this KV group, as f32 in shared memory
  for (int i = threadIdx.x; i < G * C::UK; i += kNW * 32) {
    const int gi = i / C::UK, u = i - gi * C::UK;
    float f[8];
    bf16x8_f32(*reinterpret_cast<const uint4*>(a.q + b * a.ldq + (g * G + gi) * a.rk + u * 8), f);
#pragma unroll
    for (int e = 0; e < 8; ++e) qsf[gi][u * 8 + e] = f[e];
  }
  __syncthreads();

  float m[G], l[G], o[G][C::CPL];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    m[gi] = -INFINITY;
    l[gi] = 0.f;
#pragma unroll
    for (int c = 0; c < C::CPL; ++c) o[gi][c] = 0.f;
  }
  for (int t = 0; t < ntile; ++t) {
    const int stage = t % C::NST;
    mbar_wait(&wbar[stage], (t / C::NST) & 1);
    const uint16_t* Kt = reinterpret_cast<const uint16_t*>(ring + stage * C::STAGE);
    const uint16_t* Vt = reinterpret_cast<const uint16_t*>(ring + stage * C::STAGE + C::KT);
    const int nr = min(C::TR, w1 - (w0 + t * C::TR));  // rows of this tile (warp-uniform)
    const bool valid = lane < nr;
    // ---- scores: lane = row, chunks in rotated order (conflict-free smem)
    float s[G];
#pragma unroll
    for (int gi = 0; gi < G; ++gi) s[gi] = 0.f;
#pragma unroll
    for (int k = 0; k < C::UK; ++k) {
      int kc = k + (lane % C::UK);
      if (kc >= C::UK) kc -= C::UK;
      float kf[8];
      bf16x8_f32(valid ? *reinterpret_cast<const uint4*>(Kt + lane * RK + kc * 8) : make_uint4(0, 0, 0, 0), kf);
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        const float4 q0 = *reinterpret_cast<const float4*>(&qsf[gi][kc * 8]);
        const float4 q1 = *reinterpret_cast<const float4*>(&qsf[gi][kc * 8 + 4]);
        s[gi] = fmaf(q0.x, kf[0], s[gi]);
        s[gi] = fmaf(q0.y, kf[1], s[gi]);
        s[gi] = fmaf(q0.z, kf[2], s[gi]);
        s[gi] = fmaf(q0.w, kf[3], s[gi]);
        s[gi] = fmaf(q1.x, kf[4], s[gi]);
        s[gi] = fmaf(q1.y, kf[5], s[gi]);
        s[gi] = fmaf(q1.z, kf[6], s[gi]);
        s[gi] = fmaf(q1.w, kf[7], s[gi]);
      }
    }
    // ---- online softmax per head (warp-wide), P rounded to bf16 before PV, l from unrounded P
    float pb[G];
#pragma unroll
    for (int gi = 0; gi < G; ++gi) {
      const float x = valid ? s[gi] * scl : -INFINITY;
      float tm = x;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, off));
      const float mn = fmaxf(m[gi], tm);
      const float alpha = exp2f(m[gi] - mn);  // 0 on the first tile
      const float p = valid ? exp2f(x - mn) : 0.f;
      float ps = p;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
      l[gi] = l[gi] * alpha + ps;
      m[gi] = mn;
#pragma unroll
      for (int c = 0; c < C::CPL; ++c) o[gi][c] *= alpha;
      pb[gi] = __bfloat162float(__float2bfloat16_rn(p));
    }
    // ---- PV: lane owns columns lane*CPL .. +CPL-1
#pragma unroll 8
    for (int j = 0; j < nr; ++j) {  // only the rows copied into this stage
      float vf[C::CPL];
      if constexpr (C::CPL == 2) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(Vt + j * RV + lane * 2);
        vf[0] = __uint_as_float(w << 16);
        vf[1] = __uint_as_float(w & 0xFFFF0000u);
      } else if constexpr (C::CPL == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(Vt + j * RV + lane * 4);
        vf[0] = __uint_as_float(w.x << 16);
        vf[1] = __uint_as_float(w.x & 0xFFFF0000u);
        vf[2] = __uint_as_float(w.y << 16);
        vf[3] = __uint_as_float(w.y & 0xFFFF0000u);
      } else {
#pragma unroll
        for (int c = 0; c < C::CPL; ++c) {
          const int col = lane * C::CPL + c;
          vf[c] = col < RV ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(Vt)[j * RV + col]) : 0.f;
        }
      }
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        const float pj = __shfl_sync(0xffffffffu, pb[gi], j);
#pragma unroll
        for (int c = 0; c < C::CPL; ++c) o[gi][c] = fmaf(pj, vf[c], o[gi][c]);
      }
    }
    __syncwarp();
    // refill this stage with tile t + NST
    if (lane == 0 && t + C::NST < ntile) issue(t + C::NST, w0, w1, stage);
  }
  // ---- merge the 8 warp partials of this CTA in shared memory
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    if (lane == 0) {
      wm[warp][gi] = m[gi];
      wl[warp][gi] = l[gi];
    }
#pragma unroll
    for (int c = 0; c < C::CPL; ++c)
      if (lane * C::CPL + c < RV) wo[warp][gi][lane * C::CPL + c] = o[gi][c];
  }
  __syncthreads();
  const int RVO = a.rv;
  for (int i = threadIdx.x; i < G * RVO; i += kNW * 32) {
    const int gi = i / RVO, c = i - gi * RVO;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kNW; ++w) M = fmaxf(M, wm[w][gi]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kNW; ++w) {
      const float f = wm[w][gi] == -INFINITY ? 0.f : exp2f(wm[w][gi] - M);
      L += f * wl[w][gi];
      if (c < RV) O += f * wo[w][gi][c];
    }
    float* dst = a.part + ((static_cast<int64_t>(b) * a.Nh + g * G + gi) * nslots + slot0 + split) * (RVO + 2);
    dst[c] = c < RV ? O : 0.f;
    if (c == 0) {
      dst[RVO] = M;
      dst[RVO + 1] = L;
    }
  }
  // ---- the last CTA of this (sequence, KV head) merges the splits (and both pools)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(&a.counters[b * a.Nkv + g], 1);
    s_last = prev == nslots - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // (m, l) of every slot: one parallel load into shared memory (the ring is free now), then the
  // per-head max and merge weights; the o loads below are independent (8 in flight per thread)
  float* sm_m = reinterpret_cast<float*>(dsm);         // [G][nslots]
  float* sm_l = sm_m + G * nslots;                      // [G][nslots]
  for (int i = threadIdx.x; i < G * nslots; i += kNW * 32) {
    const int gi = i / nslots, s2 = i - gi * nslots;
    const float* hp = a.part + ((static_cast<int64_t>(b) * a.Nh + g * G + gi) * nslots + s2) * (RVO + 2);
    sm_m[i] = __ldcg(hp + RVO);
    sm_l[i] = __ldcg(hp + RVO + 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * RVO; i += kNW * 32) {
    const int gi = i / RVO, c = i - gi * RVO;
    const float* hp = a.part + ((static_cast<int64_t>(b) * a.Nh + g * G + gi) * nslots) * (RVO + 2);
    float M = -INFINITY;
    for (int s2 = 0; s2 < nslots; ++s2) M = fmaxf(M, sm_m[gi * nslots + s2]);
    float L = 0.f, O = 0.f;
#pragma unroll 8
    for (int s2 = 0; s2 < nslots; ++s2) {
      const float ms = sm_m[gi * nslots + s2];
      const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
      L = fmaf(f, sm_l[gi * nslots + s2], L);
      O = fmaf(f, __ldcg(hp + s2 * (RVO + 2) + c), O);
    }
    __nv_bfloat16 ob = __float2bfloat16_rn(O / L);
    a.o[b * a.ldo + (g * G + gi) * RVO + c] = *reinterpret_cast<uint16_t*>(&ob);
    if (c == 0 && a.lse) a.lse[b * a.Nh + g * G + gi] = (M + log2f(L)) / kLog2eD;
  }
  if (threadIdx.x == 0) a.counters[b * a.Nkv + g] = 0;
}

// ---- NEXT-4: the same kernel over an FP8 E4M3 cache (GEAR-ZDC, reading c23).  A cached row is
// r codes, its f32 scale and 12 pad bytes (RB = r + 16 bytes, 16-byte aligned for the bulk
// copies); scores use the codes, scaled once per row: s = (q . code_k) * scale_k; PV folds the
// row's V scale into the rounded probability: o += (bf16(p) * scale_v) * code_v.
// Static shared memory of one FP8 CTA.
template <int G, int RMAX>
struct DA2Smem {
  __align__(16) float qsf[G][RMAX];
  float wm[kNW][G], wl[kNW][G];
  float wo[kNW][G][RMAX];
  uint64_t bars[kNW][4];  // one mbarrier per ring stage of each warp (NST <= 4)
  int s_last;
};

template <int RK>
struct DA2F8 {
  static constexpr int TR = 32, RB = RK + 16;
  static constexpr int CPL = RK / 32;
  static constexpr uint32_t KT = TR * RB, VT = TR * RB, STAGE = KT + VT;
  static constexpr int NST = 2;  // 4 stages (and one wave of this kernel's own occupancy) measured slower
  static constexpr uint32_t WARP_BYTES = NST * STAGE;
};

__device__ __forceinline__ float e4m3_to_f32(uint32_t code) {
  const __half_raw h = __nv_cvt_fp8_to_halfraw(static_cast<__nv_fp8_storage_t>(code), __NV_E4M3);
  return __half2float(__half(h));
}
// two E4M3 codes (low 16 bits of w) -> two floats (one packed conversion)
__device__ __forceinline__ float2 e4m3x2_to_f32x2(uint32_t w) {
  const __half2_raw h = __nv_cvt_fp8x2_to_halfraw2(static_cast<__nv_fp8x2_storage_t>(w & 0xFFFFu), __NV_E4M3);
  return __half22float2(__half2(h));
}

template <int RK, int G>
__global__ void __launch_bounds__(kNW * 32)
    decode_attn2_f8_kernel(const DecodeAttnArgs a, const uint8_t* __restrict__ kp, const uint8_t* __restrict__ vp) {
  using C = DA2F8<RK>;
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ DA2Smem<G, RK> sh;
  const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (static_cast<int64_t>(b) * a.Nkv + g) * a.S_cap;
  const float scl = a.scale * kLog2eD;
  uint8_t* ring = dsm + warp * C::WARP_BYTES;
  uint64_t* wbar = sh.bars[warp];
  static_assert(C::NST <= 4, "one mbarrier per stage");
  if (lane == 0) {
    for (int i = 0; i < C::NST; ++i) mbar_init(&wbar[i], 1);
    fence_barrier_init();
  }
  __syncwarp();
  pdl_trigger();
  pdl_wait();
  const int len = a.len_ptr ? min(*a.len_ptr + 1, a.S_cap) : a.len;
  const int chunk = (len + a.splits - 1) / a.splits;
  const int c0 = split * chunk, c1 = min(len, c0 + chunk);
  const int per = (max(0, c1 - c0) + kNW - 1) / kNW;
  const int w0 = c0 + warp * per, w1 = max(w0, min(c1, w0 + per));
  const int ntile = (w1 - w0 + C::TR - 1) / C::TR;
  auto issue = [&](int t, int stage) {
    const int r0 = w0 + t * C::TR;
    const uint32_t nr = static_cast<uint32_t>(min(C::TR, w1 - r0));
    mbar_arrive_expect_tx(&wbar[stage], nr * 2u * C::RB);
    bulk_g2s(ring + stage * C::STAGE, kp + (row0 + r0) * C::RB, nr * C::RB, &wbar[stage]);
    bulk_g2s(ring + stage * C::STAGE + C::KT, vp + (row0 + r0) * C::RB, nr * C::RB, &wbar[stage]);
  };
  if (lane == 0)
    for (int t = 0; t < min(ntile, C::NST); ++t) issue(t, t);
  for (int i = threadIdx.x; i < G * (RK / 8); i += kNW * 32) {
    const int gi = i / (RK / 8), u = i - gi * (RK / 8);
    float f[8];
    bf16x8_f32(*reinterpret_cast<const uint4*>(a.q + b * a.ldq + (g * G + gi) * a.rk + u * 8), f);
#pragma unroll
    for (int e = 0; e < 8; ++e) sh.qsf[gi][u * 8 + e] = f[e];
  }
  __syncthreads();
  float m[G], l[G], o[G][C::CPL];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    m[gi] = -INFINITY;
    l[gi] = 0.f;
#pragma unroll
    for (int c = 0; c < C::CPL; ++c) o[gi][c] = 0.f;
  }
  for (int t = 0; t < ntile; ++t) {
    const int stage = t % C::NST;
    mbar_wait(&wbar[stage], (t / C::NST) & 1);
    const uint8_t* Kt = ring + stage * C::STAGE;
    const uint8_t* Vt = Kt + C::KT;
    const int nr = min(C::TR, w1 - (w0 + t * C::TR));
    const bool valid = lane < nr;
    float s[G];
#pragma unroll
    for (int gi = 0; gi < G; ++gi) s[gi] = 0.f;
    if (valid) {
      const uint8_t* kr = Kt + lane * C::RB;
#pragma unroll
      for (int k = 0; k < RK / 16; ++k) {
        int kc = k + (lane % (RK / 16));
        if (kc >= RK / 16) kc -= RK / 16;
        const uint4 u = *reinterpret_cast<const uint4*>(kr + kc * 16);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const float2 kf = e4m3x2_to_f32x2(w[wi] >> (8 * e));
#pragma unroll
            for (int gi = 0; gi < G; ++gi) {
              s[gi] = fmaf(sh.qsf[gi][kc * 16 + wi * 4 + e], kf.x, s[gi]);
              s[gi] = fmaf(sh.qsf[gi][kc * 16 + wi * 4 + e + 1], kf.y, s[gi]);
            }
          }
        }
      }
      const float ksc = *reinterpret_cast<const float*>(kr + RK);
#pragma unroll
      for (int gi = 0; gi < G; ++gi) s[gi] *= ksc;
    }
    float pb[G];
#pragma unroll
    for (int gi = 0; gi < G; ++gi) {
      const float x = valid ? s[gi] * scl : -INFINITY;
      float tm = x;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, off));
      const float mn = fmaxf(m[gi], tm);
      const float alpha = exp2f(m[gi] - mn);
      const float p = valid ? exp2f(x - mn) : 0.f;
      float ps = p;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
      l[gi] = l[gi] * alpha + ps;
      m[gi] = mn;
#pragma unroll
      for (int c = 0; c < C::CPL; ++c) o[gi][c] *= alpha;
      pb[gi] = __bfloat162float(__float2bfloat16_rn(p));  // P rounded before PV
    }
    // o += (P * scale_v) code_v: lane owns columns lane*CPL .. +CPL-1 (scale_v folded per row)
    const float vsc_l = valid ? *reinterpret_cast<const float*>(Vt + lane * C::RB + RK) : 0.f;
#pragma unroll
    for (int gi = 0; gi < G; ++gi) pb[gi] *= vsc_l;
    for (int j = 0; j < nr; ++j) {
      float vf[C::CPL];
      if constexpr (C::CPL == 2) {
        const float2 f = e4m3x2_to_f32x2(*reinterpret_cast<const uint16_t*>(Vt + j * C::RB + lane * 2));
        vf[0] = f.x;
        vf[1] = f.y;
      } else if constexpr (C::CPL == 4) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(Vt + j * C::RB + lane * 4);
        const float2 f0 = e4m3x2_to_f32x2(w), f1 = e4m3x2_to_f32x2(w >> 16);
        vf[0] = f0.x;
        vf[1] = f0.y;
        vf[2] = f1.x;
        vf[3] = f1.y;
      } else {
#pragma unroll
        for (int c = 0; c < C::CPL; ++c) vf[c] = e4m3_to_f32(Vt[j * C::RB + lane * C::CPL + c]);
      }
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        const float pj = __shfl_sync(0xffffffffu, pb[gi], j);
#pragma unroll
        for (int c = 0; c < C::CPL; ++c) o[gi][c] = fmaf(pj, vf[c], o[gi][c]);
      }
    }
    __syncwarp();
    if (lane == 0 && t + C::NST < ntile) issue(t + C::NST, stage);
  }
  // warp partials -> the CTA's partial -> the last CTA of (b, g) merges the splits (as above)
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    if (lane == 0) {
      sh.wm[warp][gi] = m[gi];
      sh.wl[warp][gi] = l[gi];
    }
#pragma unroll
    for (int c = 0; c < C::CPL; ++c) sh.wo[warp][gi][lane * C::CPL + c] = o[gi][c];
  }
  __syncthreads();
  const int nslots = a.splits;
  for (int i = threadIdx.x; i < G * RK; i += kNW * 32) {
    const int gi = i / RK, c = i - gi * RK;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kNW; ++w) M = fmaxf(M, sh.wm[w][gi]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kNW; ++w) {
      const float f = sh.wm[w][gi] == -INFINITY ? 0.f : exp2f(sh.wm[w][gi] - M);
      L += f * sh.wl[w][gi];
      O += f * sh.wo[w][gi][c];
    }
    float* dst = a.part + ((static_cast<int64_t>(b) * a.Nh + g * G + gi) * nslots + split) * (RK + 2);
    dst[c] = O;
    if (c == 0) {
      dst[RK] = M;
      dst[RK + 1] = L;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sh.s_last = atomicAdd(&a.counters[b * a.Nkv + g], 1) == nslots - 1;
  __syncthreads();
  if (!sh.s_last) return;
  __threadfence();
  for (int i = threadIdx.x; i < G * RK; i += kNW * 32) {
    const int gi = i / RK, c = i - gi * RK;
    const float* hp = a.part + ((static_cast<int64_t>(b) * a.Nh + g * G + gi) * nslots) * (RK + 2);
    float M = -INFINITY;
    for (int s2 = 0; s2 < nslots; ++s2) M = fmaxf(M, __ldcg(hp + s2 * (RK + 2) + RK));
    float L = 0.f, O = 0.f;
    for (int s2 = 0; s2 < nslots; ++s2) {
      const float ms = __ldcg(hp + s2 * (RK + 2) + RK);
      const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
      L = fmaf(f, __ldcg(hp + s2 * (RK + 2) + RK + 1), L);
      O = fmaf(f, __ldcg(hp + s2 * (RK + 2) + c), O);
    }
    __nv_bfloat16 ob = __float2bfloat16_rn(O / L);
    a.o[b * a.ldo + (g * G + gi) * RK + c] = *reinterpret_cast<uint16_t*>(&ob);
    if (c == 0 && a.lse) a.lse[b * a.Nh + g * G + gi] = (M + log2f(L)) / kLog2eD;
  }
  if (threadIdx.x == 0) a.counters[b * a.Nkv + g] = 0;
}

template <int RK, int G>
static cudaError_t launch2_f8_t(const DecodeAttnArgs& a, cudaStream_t stream) {
  using C = DA2F8<RK>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_attn2_f8_kernel<RK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kNW * C::WARP_BYTES));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  DecodeAttnArgs b = a;  // split count: the caller's (decode2_splits, the bf16 kernel's wave)
  dim3 grid(b.splits, b.Nkv, b.B);
  return launch_k(decode_attn2_f8_kernel<RK, G>, grid, dim3(kNW * 32), static_cast<size_t>(kNW * C::WARP_BYTES), stream,
                  g_pdl && (g_pdl_mask & 2), b, reinterpret_cast<const uint8_t*>(b.k),
                  reinterpret_cast<const uint8_t*>(b.v));
}

template <int G>
static cudaError_t launch2_f8_g(const DecodeAttnArgs& a, cudaStream_t s) {
  switch (a.rk) {
    case 32: return launch2_f8_t<32, G>(a, s);
    case 64: return launch2_f8_t<64, G>(a, s);
    case 96: return launch2_f8_t<96, G>(a, s);
    case 128: return launch2_f8_t<128, G>(a, s);
    default: return cudaErrorNotSupported;
  }
}

cudaError_t launch_decode2_f8(const DecodeAttnArgs& a, cudaStream_t s) {
  if (a.k1 || a.rk != a.rv || !a.counters || a.splits > 128) return cudaErrorInvalidValue;
  switch (a.Nh / a.Nkv) {
    case 1: return launch2_f8_g<1>(a, s);
    case 2: return launch2_f8_g<2>(a, s);
    case 4: return launch2_f8_g<4>(a, s);
    case 8: return launch2_f8_g<8>(a, s);
    default: return cudaErrorNotSupported;
  }
}

template <int RK, int G>
static int ctas_per_sm_t() {
  using C = DA2<RK, RK>;
  static int n = 0;
  if (n == 0) {
    cudaFuncSetAttribute(decode_attn2_kernel<RK, RK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kNW * C::WARP_BYTES));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_attn2_kernel<RK, RK, G>, kNW * 32,
                                                  static_cast<size_t>(kNW * C::WARP_BYTES));
    if (n < 1) n = 1;
  }
  return n;
}

template <int G>
static int ctas_per_sm_g(int width) {
  switch (width) {
    case 32: return ctas_per_sm_t<32, G>();
    case 64: return ctas_per_sm_t<64, G>();
    case 96: return ctas_per_sm_t<96, G>();
    default: return ctas_per_sm_t<128, G>();
  }
}

// Split count: as many CTAs as fit in ONE wave (occupancy x SMs), >= 32 rows per warp.
int decode2_splits(int B, int Nkv, int len, int width, int G) {
  static const int forced = knob("ZDC_V2_SPLITS", 0);  // A/B override
  if (forced > 0) return forced > 64 ? 64 : forced;
  int fit = 1;
  switch (G) {
    case 1: fit = ctas_per_sm_g<1>(width); break;
    case 2: fit = ctas_per_sm_g<2>(width); break;
    case 4: fit = ctas_per_sm_g<4>(width); break;
    default: fit = ctas_per_sm_g<8>(width); break;
  }
  const int pairs = B * Nkv;
  int s = fit * num_sms() / pairs;
  const int max_useful = (len + kNW * 32 - 1) / (kNW * 32);
  if (s > max_useful) s = max_useful;
  if (s > 64) s = 64;
  if (s < 1) s = 1;
  return s;
}

template <int RK, int G>
static cudaError_t launch2_t(const DecodeAttnArgs& a, const uint16_t* kp, const uint16_t* vp, int pool, int slot0,
                             int nslots, cudaStream_t stream) {
  using C = DA2<RK, RK>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_attn2_kernel<RK, RK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kNW * C::WARP_BYTES));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(a.splits, a.Nkv, a.B);
  return launch_k(decode_attn2_kernel<RK, RK, G>, grid, dim3(kNW * 32), static_cast<size_t>(kNW * C::WARP_BYTES), stream,
                  g_pdl && (g_pdl_mask & 2), a, kp, vp, pool, slot0, nslots);
}

template <int G>
static cudaError_t launch2_g(const DecodeAttnArgs& a, int width, const uint16_t* kp, const uint16_t* vp, int pool,
                             int slot0, int nslots, cudaStream_t s) {
  switch (width) {
    case 32: return launch2_t<32, G>(a, kp, vp, pool, slot0, nslots, s);
    case 64: return launch2_t<64, G>(a, kp, vp, pool, slot0, nslots, s);
    case 96: return launch2_t<96, G>(a, kp, vp, pool, slot0, nslots, s);
    case 128: return launch2_t<128, G>(a, kp, vp, pool, slot0, nslots, s);
    default: return cudaErrorNotSupported;
  }
}

// Returns cudaErrorNotSupported for widths the v2 kernel does not instantiate (16/48/80/112):
// the caller then uses v1.
cudaError_t launch_decode2_partial(const DecodeAttnArgs& a, int width, const uint16_t* kp, const uint16_t* vp,
                                   int pool, int slot0, int nslots, cudaStream_t s) {
  switch (a.Nh / a.Nkv) {
    case 1: return launch2_g<1>(a, width, kp, vp, pool, slot0, nslots, s);
    case 2: return launch2_g<2>(a, width, kp, vp, pool, slot0, nslots, s);
    case 4: return launch2_g<4>(a, width, kp, vp, pool, slot0, nslots, s);
    case 8: return launch2_g<8>(a, width, kp, vp, pool, slot0, nslots, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace zdc
