// decode_attn_tc.cu — a3 decode attention on the tensor cores (Eqs. 2-3,
// P:249-260; scale 1/sqrt(d_h), reading c2) for grouped-query layers: each KV head g serves G query
// heads, so per cached row the G dot products and the G-wide P·V are a real contraction
// (2 G r FLOP per K'/V' element pair: 8 FLOP/byte at G = 8, r = 64, about the CUDA-core FP32 ridge),
// and config 4 (Llama-2-70B, batch 64, context 8K) reads ~1.1 GB of K'/V' per layer-step.
//
// A work item is (sequence b, KV head g, key split).  Keys sit on the MMA's M dimension:
//   S^T[128 keys][16]  = K'[128 keys][r] · Q'_g[16][r]^T         (rows G..15 of Q'_g unused)
//   O^T[128][16]      += V'^T[r (M; rows >= r unused)][128 keys] · P^T[128 keys][16]
// with K' read K-major and V' MN-major straight from the cache layout (TMA, 128-byte swizzle),
// FP32 accumulators in TMEM.  Softmax: one key per thread (warps 0-3 own the 128 TMEM lanes) with
// lazy rescaling (the reference max only moves when a tile exceeds it by more than 2^8, DESIGN.md
// reading c20): a tile normally costs one barrier that ORs "some score exceeds the reference"; only
// then are the exact per-head tile maxima exchanged.  P is rounded to bf16 before PV with l taken
// from the unrounded P.  Two CTAs per SM (r = 64) keep two softmax -> PV chains in flight.  Splits of one (b, g) are LSE-merged by the last CTA to finish (no combine
// launch).  Persistent CTAs take items round-robin.  Warps: 0-3 softmax, 4 TMA producer, 5 MMA.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>

namespace zdc {

namespace {

constexpr float kLog2eT = 1.4426950408889634f;
constexpr float kLn2T = 0.6931471805599453f;
constexpr float kLazyT = 8.0f;  // log2 units

template <int HD, int ST_ = 3>
struct DTC {
  static constexpr int NCH = HD / 64;             // 64-element (128-byte swizzle) chunks of a row
  static constexpr uint32_t CHUNK = 128 * 128;    // one 128-row chunk
  static constexpr uint32_t TILE = CHUNK * NCH;   // 128 K' or V' rows
  static constexpr int ST = ST_;                  // K and V stages
  static constexpr int CPS = HD == 64 ? 2 : 1;    // CTAs per SM (two independent softmax->PV chains)
  // V stages first: the MN-major V' read at M = 128 (HD = 64) touches [stage + CHUNK, + 2 CHUNK),
  // which for the last V stage is K stage 0 (read, never used): no slack needed
  static constexpr uint32_t OFF_V = 0;
  static constexpr uint32_t OFF_K = ST * TILE;
  static constexpr uint32_t OFF_Q = OFF_K + ST * TILE;  // [NCH][16 rows x 128 B]
  static constexpr uint32_t OFF_P = OFF_Q + NCH * 2048;  // P^T [16][128 keys]: 2 chunks of 2 KB
  static constexpr uint32_t OFF_RED = OFF_P + 4096;      // [2][4 warps][16] maxima + [4][16] sums
  static constexpr uint32_t OFF_BAR = OFF_RED + 2048;
  static constexpr uint32_t SMEM = OFF_BAR + 512 + 1024;
  static constexpr uint32_t TMEM_COLS = 64;  // S^T double buffer [0, 32), O^T [32, 48)
};

__device__ __forceinline__ void softmax_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
// barrier of the 4 softmax warps that also ORs a predicate over their 128 threads
__device__ __forceinline__ bool softmax_any(bool v) {
  uint32_t r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n barrier.red.or.pred q, 1, 128, p;\n selp.u32 %0, 1, 0, q;\n}\n"
      : "=r"(r)
      : "r"(static_cast<uint32_t>(v))
      : "memory");
  return r != 0;
}

struct TcItem {
  int b, g, split, s0, n_keys, n_tiles;
};

}  // namespace

template <int HD, int G, int STG>
__global__ void __launch_bounds__(192, DTC<HD, STG>::CPS)
    decode_attn_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                          const __grid_constant__ CUtensorMap tv, const DecodeAttnArgs a) {
  using C = DTC<HD, STG>;
  constexpr int ST = C::ST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar;
  uint64_t* q_empty = bar + 1;
  uint64_t* k_full = bar + 2;
  uint64_t* k_empty = k_full + ST;
  uint64_t* v_full = k_empty + ST;
  uint64_t* v_empty = v_full + ST;
  uint64_t* s_full = v_empty + ST;  // [2]
  uint64_t* s_free = s_full + 2;    // [2]
  uint64_t* p_full = s_free + 2;
  uint64_t* pv_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);
  float* red_m = reinterpret_cast<float*>(smem + C::OFF_RED);  // [2][4][16]
  float* red_l = red_m + 2 * 4 * 16;                            // [4][16]

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < ST; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(pv_done, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Q' (written by the a1 projection) and the cache length are only read after the PDL wait
  pdl_wait();
  pdl_trigger();
  const int len1 = min(*a.len_ptr + 1, a.S_cap);  // cached rows incl. the new token's (appended by a1)
  int chunk = (len1 + a.splits - 1) / a.splits;
  chunk = (chunk + 127) / 128 * 128;
  const int n_items = a.B * a.Nkv * a.splits;
  auto item_at = [&](int k) -> TcItem {
    TcItem it;
    it.split = k % a.splits;
    const int bg = k / a.splits;
    it.g = bg % a.Nkv;
    it.b = bg / a.Nkv;
    it.s0 = it.split * chunk;
    const int e0 = min(len1, it.s0 + chunk);
    it.n_keys = e0 > it.s0 ? e0 - it.s0 : 0;
    it.n_tiles = (it.n_keys + 127) / 128;
    return it;
  };

  if (warp == 4) {
    // ------------------------------------------------ TMA producer: Q'_g, then K'/V' tiles
    if (lane == 0) {
      int gk = 0, rq = 0;
      for (int k = blockIdx.x; k < n_items; k += gridDim.x) {
        const TcItem it = item_at(k);
        if (it.n_tiles == 0) continue;
        if (rq > 0) mbar_wait(q_empty, (rq - 1) & 1);
        mbar_arrive_expect_tx(q_full, C::NCH * G * 128);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_2d(smem + C::OFF_Q + c * 2048, &tq, q_full, c * 64, it.b * a.Nh + it.g * G);
        ++rq;
        const int row0 = (it.b * a.Nkv + it.g) * a.S_cap + it.s0;
        for (int j = 0; j < it.n_tiles; ++j, ++gk) {
          const int s = gk % ST;
          const uint32_t par = ((gk / ST) & 1) ^ 1;
          mbar_wait(&k_empty[s], par);
          mbar_arrive_expect_tx(&k_full[s], C::TILE);
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_2d(smem + C::OFF_K + s * C::TILE + c * C::CHUNK, &tk, &k_full[s], c * 64, row0 + j * 128);
          mbar_wait(&v_empty[s], par);
          mbar_arrive_expect_tx(&v_full[s], C::TILE);
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_2d(smem + C::OFF_V + s * C::TILE + c * C::CHUNK, &tv, &v_full[s], c * 64, row0 + j * 128);
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------ MMA issuer: S(j+1) ahead of PV(j)
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 16, 0, 0);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, 16, 1, 0);  // A = V'^T read MN-major
      const uint32_t q_addr = smem_u32(smem + C::OFF_Q), p_addr = smem_u32(smem + C::OFF_P);
      auto issue_s = [&](int t) {
        const int s = t % ST, buf = t & 1;
        mbar_wait(&k_full[s], (t / ST) & 1);
        if (t >= 2) mbar_wait(&s_free[buf], ((t >> 1) - 1) & 1);  // the softmax read S(t-2)
        tc_fence_after();
        const uint32_t k_addr = smem_u32(smem + C::OFF_K + s * C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_ss(tmem + buf * 16, make_sdesc(k_addr + c * C::CHUNK + kk * 32, 16, 1024, kSw128),
                         make_sdesc(q_addr + c * 2048 + kk * 32, 16, 1024, kSw128), idesc_s, (c | kk) != 0 ? 1u : 0u);
        umma_commit(&s_full[buf]);
        umma_commit(&k_empty[s]);
      };
      auto issue_pv = [&](int t, bool first) {
        const int s = t % ST;
        mbar_wait(p_full, t & 1);
        mbar_wait(&v_full[s], (t / ST) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(smem + C::OFF_V + s * C::TILE);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ss(tmem + 32, make_sdesc(v_addr + kk * 16 * 128, C::CHUNK, 1024, kSw128),
                       make_sdesc(p_addr + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024, kSw128), idesc_o,
                       (first && kk == 0) ? 0u : 1u);
        umma_commit(&v_empty[s]);
        umma_commit(pv_done);
      };
      int gt = 0, rq = 0;
      for (int k = blockIdx.x; k < n_items; k += gridDim.x) {
        const TcItem it = item_at(k);
        if (it.n_tiles == 0) continue;
        mbar_wait(q_full, rq & 1);
        ++rq;
        issue_s(gt);
        for (int j = 0; j < it.n_tiles; ++j) {
          if (j + 1 < it.n_tiles) issue_s(gt + j + 1);
          issue_pv(gt + j, j == 0);
        }
        umma_commit(q_empty);  // Q'_g no longer read once these MMAs complete
        gt += it.n_tiles;
      }
    }
  } else {
    // ------------------------------------------------ softmax + epilogue: thread t = key t of a tile
    const int t = static_cast<int>(warp * 32 + lane);
    const uint32_t lane_base = (warp * 32) << 16;
    const float sl = a.scale * kLog2eT;
    int gt = 0;
    for (int k = blockIdx.x; k < n_items; k += gridDim.x) {
      const TcItem it = item_at(k);
      float m_ref[G], l_part[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        m_ref[q] = -INFINITY;
        l_part[q] = 0.f;
      }
      for (int j = 0; j < it.n_tiles; ++j) {
        const int ti = gt + j, buf = ti & 1;
        mbar_wait(&s_full[buf], (ti >> 1) & 1);
        tc_fence_after();
        uint32_t sv[16];
        tmem_ld16(tmem + lane_base + buf * 16, sv);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[buf]);
        const bool valid = j * 128 + t < it.n_keys;
        float sc[G];
        bool need = false;
#pragma unroll
        for (int q = 0; q < G; ++q) {
          sc[q] = valid ? __uint_as_float(sv[q]) * sl : -INFINITY;
          need |= sc[q] > m_ref[q] + kLazyT;
        }
        // fast path: no score of the tile exceeds the reference by more than 2^8 (one barrier with
        // an OR); otherwise the exact tile maxima decide which references rise (lazy rescaling)
        bool any_raise = false;
        float alpha[G], p[G];
#pragma unroll
        for (int q = 0; q < G; ++q) alpha[q] = 1.f;
        if (softmax_any(need)) {
#pragma unroll
          for (int q = 0; q < G; ++q) {
            float mx = sc[q];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            if (lane == 0) red_m[((ti & 1) * 4 + warp) * 16 + q] = mx;
          }
          softmax_sync();
#pragma unroll
          for (int q = 0; q < G; ++q) {
            const float* rm = red_m + (ti & 1) * 64 + q;
            const float tmax = fmaxf(fmaxf(rm[0], rm[16]), fmaxf(rm[32], rm[48]));
            if (tmax > m_ref[q] + kLazyT) {
              alpha[q] = exp2f(m_ref[q] - tmax);  // 0 on the first tile
              m_ref[q] = tmax;
              any_raise = true;
            }
          }
        }
#pragma unroll
        for (int q = 0; q < G; ++q) {
          const float mr = m_ref[q] == -INFINITY ? 0.f : m_ref[q];
          p[q] = valid ? fast_exp2(sc[q] - mr) : 0.f;
          l_part[q] = l_part[q] * alpha[q] + p[q];
        }
        // O^T and the P^T buffer are free once PV(ti - 1) has completed
        if (j > 0) {
          mbar_wait(pv_done, (ti - 1) & 1);
          tc_fence_after();
          if (any_raise && t < HD) {  // lanes >= HD of O^T are unused
            uint32_t ov[16];
            tmem_ld16(tmem + lane_base + 32, ov);
            tc_wait_ld();
#pragma unroll
            for (int q = 0; q < G; ++q) ov[q] = __float_as_uint(__uint_as_float(ov[q]) * alpha[q]);
            tmem_st16(tmem + lane_base + 32, ov);
            tc_wait_st();
          }
        }
        // P^T[q][key t] (K-major, 128-byte swizzle; keys [0,64) in chunk 0, [64,128) in chunk 1)
        uint8_t* pb = smem + C::OFF_P + (t >> 6) * 2048;
#pragma unroll
        for (int q = 0; q < G; ++q) {
          const uint32_t byte = static_cast<uint32_t>(q) * 128 + static_cast<uint32_t>(t & 63) * 2;
          *reinterpret_cast<uint16_t*>(pb + (byte ^ (((byte >> 7) & 7) << 4))) = f32_to_bf16_bits(p[q]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
      }
      // ---- epilogue: l = sum over the 128 threads; O^T column q / l -> O' (or this split's partial)
      float lq[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        float v = l_part[q];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) red_l[warp * 16 + q] = v;
      }
      softmax_sync();
#pragma unroll
      for (int q = 0; q < G; ++q) lq[q] = red_l[q] + red_l[16 + q] + red_l[32 + q] + red_l[48 + q];
      float ov[G];
#pragma unroll
      for (int q = 0; q < G; ++q) ov[q] = 0.f;
      if (it.n_tiles > 0) {
        mbar_wait(pv_done, (gt + it.n_tiles - 1) & 1);
        tc_fence_after();
        if (t < HD) {
          uint32_t r[16];
          tmem_ld16(tmem + lane_base + 32, r);
          tc_wait_ld();
#pragma unroll
          for (int q = 0; q < G; ++q) ov[q] = __uint_as_float(r[q]);
        }
        tc_fence_before();
      }
      gt += it.n_tiles;
      if (a.splits == 1) {
        if (t < HD) {
#pragma unroll
          for (int q = 0; q < G; ++q)
            a.o[it.b * a.ldo + (it.g * G + q) * HD + t] = f32_to_bf16_bits(ov[q] / lq[q]);
        }
        if (t < G && a.lse) {
#pragma unroll
          for (int q = 0; q < G; ++q)
            if (q == t) a.lse[it.b * a.Nh + it.g * G + q] = (m_ref[q] + log2f(lq[q])) * kLn2T;
        }
        softmax_sync();  // red_l is rewritten by the next item
        continue;
      }
      // split partial (m, l in log2 units; o unnormalised relative to m), then the last CTA of
      // (b, g) merges: O' = sum_s o_s 2^(m_s - M) / sum_s l_s 2^(m_s - M), LSE = (M + log2 L) ln 2
      if (t < HD) {
#pragma unroll
        for (int q = 0; q < G; ++q) {
          float* dst = a.part + ((static_cast<int64_t>(it.b) * a.Nh + it.g * G + q) * a.splits + it.split) * (HD + 2);
          dst[t] = ov[q];
          if (t == 0) {
            dst[HD] = it.n_tiles > 0 ? m_ref[q] : -INFINITY;
            dst[HD + 1] = it.n_tiles > 0 ? lq[q] : 0.f;
          }
        }
      }
      __threadfence();
      softmax_sync();
      if (t == 0) *s_flag = atomicAdd(&a.counters[it.b * a.Nkv + it.g], 1) == a.splits - 1;
      softmax_sync();
      if (*s_flag) {
        __threadfence();
        for (int i = t; i < G * HD; i += 128) {
          const int q = i / HD, c = i - q * HD;
          const float* hp = a.part + (static_cast<int64_t>(it.b) * a.Nh + it.g * G + q) * a.splits * (HD + 2);
          float M = -INFINITY;
          for (int s2 = 0; s2 < a.splits; ++s2) M = fmaxf(M, __ldcg(hp + s2 * (HD + 2) + HD));
          float O = 0.f, Ls = 0.f;
          for (int s2 = 0; s2 < a.splits; ++s2) {
            const float ms = __ldcg(hp + s2 * (HD + 2) + HD);
            const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
            O = fmaf(f, __ldcg(hp + s2 * (HD + 2) + c), O);
            Ls = fmaf(f, __ldcg(hp + s2 * (HD + 2) + HD + 1), Ls);
          }
          a.o[it.b * a.ldo + (it.g * G + q) * HD + c] = f32_to_bf16_bits(O / Ls);
          if (c == 0 && a.lse) a.lse[it.b * a.Nh + it.g * G + q] = (M + log2f(Ls)) * kLn2T;
        }
        if (t == 0) a.counters[it.b * a.Nkv + it.g] = 0;
      }
      softmax_sync();
    }
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// splits per (b, g): one whenever the (b, g) pairs alone cover the resident CTAs -- a split adds a
// Q' load, a pipeline ramp, a partial and a merge per item, which measured costlier than an
// unfilled last round (c4: 1 split 217 us, 2 splits 251 us, 4 splits 264 us per layer-step);
// otherwise the fewest that fill the persistent CTAs' last round to >= 90 % (each split keeping >= 2
// key tiles at the capacity bound)
int decode_tc_splits(int B, int Nkv, int len) {
  static const int forced = knob("ZDC_TC_SPLITS", 0);  // A/B override
  if (forced > 0) return std::min(64, forced);
  const int pairs = B * Nkv, nsm = 2 * num_sms();  // resident CTAs at r = 64 (r = 128: a bound)
  if (pairs >= nsm) return 1;
  const int max_s = std::max(1, std::min(64, (len + 255) / 256));
  for (int s = 1; s <= max_s; ++s) {
    const int items = pairs * s;
    const int rounds = (items + nsm - 1) / nsm;
    if (items >= 0.9 * rounds * nsm) return s;
  }
  return max_s;
}

bool decode_attention_tc_supported(int rk, int rv, int G) {
  return rk == rv && (rk == 64 || rk == 128) && (G == 2 || G == 4 || G == 8 || G == 16);
}

template <int HD, int G, int STG>
static cudaError_t launch_tc_s(const DecodeAttnArgs& a, cudaStream_t stream) {
  using C = DTC<HD, STG>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_attn_tc_kernel<HD, G, STG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::SMEM));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap tq, tk, tv;
  const uint64_t kv_rows = static_cast<uint64_t>(a.B) * a.Nkv * a.S_cap;
  if (!make_tmap_2d(&tq, a.q, HD, static_cast<uint64_t>(a.B) * a.Nh, HD * 2, 64, G, 128)) return cudaErrorInvalidValue;
  if (!make_tmap_2d(&tk, a.k, HD, kv_rows, HD * 2, 64, 128, 128)) return cudaErrorInvalidValue;
  if (!make_tmap_2d(&tv, a.v, HD, kv_rows, HD * 2, 64, 128, 128)) return cudaErrorInvalidValue;
  const int n_items = a.B * a.Nkv * a.splits;
  prof_mark(stream, true, kProfAttnDecode);
  cudaError_t e = launch_k(decode_attn_tc_kernel<HD, G, STG>, dim3(std::min(n_items, C::CPS * num_sms())), dim3(192), C::SMEM,
                           stream, g_pdl && (g_pdl_mask & 2), tq, tk, tv, a);
  prof_mark(stream, false, kProfAttnDecode);
  ++g_launches;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// stages per CTA (two CTAs per SM at r = 64): ZDC_TC_STAGES = 2 or 3 (default 2: c4 207.2 vs 209.0 us)
static const int g_tc_stages = knob("ZDC_TC_STAGES", 2);
template <int HD, int G>
static cudaError_t launch_tc_t(const DecodeAttnArgs& a, cudaStream_t stream) {
  return g_tc_stages == 3 ? launch_tc_s<HD, G, 3>(a, stream) : launch_tc_s<HD, G, 2>(a, stream);
}

cudaError_t launch_decode_attention_tc(const DecodeAttnArgs& a, cudaStream_t stream) {
  const int G = a.Nh / a.Nkv;
  if (!decode_attention_tc_supported(a.rk, a.rv, G) || a.k1 || !a.len_ptr || !a.counters || a.splits < 1 ||
      a.splits > 64 || a.ldq != static_cast<int64_t>(a.Nh) * a.rk)
    return cudaErrorNotSupported;
  switch (a.rk * 100 + G) {
    case 6402: return launch_tc_t<64, 2>(a, stream);
    case 6404: return launch_tc_t<64, 4>(a, stream);
    case 6408: return launch_tc_t<64, 8>(a, stream);
    case 6416: return launch_tc_t<64, 16>(a, stream);
    case 12802: return launch_tc_t<128, 2>(a, stream);
    case 12804: return launch_tc_t<128, 4>(a, stream);
    case 12808: return launch_tc_t<128, 8>(a, stream);
    case 12816: return launch_tc_t<128, 16>(a, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace zdc
