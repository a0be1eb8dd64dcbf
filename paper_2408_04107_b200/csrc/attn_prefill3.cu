// attn_prefill3.cu — a3 prefill attention, v3 (the default): same math and rounding points as v1
// (attn_prefill.cu header: Eqs. 2-3, scale 1/sqrt(d_h), LSE out), restructured after
// the round-1 ncu capture (profiles/r01) showed the softmax warps mostly waiting for S:
//   * K' and V' have independent TMA producer warps and 3-stage rings (v1's single producer
//     interleaved them, so K(j+3) waited for PV(j) to free a V slot);
//   * mbarrier arrivals are one per warp (elected lane) instead of one per thread;
//   * P is written with st.shared (not generic stores) and only diagonal tiles take the masked path;
//   * 8 softmax warps: warps w and w+4 share TMEM lane quarter w%4 and split the 128 keys of a tile.
// Warps 0-7 softmax, 8 K producer, 9 V producer, 10 MMA issuer.
#include "common.cuh"
#include "kernels.h"

namespace zdc {

static constexpr float kLog2e3 = 1.4426950408889634f;
static constexpr float kLn2_3 = 0.6931471805599453f;

template <int HD>
struct Attn3Cfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int CW = HD % 64 == 0 ? 64 : HD % 32 == 0 ? 32 : 16;
  static constexpr int NCH = HD / CW;
  static constexpr int SWB = CW * 2;
  static constexpr uint32_t LAYOUT = SWB == 128 ? kSw128 : SWB == 64 ? kSw64 : kSw32;
  static constexpr uint32_t CHUNK = BM * SWB;
  static constexpr uint32_t TILE = CHUNK * NCH;
  static constexpr uint32_t P_BYTES = BM * BN * 2;
  static constexpr int STAGES = (TILE * 7 + P_BYTES <= 200 * 1024) ? 3 : 2;
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = TILE;
  static constexpr uint32_t OFF_V = OFF_K + STAGES * TILE;
  static constexpr uint32_t OFF_P = OFF_V + STAGES * TILE;
  static constexpr uint32_t OFF_BAR = OFF_P + P_BYTES;
  static constexpr uint32_t SMEM = OFF_BAR + 256 + 1024;
  static constexpr uint32_t TMEM_COLS = 512;  // S0 [0,128) S1 [128,256) O [256, 256+HD)
  static constexpr uint32_t O_COL = 256;
};

__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

template <int HD>
__global__ void __launch_bounds__(352, 1)
    prefill_attn3_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                         const __grid_constant__ CUtensorMap tv, const PrefillAttnArgs a) {
  using C = Attn3Cfg<HD>;
  constexpr int ST = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;             // [ST]
  uint64_t* k_empty = k_full + ST;        // [ST]
  uint64_t* v_full = k_empty + ST;        // [ST]
  uint64_t* v_empty = v_full + ST;        // [ST]
  uint64_t* s_full = v_empty + ST;        // [2]
  uint64_t* s_empty = s_full + 2;         // [2]
  uint64_t* p_full = s_empty + 2;
  uint64_t* pv_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);
  __shared__ float xmax[2][2][128];  // [S buffer][half][row]
  __shared__ float xsum[2][128];

  const int n_qt = (a.n_q + C::BM - 1) / C::BM;
  const int qt = n_qt - 1 - static_cast<int>(blockIdx.x);  // heavy (long causal rows) tiles first
  const int h = blockIdx.y, b = blockIdx.z;
  const int G = a.Nh / a.Nkv, g = h / G;
  const int q0 = qt * C::BM;
  const int last_q = min(q0 + C::BM, a.n_q) - 1;
  const int n_kv = (a.q_pos0 + last_q + 1 + C::BN - 1) / C::BN;
  const int q_row = b * a.S + a.q_row0 + q0;
  auto kv_tile_row = [&](int j) -> int {
    const int pos = j * C::BN;
    if (a.kv_mode == 0) return (b * a.Nkv + g) * a.S_cap + pos;
    const int qq = pos / a.sp_chunk, rr = pos - qq * a.sp_chunk;  // SP gather buffer
    if (a.kv_mode == 2) {  // zigzag, half-major buffer [half][owner][K|V][B][Nkv][chunk][r] (overlapped exchange)
      const int h = qq < a.sp_P ? 0 : 1, ow = h == 0 ? qq : 2 * a.sp_P - 1 - qq;
      return (((h * a.sp_P + ow) * 2 * a.B + b) * a.Nkv + g) * a.sp_chunk + rr;
    }
    int owner, local;
    if (!a.sp_zigzag) {
      owner = qq;
      local = rr;
    } else {
      owner = qq < a.sp_P ? qq : 2 * a.sp_P - 1 - qq;
      local = (qq < a.sp_P ? 0 : a.sp_chunk) + rr;
    }
    return ((owner * 2 * a.B + b) * a.Nkv + g) * a.sp_n_local + local;
  };
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&tq);
      tma_prefetch_desc(&tk);
      tma_prefetch_desc(&tv);
      mbar_init(q_full, 1);
      for (int i = 0; i < ST; ++i) {
        mbar_init(&k_full[i], 1);
        mbar_init(&k_empty[i], 1);
        mbar_init(&v_full[i], 1);
        mbar_init(&v_empty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&s_full[i], 1);
        mbar_init(&s_empty[i], 8);  // one arrival per softmax warp
      }
      mbar_init(p_full, 8);
      mbar_init(pv_done, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------ K' (and Q') producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      mbar_arrive_expect_tx(q_full, C::TILE);
#pragma unroll
      for (int c = 0; c < C::NCH; ++c)
        tma_load_2d(smem + C::OFF_Q + c * C::CHUNK, &tq, q_full, h * HD + c * C::CW, q_row);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % ST;
        mbar_wait(&k_empty[s], ((j / ST) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[s], C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_2d_hint(smem + C::OFF_K + s * C::TILE + c * C::CHUNK, &tk, &k_full[s], c * C::CW,
                           kv_tile_row(j), keep);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------ V' producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % ST;
        mbar_wait(&v_empty[s], ((j / ST) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[s], C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_2d_hint(smem + C::OFF_V + s * C::TILE + c * C::CHUNK, &tv, &v_full[s], c * C::CW,
                           static_cast<int>(kv_tile_row(j) + a.v_row_off), keep);
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_s = make_idesc_bf16(C::BM, C::BN, 0, 0);
      constexpr uint32_t idesc_o = make_idesc_bf16(C::BM, HD, 0, 1);
      const uint32_t q_addr = smem_u32(smem + C::OFF_Q);
      const uint32_t p_addr = smem_u32(smem + C::OFF_P);
      auto issue_s = [&](int j) {
        const int s = j % ST, sb = j & 1;
        mbar_wait(&k_full[s], (j / ST) & 1);
        mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(smem + C::OFF_K + s * C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
#pragma unroll
          for (int kk = 0; kk < C::CW / 16; ++kk) {
            const uint64_t ad = make_sdesc(q_addr + c * C::CHUNK + kk * 32, 16, 8 * C::SWB, C::LAYOUT);
            const uint64_t bd = make_sdesc(k_addr + c * C::CHUNK + kk * 32, 16, 8 * C::SWB, C::LAYOUT);
            umma_bf16_ss(tmem + sb * 128, ad, bd, idesc_s, (c | kk) != 0 ? 1u : 0u);
          }
        umma_commit(&k_empty[s]);
        umma_commit(&s_full[sb]);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) issue_s(j + 1);
        const int s = j % ST;
        mbar_wait(p_full, j & 1);
        mbar_wait(&v_full[s], (j / ST) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(smem + C::OFF_V + s * C::TILE);
#pragma unroll
        for (int kk = 0; kk < C::BN / 16; ++kk) {
          const uint64_t ad = make_sdesc(p_addr + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, kSw128);
          const uint64_t bd = make_sdesc(v_addr + kk * 16 * C::SWB, C::CHUNK, 8 * C::SWB, C::LAYOUT);
          umma_bf16_ss(tmem + C::O_COL, ad, bd, idesc_o, (j | kk) != 0 ? 1u : 0u);
        }
        umma_commit(&v_empty[s]);
        umma_commit(pv_done);
      }
    }
  } else {
    // ------------------------------------------------ softmax warps 0..7
    const int hw = warp >> 2, qq = warp & 3;
    const int r = qq * 32 + lane;
    const int qpos = a.q_pos0 + q0 + r;
    const uint32_t lane_base = (qq * 32) << 16;
    const float sl = a.scale * kLog2e3;
    float m_run = -INFINITY, l_half = 0.f;
    const uint32_t p_base = smem_u32(smem + C::OFF_P + hw * 16384);  // this half's [128][64] chunk
    for (int j = 0; j < n_kv; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[2][32];
      tmem_ld32(tmem + lane_base + sb * 128 + hw * 64, sv[0]);
      tmem_ld32(tmem + lane_base + sb * 128 + hw * 64 + 32, sv[1]);
      tc_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      const int key0 = j * C::BN + hw * 64;
      // the warp's 32 rows cover positions [qpos(lane 0), +31]: a masked pass only on diagonal tiles
      const bool diag_warp = key0 + 63 > a.q_pos0 + q0 + qq * 32;
      if (diag_warp) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (key0 + c * 32 + e > qpos) sv[c][e] = __float_as_uint(-INFINITY);
      }
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < 32; ++e) mx4[e & 3] = fmaxf(mx4[e & 3], __uint_as_float(sv[c][e]));
      xmax[sb][hw][r] = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      asm volatile("bar.sync 1, 256;" ::: "memory");
      // scale > 0: max(s) * scale = max(s * scale)
      const float tmax = fmaxf(xmax[sb][0][r], xmax[sb][1][r]) * sl;
      const float m_new = fmaxf(m_run, tmax);
      const float alpha = exp2f(m_run - m_new);  // 0 on the first tile
      float ps4[4] = {0.f, 0.f, 0.f, 0.f};
      uint32_t pk[2][16];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          // 2^(s * scale*log2e - m): one FFMA + MUFU.EX2 per score (masked scores are -inf -> 0)
          const float p0 = fast_exp2(fmaf(__uint_as_float(sv[c][2 * e]), sl, -m_new));
          const float p1 = fast_exp2(fmaf(__uint_as_float(sv[c][2 * e + 1]), sl, -m_new));
          ps4[e & 3] += p0 + p1;
          pk[c][e] = pack_bf16x2(p0, p1);
        }
      l_half = l_half * alpha + ((ps4[0] + ps4[1]) + (ps4[2] + ps4[3]));
      m_run = m_new;
      // O (TMEM) and the P buffer are free once PV_{j-1} has completed
      if (j > 0) {
        mbar_wait(pv_done, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c0 = hw * 16; c0 < HD; c0 += 32) {
            uint32_t ov[16];
            tmem_ld16(tmem + lane_base + C::O_COL + c0, ov);
            tc_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            tmem_st16(tmem + lane_base + C::O_COL + c0, ov);
          }
          tc_wait_st();
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        sts128(p_base + sw128_off(r, u), make_uint4(pk[u >> 2][(u & 3) * 4 + 0], pk[u >> 2][(u & 3) * 4 + 1],
                                                   pk[u >> 2][(u & 3) * 4 + 2], pk[u >> 2][(u & 3) * 4 + 3]));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // ---- epilogue: O / l -> bf16, LSE (l = sum of the two halves' partial sums)
    xsum[hw][r] = l_half;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const float l_run = xsum[0][r] + xsum[1][r];
    mbar_wait(pv_done, (n_kv - 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l_run;
    const bool valid = q0 + r < a.n_q;
    uint16_t* orow = a.o + static_cast<int64_t>(q_row + r) * a.ldo + h * HD;
#pragma unroll
    for (int c0 = hw * 16; c0 < HD; c0 += 32) {
      uint32_t ov[16];
      tmem_ld16(tmem + lane_base + C::O_COL + c0, ov);
      tc_wait_ld();
      if (valid) {
        uint4 w0, w1;
        w0.x = pack_bf16x2(__uint_as_float(ov[0]) * inv_l, __uint_as_float(ov[1]) * inv_l);
        w0.y = pack_bf16x2(__uint_as_float(ov[2]) * inv_l, __uint_as_float(ov[3]) * inv_l);
        w0.z = pack_bf16x2(__uint_as_float(ov[4]) * inv_l, __uint_as_float(ov[5]) * inv_l);
        w0.w = pack_bf16x2(__uint_as_float(ov[6]) * inv_l, __uint_as_float(ov[7]) * inv_l);
        w1.x = pack_bf16x2(__uint_as_float(ov[8]) * inv_l, __uint_as_float(ov[9]) * inv_l);
        w1.y = pack_bf16x2(__uint_as_float(ov[10]) * inv_l, __uint_as_float(ov[11]) * inv_l);
        w1.z = pack_bf16x2(__uint_as_float(ov[12]) * inv_l, __uint_as_float(ov[13]) * inv_l);
        w1.w = pack_bf16x2(__uint_as_float(ov[14]) * inv_l, __uint_as_float(ov[15]) * inv_l);
        *reinterpret_cast<uint4*>(orow + c0) = w0;
        *reinterpret_cast<uint4*>(orow + c0 + 8) = w1;
      }
    }
    if (hw == 0 && valid && a.lse)
      a.lse[(static_cast<int64_t>(b) * a.Nh + h) * a.S + a.q_row0 + q0 + r] = (m_run + log2f(l_run)) * kLn2_3;
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int HD>
static cudaError_t launch_attn3_t(const PrefillAttnArgs& a, cudaStream_t stream) {
  using C = Attn3Cfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attn3_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::SMEM));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap tq, tk, tv;
  const uint64_t q_rows = static_cast<uint64_t>(a.B) * a.S;
  const uint64_t kv_rows = a.kv_rows_total ? static_cast<uint64_t>(a.kv_rows_total)
                                           : static_cast<uint64_t>(a.B) * a.Nkv * a.S_cap;
  if (!make_tmap_2d(&tq, a.q, static_cast<uint64_t>(a.ldq), q_rows, a.ldq * 2, C::CW, C::BM, C::SWB))
    return cudaErrorInvalidValue;
  if (!make_tmap_2d(&tk, a.k, HD, kv_rows, HD * 2, C::CW, C::BN, C::SWB)) return cudaErrorInvalidValue;
  if (!make_tmap_2d(&tv, a.v, HD, kv_rows, HD * 2, C::CW, C::BN, C::SWB)) return cudaErrorInvalidValue;
  dim3 grid((a.n_q + C::BM - 1) / C::BM, a.Nh, a.B);
  prof_mark(stream, true, kProfAttnPrefill);
  prefill_attn3_kernel<HD><<<grid, 352, C::SMEM, stream>>>(tq, tk, tv, a);
  prof_mark(stream, false, kProfAttnPrefill);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_prefill_attention_v3(const PrefillAttnArgs& a, cudaStream_t stream) {
  switch (a.rk) {
    case 16: return launch_attn3_t<16>(a, stream);
    case 32: return launch_attn3_t<32>(a, stream);
    case 48: return launch_attn3_t<48>(a, stream);
    case 64: return launch_attn3_t<64>(a, stream);
    case 80: return launch_attn3_t<80>(a, stream);
    case 96: return launch_attn3_t<96>(a, stream);
    case 112: return launch_attn3_t<112>(a, stream);
    case 128: return launch_attn3_t<128>(a, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace zdc
