// attn_prefill.cu — a3 for prompt processing: causal attention at head dimension r run directly
// on the compressed Q'/K'/V' (Lemma 2: Q'(K')^T ~ QK^T needs no decompression; the
// V' decompression happens inside a5).  Eqs. 2-3 with the ORIGINAL
// scale 1/sqrt(d_h) (reading c2), and the log of each row's softmax denominator (LSE) written
// out in f32 — the "reused softmax denominators" of P:1442 that a4 ranks.
//
// One CTA per (128-query tile, head, sequence), FlashAttention-style online softmax with the
// two contractions on tcgen05:
//   S_j  = Q' K'_j^T   tcgen05.mma M=128 N=128 K=r   (A = Q' smem K-major, B = K' smem K-major)
//   O   += P_j V'_j    tcgen05.mma M=128 N=r  K=128  (A = P smem K-major,  B = V' smem MN-major)
// S is double-buffered in TMEM so the MMA of S_{j+1} overlaps the softmax of S_j; O stays in
// TMEM for the whole KV loop and is rescaled in place when the running max moves.
// Warps 0-7: softmax (thread = query row = TMEM lane; warps w and w+4 split the 128 keys of a
// tile); warp 8: TMA producer; warp 9: MMA issuer.
// Rounding points: P = exp(s - m) rounded to bf16 before PV, l from the
// unrounded P; O' rounded to bf16 after the division by l.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace zdc {

static constexpr float kLog2eF = 1.4426950408889634f;
static constexpr float kLn2F = 0.6931471805599453f;

template <int HD>
struct AttnCfg {
  static constexpr int BM = 128, BN = 128;                 // query rows / keys per tile
  static constexpr int CW = HD % 64 == 0 ? 64 : HD % 32 == 0 ? 32 : 16;  // elements per swizzle chunk row
  static constexpr int NCH = HD / CW;                      // chunks across the head dim
  static constexpr int SWB = CW * 2;                       // swizzle width in bytes (32/64/128)
  static constexpr uint32_t LAYOUT = SWB == 128 ? kSw128 : SWB == 64 ? kSw64 : kSw32;
  static constexpr uint32_t CHUNK = BM * SWB;              // bytes of one [128][CW] chunk
  static constexpr uint32_t TILE = CHUNK * NCH;            // bytes of one [128][HD] tile
  static constexpr uint32_t P_BYTES = BM * BN * 2;         // P as two [128][64] SW128 chunks
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = TILE;
  static constexpr uint32_t OFF_V = OFF_K + 2 * TILE;
  static constexpr uint32_t OFF_P = OFF_V + 2 * TILE;
  static constexpr uint32_t OFF_BAR = OFF_P + P_BYTES;
  static constexpr uint32_t SMEM = OFF_BAR + 256 + 1024;
  static constexpr uint32_t TMEM_COLS = 512;               // S0 [0,128) S1 [128,256) O [256, 256+HD)
  static constexpr uint32_t O_COL = 256;
};

template <int HD>
__global__ void __launch_bounds__(320, 1)
    prefill_attn_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                        const __grid_constant__ CUtensorMap tv, const PrefillAttnArgs a) {
  using C = AttnCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* s_full = bar + 9;   // [2]
  uint64_t* s_empty = bar + 11; // [2]
  uint64_t* p_full = bar + 13;
  uint64_t* pv_done = bar + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  // heavy (long causal row) tiles first
  const int n_qt = (a.n_q + C::BM - 1) / C::BM;
  const int qt = n_qt - 1 - static_cast<int>(blockIdx.x);
  const int h = blockIdx.y, b = blockIdx.z;
  const int G = a.Nh / a.Nkv, g = h / G;
  const int q0 = qt * C::BM;                                 // first query row of the tile (chunk-relative)
  const int last_q = min(q0 + C::BM, a.n_q) - 1;
  const int kv_end = a.q_pos0 + last_q + 1;                   // keys [0, kv_end) are visible to some row
  const int n_kv = (kv_end + C::BN - 1) / C::BN;
  const int q_row = b * a.S + a.q_row0 + q0;                  // row in the Q'/O' matrices
  // row of the first key of KV tile j in the K'/V' tensor maps (V row = K row + v_row_off)
  auto kv_tile_row = [&](int j) -> int {
    const int pos = j * C::BN;
    if (a.kv_mode == 0) return (b * a.Nkv + g) * a.S_cap + pos;
    const int q = pos / a.sp_chunk, r = pos - q * a.sp_chunk;   // SP gather buffer
    int owner, local;
    if (!a.sp_zigzag) {
      owner = q;
      local = r;
    } else {
      owner = q < a.sp_P ? q : 2 * a.sp_P - 1 - q;
      local = (q < a.sp_P ? 0 : a.sp_chunk) + r;
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
      for (int i = 0; i < 2; ++i) {
        mbar_init(&k_full[i], 1);
        mbar_init(&k_empty[i], 1);
        mbar_init(&v_full[i], 1);
        mbar_init(&v_empty[i], 1);
        mbar_init(&s_full[i], 1);
        mbar_init(&s_empty[i], 256);
      }
      mbar_init(p_full, 256);
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
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      mbar_arrive_expect_tx(q_full, C::TILE);
#pragma unroll
      for (int c = 0; c < C::NCH; ++c)
        tma_load_2d(smem + C::OFF_Q + c * C::CHUNK, &tq, q_full, h * HD + c * C::CW, q_row);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&k_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&k_full[s], C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_2d_hint(smem + C::OFF_K + s * C::TILE + c * C::CHUNK, &tk, &k_full[s], c * C::CW,
                           kv_tile_row(j), keep);
        mbar_wait(&v_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&v_full[s], C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_2d_hint(smem + C::OFF_V + s * C::TILE + c * C::CHUNK, &tv, &v_full[s], c * C::CW,
                           static_cast<int>(kv_tile_row(j) + a.v_row_off), keep);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_s = make_idesc_bf16(C::BM, C::BN, 0, 0);
      constexpr uint32_t idesc_o = make_idesc_bf16(C::BM, HD, 0, 1);
      const uint32_t q_addr = smem_u32(smem + C::OFF_Q);
      const uint32_t p_addr = smem_u32(smem + C::OFF_P);
      auto issue_s = [&](int j) {
        const int s = j & 1;
        mbar_wait(&k_full[s], (j >> 1) & 1);
        mbar_wait(&s_empty[s], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(smem + C::OFF_K + s * C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
#pragma unroll
          for (int kk = 0; kk < C::CW / 16; ++kk) {
            const uint64_t ad = make_sdesc(q_addr + c * C::CHUNK + kk * 32, 16, 8 * C::SWB, C::LAYOUT);
            const uint64_t bd = make_sdesc(k_addr + c * C::CHUNK + kk * 32, 16, 8 * C::SWB, C::LAYOUT);
            umma_bf16_ss(tmem + s * 128, ad, bd, idesc_s, (c | kk) != 0 ? 1u : 0u);
          }
        umma_commit(&k_empty[s]);
        umma_commit(&s_full[s]);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) issue_s(j + 1);
        const int s = j & 1;
        mbar_wait(p_full, j & 1);
        mbar_wait(&v_full[s], (j >> 1) & 1);
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
    // ------------------------------------------------ softmax warps 0..7: thread = query row;
    // warps w and w+4 share TMEM lane quarter w%4 and split the 128 keys of a tile (64 each), so
    // every scheduler runs two softmax warps.  Only the row max is exchanged per tile; each half
    // keeps its own partial row sum until the epilogue.
    __shared__ float xmax[2][2][128];  // [tile parity][half][row]
    __shared__ float xsum[2][128];
    const int hw = warp >> 2, qq = warp & 3;
    const int r = qq * 32 + lane;
    const int qpos = a.q_pos0 + q0 + r;                      // global position of this query row
    const uint32_t lane_base = (qq * 32) << 16;
    const float sl = a.scale * kLog2eF;
    float m_run = -INFINITY, l_half = 0.f;
    uint8_t* p_smem = smem + C::OFF_P + hw * 16384;          // this half's [128][64] SW128 chunk
    for (int j = 0; j < n_kv; ++j) {
      const int s = j & 1;
      mbar_wait(&s_full[s], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[2][32];
#pragma unroll
      for (int c = 0; c < 2; ++c) tmem_ld32(tmem + lane_base + s * 128 + hw * 64 + c * 32, sv[c]);
      tc_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_empty[s]);
      const int key0 = j * C::BN + hw * 64;
      const bool diag = key0 + 63 > qpos;                    // some key of this half is in the future
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float x = __uint_as_float(sv[c][e]);
          if (diag && key0 + c * 32 + e > qpos) {
            x = -INFINITY;
            sv[c][e] = __float_as_uint(x);
          }
          mx4[e & 3] = fmaxf(mx4[e & 3], x);
        }
      xmax[s][hw][r] = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      asm volatile("bar.sync 1, 256;" ::: "memory");
      // scale > 0: max(s) * scale = max(s * scale)
      const float tmax = fmaxf(xmax[s][0][r], xmax[s][1][r]) * sl;
      const float m_new = fmaxf(m_run, tmax);
      const float alpha = exp2f(m_run - m_new);              // 0 on the first tile
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
      // O (TMEM) and the P buffer (smem) are free once PV_{j-1} has completed
      if (j > 0) {
        mbar_wait(pv_done, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c0 = hw * 16; c0 < HD; c0 += 32) {        // this half's 16-column chunks of O
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
      // P row r, keys [hw*64, hw*64+64) -> this half's K-major SW128 chunk
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint4 val = make_uint4(pk[u >> 2][(u & 3) * 4 + 0], pk[u >> 2][(u & 3) * 4 + 1],
                               pk[u >> 2][(u & 3) * 4 + 2], pk[u >> 2][(u & 3) * 4 + 3]);
        *reinterpret_cast<uint4*>(p_smem + sw128_off(r, u)) = val;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      mbar_arrive(p_full);
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
      a.lse[(static_cast<int64_t>(b) * a.Nh + h) * a.S + a.q_row0 + q0 + r] = (m_run + log2f(l_run)) * kLn2F;
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// =====================================================================================
// v2: two 128-row query tiles per CTA (A = rows [256i, 256i+128), B = the next 128) share every
// K'/V' tile load; two softmax warpgroups (warps 0-3 -> tile A, 4-7 -> tile B) ping-pong with the
// MMA warp so the tensor core computes one tile's S / PV while the other tile's softmax runs.
// The running max is only moved (and O rescaled in TMEM) when it grows by more than 2^8
// ("conditional rescaling"): P = 2^(s - m_used) <= 256 stays exact enough in f32 / bf16 and the
// final O / l and LSE = m_used + log2 l are unchanged mathematically.
// TMEM: S_A [0,128) S_B [128,256) O_A [256, 256+HD) O_B [256+HD, 256+2HD).
template <int HD>
struct Attn2Cfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int CW = HD % 64 == 0 ? 64 : HD % 32 == 0 ? 32 : 16;
  static constexpr int NCH = HD / CW;
  static constexpr int SWB = CW * 2;
  static constexpr uint32_t LAYOUT = SWB == 128 ? kSw128 : SWB == 64 ? kSw64 : kSw32;
  static constexpr uint32_t CHUNK = BM * SWB;
  static constexpr uint32_t TILE = CHUNK * NCH;
  static constexpr uint32_t P_BYTES = BM * BN * 2;
  static constexpr uint32_t OFF_Q = 0;                    // Q_A, Q_B
  static constexpr uint32_t OFF_K = 2 * TILE;             // 2 stages
  static constexpr uint32_t OFF_V = OFF_K + 2 * TILE;     // 2 stages
  static constexpr uint32_t OFF_P = OFF_V + 2 * TILE;     // P_A, P_B
  static constexpr uint32_t OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr uint32_t SMEM = OFF_BAR + 256 + 1024;
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr float kRescaleThreshold = 8.0f;        // log2 units
};

template <int HD>
__global__ void __launch_bounds__(320, 1)
    prefill_attn2_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                         const __grid_constant__ CUtensorMap tv, const PrefillAttnArgs a) {
  using C = Attn2Cfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;    // [2]
  uint64_t* k_empty = bar + 3;   // [2]
  uint64_t* v_full = bar + 5;    // [2]
  uint64_t* v_empty = bar + 7;   // [2]
  uint64_t* s_full = bar + 9;    // [2] per query tile
  uint64_t* p_full = bar + 11;   // [2]
  uint64_t* pv_done = bar + 13;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int n_pairs = (a.n_q + 2 * C::BM - 1) / (2 * C::BM);
  const int pi = n_pairs - 1 - static_cast<int>(blockIdx.x);  // heavy pairs first
  const int h = blockIdx.y, b = blockIdx.z;
  const int G = a.Nh / a.Nkv, g = h / G;
  int q0[2], nkv[2];
  for (int x = 0; x < 2; ++x) {
    q0[x] = pi * 2 * C::BM + x * C::BM;
    if (q0[x] < a.n_q) {
      const int last_q = min(q0[x] + C::BM, a.n_q) - 1;
      nkv[x] = (a.q_pos0 + last_q + 1 + C::BN - 1) / C::BN;
    } else {
      nkv[x] = 0;
    }
  }
  const int n_kv = max(nkv[0], nkv[1]);
  auto kv_tile_row = [&](int j) -> int {
    const int pos = j * C::BN;
    if (a.kv_mode == 0) return (b * a.Nkv + g) * a.S_cap + pos;
    const int q = pos / a.sp_chunk, r = pos - q * a.sp_chunk;
    int owner, local;
    if (!a.sp_zigzag) {
      owner = q;
      local = r;
    } else {
      owner = q < a.sp_P ? q : 2 * a.sp_P - 1 - q;
      local = (q < a.sp_P ? 0 : a.sp_chunk) + r;
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
      for (int i = 0; i < 2; ++i) {
        mbar_init(&k_full[i], 1);
        mbar_init(&k_empty[i], 1);
        mbar_init(&v_full[i], 1);
        mbar_init(&v_empty[i], 1);
        mbar_init(&s_full[i], 1);
        mbar_init(&p_full[i], 128);
        mbar_init(&pv_done[i], 1);
      }
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
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      mbar_arrive_expect_tx(q_full, 2 * C::TILE);
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_2d(smem + C::OFF_Q + x * C::TILE + c * C::CHUNK, &tq, q_full, h * HD + c * C::CW,
                      b * a.S + a.q_row0 + q0[x]);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        const int row = kv_tile_row(j);
        mbar_wait(&k_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&k_full[s], C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_2d_hint(smem + C::OFF_K + s * C::TILE + c * C::CHUNK, &tk, &k_full[s], c * C::CW, row, keep);
        mbar_wait(&v_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&v_full[s], C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_2d_hint(smem + C::OFF_V + s * C::TILE + c * C::CHUNK, &tv, &v_full[s], c * C::CW,
                           static_cast<int>(row + a.v_row_off), keep);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_s = make_idesc_bf16(C::BM, C::BN, 0, 0);
      constexpr uint32_t idesc_o = make_idesc_bf16(C::BM, HD, 0, 1);
      auto issue_s = [&](int x, int j) {
        const uint32_t q_addr = smem_u32(smem + C::OFF_Q + x * C::TILE);
        const uint32_t k_addr = smem_u32(smem + C::OFF_K + (j & 1) * C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
#pragma unroll
          for (int kk = 0; kk < C::CW / 16; ++kk) {
            const uint64_t ad = make_sdesc(q_addr + c * C::CHUNK + kk * 32, 16, 8 * C::SWB, C::LAYOUT);
            const uint64_t bd = make_sdesc(k_addr + c * C::CHUNK + kk * 32, 16, 8 * C::SWB, C::LAYOUT);
            umma_bf16_ss(tmem + x * 128, ad, bd, idesc_s, (c | kk) != 0 ? 1u : 0u);
          }
        umma_commit(&s_full[x]);
      };
      auto issue_pv = [&](int x, int j) {
        const uint32_t p_addr = smem_u32(smem + C::OFF_P + x * C::P_BYTES);
        const uint32_t v_addr = smem_u32(smem + C::OFF_V + (j & 1) * C::TILE);
#pragma unroll
        for (int kk = 0; kk < C::BN / 16; ++kk) {
          const uint64_t ad = make_sdesc(p_addr + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, kSw128);
          const uint64_t bd = make_sdesc(v_addr + kk * 16 * C::SWB, C::CHUNK, 8 * C::SWB, C::LAYOUT);
          umma_bf16_ss(tmem + 256 + x * HD, ad, bd, idesc_o, (j | kk) != 0 ? 1u : 0u);
        }
        umma_commit(&pv_done[x]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      for (int x = 0; x < 2; ++x)
        if (nkv[x] > 0) issue_s(x, 0);
      umma_commit(&k_empty[0]);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j & 1;
        mbar_wait(&v_full[s], (j >> 1) & 1);
        bool next_k_ready = false;
        for (int x = 0; x < 2; ++x) {
          if (j >= nkv[x]) continue;
          mbar_wait(&p_full[x], j & 1);
          tc_fence_after();
          issue_pv(x, j);
          if (j + 1 < nkv[x]) {
            if (!next_k_ready) {
              mbar_wait(&k_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
              tc_fence_after();
              next_k_ready = true;
            }
            issue_s(x, j + 1);
          }
        }
        umma_commit(&v_empty[s]);
        if (next_k_ready) umma_commit(&k_empty[(j + 1) & 1]);
      }
    }
  } else {
    // ------------------------------------------------ softmax: warps 0-3 tile A, 4-7 tile B
    const int x = warp >> 2;
    const int my_q0 = x ? q0[1] : q0[0];     // scalars: no dynamically indexed local arrays
    const int my_nkv = x ? nkv[1] : nkv[0];
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_base = ((warp & 3) * 32) << 16;
    const uint32_t s_col = x * 128, o_col = 256 + x * HD;
    const int qpos = a.q_pos0 + my_q0 + r;
    const float sl = a.scale * kLog2eF;
    float m_used = -INFINITY, l_run = 0.f;
    uint8_t* p_smem = smem + C::OFF_P + x * C::P_BYTES;
    for (int j = 0; j < my_nkv; ++j) {
      mbar_wait(&s_full[x], j & 1);
      tc_fence_after();
      // two passes over the S tile in TMEM (max, then exponentials) keep 32 scores live, not 128
      const int key0 = j * C::BN;
      const bool diag = key0 + C::BN - 1 > qpos;  // some key of this tile lies after the query
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t sv[32];
        tmem_ld32(tmem + lane_base + s_col + c * 32, sv);
        tc_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float v = __uint_as_float(sv[e]);
          if (diag && key0 + c * 32 + e > qpos) v = -INFINITY;
          mx4[e & 3] = fmaxf(mx4[e & 3], v);
        }
      }
      // scale > 0: max(s) * scale = max(s * scale)
      const float tmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl;
      float alpha = 1.f;
      if (tmax > m_used + C::kRescaleThreshold) {  // first tile (m_used = -inf) always moves
        alpha = exp2f(m_used - tmax);
        m_used = tmax;
      }
      // O_x and the P_x buffer are free once PV_x(j-1) completed (it was issued before S_x(j), so
      // this wait normally returns at once)
      if (j > 0) {
        mbar_wait(&pv_done[x], (j - 1) & 1);
        tc_fence_after();
      }
      // exponentiate, accumulate and store P one 32-key chunk at a time (few live registers)
      float ps4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t sv[32];
        tmem_ld32(tmem + lane_base + s_col + c * 32, sv);
        tc_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          // 2^(s * scale*log2e - m_used): one FFMA + MUFU.EX2 per score
          float p0 = fast_exp2(fmaf(__uint_as_float(sv[2 * e]), sl, -m_used));
          float p1 = fast_exp2(fmaf(__uint_as_float(sv[2 * e + 1]), sl, -m_used));
          if (diag) {
            if (key0 + c * 32 + 2 * e > qpos) p0 = 0.f;
            if (key0 + c * 32 + 2 * e + 1 > qpos) p1 = 0.f;
          }
          ps4[e & 3] += p0 + p1;
          pk[e] = pack_bf16x2(p0, p1);
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {  // 4 units of 8 keys: keys c*32 + q4*8 ...
          const int u = c * 4 + q4;
          *reinterpret_cast<uint4*>(p_smem + (u >> 3) * 16384 + sw128_off(r, u & 7)) =
              make_uint4(pk[q4 * 4 + 0], pk[q4 * 4 + 1], pk[q4 * 4 + 2], pk[q4 * 4 + 3]);
        }
      }
      l_run = l_run * alpha + ((ps4[0] + ps4[1]) + (ps4[2] + ps4[3]));
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
        for (int c0 = 0; c0 < HD; c0 += 16) {
          uint32_t ov[16];
          tmem_ld16(tmem + lane_base + o_col + c0, ov);
          tc_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
          tmem_st16(tmem + lane_base + o_col + c0, ov);
        }
        tc_wait_st();
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&p_full[x]);
    }
    if (my_nkv > 0) {
      mbar_wait(&pv_done[x], (my_nkv - 1) & 1);
      tc_fence_after();
      const float inv_l = 1.f / l_run;
      const bool valid = my_q0 + r < a.n_q;
      uint16_t* orow = a.o + static_cast<int64_t>(b * a.S + a.q_row0 + my_q0 + r) * a.ldo + h * HD;
#pragma unroll
      for (int c0 = 0; c0 < HD; c0 += 16) {
        uint32_t ov[16];
        tmem_ld16(tmem + lane_base + o_col + c0, ov);
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
      if (valid && a.lse)
        a.lse[(static_cast<int64_t>(b) * a.Nh + h) * a.S + a.q_row0 + my_q0 + r] = (m_used + log2f(l_run)) * kLn2F;
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// A/B switch: ZDC_ATTN_V2=1 selects the two-tile kernel (measured slower than v1 so far: 103 vs 80 us
// per c2 layer, profiles/r01).
bool g_attn_v2 = getenv("ZDC_ATTN_V2") != nullptr;

template <int HD>
static cudaError_t launch_attn2_t(const PrefillAttnArgs& a, cudaStream_t stream) {
  using C = Attn2Cfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attn2_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  dim3 grid((a.n_q + 2 * C::BM - 1) / (2 * C::BM), a.Nh, a.B);
  prof_mark(stream, true, kProfAttnPrefill);
  prefill_attn2_kernel<HD><<<grid, 320, C::SMEM, stream>>>(tq, tk, tv, a);
  prof_mark(stream, false, kProfAttnPrefill);
  ++g_launches;
  return cudaGetLastError();
}

template <int HD>
static cudaError_t launch_attn_t(const PrefillAttnArgs& a, cudaStream_t stream) {
  if constexpr (HD <= 96) {
    if (g_attn_v2) return launch_attn2_t<HD>(a, stream);
  }
  using C = AttnCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  prefill_attn_kernel<HD><<<grid, 320, C::SMEM, stream>>>(tq, tk, tv, a);
  prof_mark(stream, false, kProfAttnPrefill);
  ++g_launches;
  return cudaGetLastError();
}

// v3 (attn_prefill3.cu) is the default; ZDC_ATTN_V1=1 / ZDC_ATTN_V2=1 select the older kernels
static const bool g_attn_v3 = getenv("ZDC_ATTN_V1") == nullptr && getenv("ZDC_ATTN_V2") == nullptr;
// v4 (attn_prefill4.cu, two query tiles per CTA, r <= 96) is the default; ZDC_ATTN_V3 selects v3
static const bool g_attn_v4 = g_attn_v3 && getenv("ZDC_ATTN_V3") == nullptr;

cudaError_t launch_prefill_attention(const PrefillAttnArgs& a, cudaStream_t stream) {
  if (a.rk != a.rv) return cudaErrorInvalidValue;
  if (g_attn_v4 && prefill_attention_v4_supported(a.rk)) return launch_prefill_attention_v4(a, stream);
  if (g_attn_v3) return launch_prefill_attention_v3(a, stream);
  switch (a.rk) {
    case 16: return launch_attn_t<16>(a, stream);
    case 32: return launch_attn_t<32>(a, stream);
    case 48: return launch_attn_t<48>(a, stream);
    case 64: return launch_attn_t<64>(a, stream);
    case 80: return launch_attn_t<80>(a, stream);
    case 96: return launch_attn_t<96>(a, stream);
    case 112: return launch_attn_t<112>(a, stream);
    case 128: return launch_attn_t<128>(a, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace zdc
