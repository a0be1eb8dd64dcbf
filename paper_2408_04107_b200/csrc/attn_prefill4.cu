// attn_prefill4.cu — a3 prefill attention, v4 (default for head dims r <= 96): the math and
// rounding points of v1/v3 (Eqs. 2-3, scale 1/sqrt(d_h), LSE out), re-pipelined so the
// tensor core and the exp units stay busy at the same time:
//   * a work item is TWO consecutive 128-row query tiles of one head ("a" and "b"); their K'/V'
//     tiles stream once for both (tile a needs a prefix of tile b's causal key range);
//   * persistent CTAs (one per SM) take the items longest-first in a snake order, so the
//     triangular causal work is balanced over the SMs instead of leaving a ragged last wave;
//   * S_a, S_b, O_a, O_b live in TMEM; the MMA warp interleaves S_a(j+1), PV_a(j), S_b(j+1),
//     PV_b(j), so while one softmax group computes exponentials the tensor core works for the other;
//   * a softmax thread owns a whole query row (128 scores of a key tile in registers): no
//     cross-warp max exchange per tile;
//   * lazy rescaling: the running reference max m is only raised (and O, l rescaled) when a tile's
//     max exceeds it by more than 2^8; otherwise P = 2^(s - m) <= 2^8 is used as is.  O and l share
//     the reference, so O' = O / l and LSE = m + log2 l are unchanged; the bf16 rounding of P keeps
//     its relative error (reading c20).
// Warps 0-3 softmax of tile a, 4-7 of tile b, 8 Q'/K' TMA producer, 9 V' producer, 10 MMA issuer.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>

namespace zdc {

static constexpr float kLog2e4 = 1.4426950408889634f;
static constexpr float kLn2_4 = 0.6931471805599453f;
static constexpr float kLazyRescale = 8.0f;  // log2 units
// P in tensor memory (as in FlashAttention-4): the softmax stores P (bf16 pairs per 32-bit column)
// with tcgen05.st and the PV MMA reads its A operand from TMEM, instead of a 16 KB shared-memory
// write + proxy fence per tile.  Fits the 512 TMEM columns for r <= 64.
#ifndef ZDC_TMEM_P
#define ZDC_TMEM_P 1
#endif

// D[tmem] (+)= A[tmem] * B[smem] (A: M = 128 lanes x K packed two bf16 per column)
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int HD>
struct Attn4Cfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int CW = HD % 64 == 0 ? 64 : HD % 32 == 0 ? 32 : 16;
  static constexpr int NCH = HD / CW;
  static constexpr int SWB = CW * 2;
  static constexpr uint32_t LAYOUT = SWB == 128 ? kSw128 : SWB == 64 ? kSw64 : kSw32;
  static constexpr uint32_t CHUNK = BM * SWB;
  static constexpr uint32_t TILE = CHUNK * NCH;  // one 128-row tile at width HD
  static constexpr uint32_t P_BYTES = BM * BN * 2;
  static constexpr uint32_t budget = 220 * 1024;
  static constexpr int STAGES = (2 * TILE + 6 * TILE + 2 * P_BYTES <= budget) ? 3 : 2;
  static constexpr uint32_t OFF_Q = 0;  // [2] tiles
  static constexpr uint32_t OFF_K = 2 * TILE;
  static constexpr uint32_t OFF_V = OFF_K + STAGES * TILE;
  static constexpr uint32_t OFF_P = OFF_V + STAGES * TILE;  // [2] P buffers
  static constexpr uint32_t OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr uint32_t SMEM = OFF_BAR + 256 + 1024;
  static constexpr bool OK = 2 * TILE + 2 * STAGES * TILE + 2 * P_BYTES <= budget;
  static constexpr uint32_t TMEM_COLS = 512;  // S_a [0,128) S_b [128,256) O_a [256,+HD) O_b [256+HD,+HD)
  static constexpr uint32_t O_COL = 256;
  static constexpr bool TP = ZDC_TMEM_P && O_COL + 2 * HD + 2 * 64 <= TMEM_COLS;  // P_a, P_b: 64 columns each
  static constexpr uint32_t P_COL = O_COL + 2 * HD;
};

__device__ __forceinline__ void sts128_4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

template <int HD>
__global__ void __launch_bounds__(352, 1)
    prefill_attn4_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                         const __grid_constant__ CUtensorMap tv, const PrefillAttnArgs a) {
  using C = Attn4Cfg<HD>;
  constexpr int ST = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* q_empty = bar + 1;
  uint64_t* k_full = bar + 2;        // [ST]
  uint64_t* k_empty = k_full + ST;   // [ST]
  uint64_t* v_full = k_empty + ST;   // [ST]
  uint64_t* v_empty = v_full + ST;   // [ST]
  uint64_t* s_full = v_empty + ST;   // [2] per query tile
  uint64_t* s_free = s_full + 2;     // [2]
  uint64_t* p_full = s_free + 2;     // [2]
  uint64_t* pv_done = p_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  // Persistent: work items = (query-tile pair, sequence, head), ordered by causal cost (longest
  // pairs first) and dealt to the CTAs in a snake order (pass r: CTA c takes item r*ncta + c for
  // even r, r*ncta + ncta-1-c for odd r), which balances the triangular work across the SMs.
  const int n_qt = (a.n_q + C::BM - 1) / C::BM;
  const int n_pairs = (n_qt + 1) / 2;
  const int n_bh = a.B * a.Nh;
  const int n_items = n_pairs * n_bh;
  const int ncta = gridDim.x, cta = blockIdx.x;
  const int G = a.Nh / a.Nkv;
  auto item_of = [&](int r) -> int { return r * ncta + ((r & 1) ? ncta - 1 - cta : cta); };
  struct Item {
    int b, h, g, q0[2], nkv[2], nmax;
  };
  auto decode_item = [&](int k) -> Item {
    Item it;
    const int pd = k / n_bh, bh = k - pd * n_bh;
    const int pair = n_pairs - 1 - pd;
    it.b = bh / a.Nh;
    it.h = bh - it.b * a.Nh;
    it.g = it.h / G;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int qt = 2 * pair + t;
      it.q0[t] = qt * C::BM;
      if (qt < n_qt) {
        const int last_q = min(it.q0[t] + C::BM, a.n_q) - 1;
        it.nkv[t] = (a.q_pos0 + last_q + 1 + C::BN - 1) / C::BN;
      } else {
        it.nkv[t] = 0;  // an odd tile count leaves the last pair with one tile
      }
    }
    it.nmax = max(it.nkv[0], it.nkv[1]);
    return it;
  };
  auto kv_tile_row = [&](const Item& it, int j) -> int {
    const int pos = j * C::BN;
    if (a.kv_mode == 0) return (it.b * a.Nkv + it.g) * a.S_cap + pos;
    const int qq = pos / a.sp_chunk, rr = pos - qq * a.sp_chunk;  // SP gather buffer
    if (a.kv_mode == 2) {  // zigzag, half-major buffer [half][owner][K|V][B][Nkv][chunk][r] (overlapped exchange)
      const int h = qq < a.sp_P ? 0 : 1, ow = h == 0 ? qq : 2 * a.sp_P - 1 - qq;
      return (((h * a.sp_P + ow) * 2 * a.B + it.b) * a.Nkv + it.g) * a.sp_chunk + rr;
    }
    int owner, local;
    if (!a.sp_zigzag) {
      owner = qq;
      local = rr;
    } else {
      owner = qq < a.sp_P ? qq : 2 * a.sp_P - 1 - qq;
      local = (qq < a.sp_P ? 0 : a.sp_chunk) + rr;
    }
    return ((owner * 2 * a.B + it.b) * a.Nkv + it.g) * a.sp_n_local + local;
  };
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 8) {
    if (lane == 0) {
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
      for (int t = 0; t < 2; ++t) {
        mbar_init(&s_full[t], 1);
        mbar_init(&s_free[t], 4);  // one arrival per softmax warp of the tile
        mbar_init(&p_full[t], 4);
        mbar_init(&pv_done[t], 1);
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
  // launched with programmatic dependent launch: Q'/K'/V' come from the a1 projection before it
  pdl_wait();
  pdl_trigger();

  if (warp == 8) {
    // ------------------------------------------------ Q' (both tiles) and K' producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      int gk = 0;  // K'/V' tiles streamed by this CTA so far
      for (int r = 0, k = item_of(0); k < n_items; k = item_of(++r)) {
        const Item it = decode_item(k);
        const int n_tiles = it.nkv[1] > 0 ? 2 : 1;
        if (r > 0) mbar_wait(q_empty, (r - 1) & 1);  // every S MMA of the previous item is done
        mbar_arrive_expect_tx(q_full, C::TILE * n_tiles);
        for (int t = 0; t < n_tiles; ++t)
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_2d(smem + C::OFF_Q + t * C::TILE + c * C::CHUNK, &tq, q_full, it.h * HD + c * C::CW,
                        it.b * a.S + a.q_row0 + it.q0[t]);
        for (int j = 0; j < it.nmax; ++j, ++gk) {
          const int s = gk % ST;
          mbar_wait(&k_empty[s], ((gk / ST) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[s], C::TILE);
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_2d_hint(smem + C::OFF_K + s * C::TILE + c * C::CHUNK, &tk, &k_full[s], c * C::CW,
                             kv_tile_row(it, j), keep);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------ V' producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      int gk = 0;
      for (int r = 0, k = item_of(0); k < n_items; k = item_of(++r)) {
        const Item it = decode_item(k);
        for (int j = 0; j < it.nmax; ++j, ++gk) {
          const int s = gk % ST;
          mbar_wait(&v_empty[s], ((gk / ST) & 1) ^ 1);
          mbar_arrive_expect_tx(&v_full[s], C::TILE);
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_2d_hint(smem + C::OFF_V + s * C::TILE + c * C::CHUNK, &tv, &v_full[s], c * C::CW,
                             static_cast<int>(kv_tile_row(it, j) + a.v_row_off), keep);
        }
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------ MMA issuer: S_a(j+1), PV_a(j), S_b(j+1), PV_b(j)
    if (elect_one()) {
      constexpr uint32_t idesc_s = make_idesc_bf16(C::BM, C::BN, 0, 0);
      constexpr uint32_t idesc_o = make_idesc_bf16(C::BM, HD, 0, 1);
      int cs[2] = {0, 0}, cp[2] = {0, 0};  // S / PV tiles issued per query tile (all items)
      auto issue_s = [&](int t, int gk) {
        const int s = gk % ST;
        mbar_wait(&k_full[s], (gk / ST) & 1);
        if (cs[t] > 0) mbar_wait(&s_free[t], (cs[t] - 1) & 1);  // the softmax warps have read S_t
        tc_fence_after();
        const uint32_t q_addr = smem_u32(smem + C::OFF_Q + t * C::TILE);
        const uint32_t k_addr = smem_u32(smem + C::OFF_K + s * C::TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
#pragma unroll
          for (int kk = 0; kk < C::CW / 16; ++kk) {
            const uint64_t ad = make_sdesc(q_addr + c * C::CHUNK + kk * 32, 16, 8 * C::SWB, C::LAYOUT);
            const uint64_t bd = make_sdesc(k_addr + c * C::CHUNK + kk * 32, 16, 8 * C::SWB, C::LAYOUT);
            umma_bf16_ss(tmem + t * 128, ad, bd, idesc_s, (c | kk) != 0 ? 1u : 0u);
          }
        umma_commit(&s_full[t]);
        ++cs[t];
      };
      auto issue_pv = [&](int t, int gk, bool first) {
        const int s = gk % ST;
        mbar_wait(&p_full[t], cp[t] & 1);
        mbar_wait(&v_full[s], (gk / ST) & 1);
        tc_fence_after();
        const uint32_t p_addr = smem_u32(smem + C::OFF_P + t * C::P_BYTES);
        const uint32_t v_addr = smem_u32(smem + C::OFF_V + s * C::TILE);
#pragma unroll
        for (int kk = 0; kk < C::BN / 16; ++kk) {
          const uint64_t bd = make_sdesc(v_addr + kk * 16 * C::SWB, C::CHUNK, 8 * C::SWB, C::LAYOUT);
          if constexpr (C::TP) {
            umma_bf16_ts(tmem + C::O_COL + t * HD, tmem + C::P_COL + t * 64 + kk * 8, bd, idesc_o,
                         (!first || kk != 0) ? 1u : 0u);
          } else {
            const uint64_t ad = make_sdesc(p_addr + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, kSw128);
            umma_bf16_ss(tmem + C::O_COL + t * HD, ad, bd, idesc_o, (!first || kk != 0) ? 1u : 0u);
          }
        }
        umma_commit(&pv_done[t]);
        ++cp[t];
      };
      int gk0 = 0;
      for (int r = 0, k = item_of(0); k < n_items; k = item_of(++r)) {
        const Item it = decode_item(k);
        mbar_wait(q_full, r & 1);
        for (int t = 0; t < 2; ++t)
          if (it.nkv[t] > 0) issue_s(t, gk0);
        if (it.nmax > 0) umma_commit(&k_empty[gk0 % ST]);
        for (int j = 0; j < it.nmax; ++j) {
          for (int t = 0; t < 2; ++t) {
            if (j + 1 < it.nkv[t]) issue_s(t, gk0 + j + 1);
            if (j < it.nkv[t]) issue_pv(t, gk0 + j, j == 0);
          }
          if (j + 1 < it.nmax) umma_commit(&k_empty[(gk0 + j + 1) % ST]);  // K'(j+1) read by both S
          umma_commit(&v_empty[(gk0 + j) % ST]);                           // V'(j) read by both PV
        }
        umma_commit(q_empty);  // Q' of this item no longer read once these MMAs complete
        gk0 += it.nmax;
      }
    }
  } else {
    // ------------------------------------------------ softmax: warps 0-3 tile a, 4-7 tile b
    const int t = warp >> 2, qq = warp & 3;
    const int r = qq * 32 + lane;  // query row of the tile = TMEM lane
    const uint32_t lane_base = (qq * 32) << 16;
    const uint32_t s_col = tmem + lane_base + t * 128;
    const uint32_t o_col = tmem + lane_base + C::O_COL + t * HD;
    const float sl = a.scale * kLog2e4;
    const uint32_t p_base = smem_u32(smem + C::OFF_P + t * C::P_BYTES);
    int base = 0;  // S / P / PV tiles of this query tile consumed so far (all items)
    for (int ri = 0, k = item_of(0); k < n_items; k = item_of(++ri)) {
      const Item it = decode_item(k);
      const int n = it.nkv[t];
      const int q0 = it.q0[t];
      const int qpos = a.q_pos0 + q0 + r;
      const int qbase = a.q_pos0 + q0 + qq * 32;  // first row of this warp
      float m_ref = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n; ++j) {
        const int gi = base + j;
        mbar_wait(&s_full[t], gi & 1);
        tc_fence_after();
        uint32_t sv[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(s_col + c * 32, sv[c]);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[t]);
        const int key0 = j * C::BN;
        if (key0 + C::BN - 1 > qbase) {  // tile crosses this warp's diagonal
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (key0 + c * 32 + e > qpos) sv[c][e] = __float_as_uint(-INFINITY);
        }
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e) mx4[e & 3] = fmaxf(mx4[e & 3], __uint_as_float(sv[c][e]));
        const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl;  // scale > 0
        // lazy rescale: raise the reference only when this tile exceeds it by > 2^kLazyRescale
        const bool raise = mx > m_ref + kLazyRescale;
        const float m_new = raise ? mx : m_ref;
        const float alpha = raise ? exp2f(m_ref - m_new) : 1.f;  // 0 on the first tile
        const float mref = m_new == -INFINITY ? 0.f : m_new;
        float ps4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            // 2^(s * scale*log2e - m): one FFMA + MUFU.EX2 per score (masked scores are -inf -> 0)
            const float p0 = fast_exp2(fmaf(__uint_as_float(sv[c][2 * e]), sl, -mref));
            const float p1 = fast_exp2(fmaf(__uint_as_float(sv[c][2 * e + 1]), sl, -mref));
            ps4[e & 3] += p0 + p1;
            sv[c][e] = pack_bf16x2(p0, p1);  // packed in place (e <= 2e)
          }
        l_run = l_run * alpha + ((ps4[0] + ps4[1]) + (ps4[2] + ps4[3]));
        m_ref = m_new;
        // O_t and the P_t buffer are free once PV_t(j-1) has completed
        if (j > 0) {
          mbar_wait(&pv_done[t], (gi - 1) & 1);
          tc_fence_after();
          if (__any_sync(0xffffffffu, raise)) {
#pragma unroll
            for (int c0 = 0; c0 < HD; c0 += 16) {
              uint32_t ov[16];
              tmem_ld16(o_col + c0, ov);
              tc_wait_ld();
#pragma unroll
              for (int e = 0; e < 16; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
              tmem_st16(o_col + c0, ov);
            }
            tc_wait_st();
          }
        }
        if constexpr (C::TP) {
          // P row -> TMEM columns [P_COL + 64 t, +64): column j = keys 2j (low half), 2j+1
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t pv[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) pv[e] = sv[c][e];
            tmem_st16(tmem + lane_base + C::P_COL + t * 64 + c * 16, pv);
          }
          tc_wait_st();
        } else {
          // P row -> shared memory, K-major 128B swizzle: keys [0,64) in chunk 0, [64,128) in chunk 1
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int c = u >> 2, e = (u & 3) * 4;  // 8 keys per 16-byte unit: sv[c][e..e+3]
            sts128_4(p_base + (u >> 3) * 16384 + sw128_off(r, u & 7), sv[c][e], sv[c][e + 1], sv[c][e + 2],
                     sv[c][e + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
      }
      // ---- epilogue: O / l -> bf16, LSE = m + log2 l (natural log out).  The next item's first
      // PV (which overwrites O_t) waits for this tile's next P, written after these reads.
      if (n > 0) {
        mbar_wait(&pv_done[t], (base + n - 1) & 1);
        tc_fence_after();
        const float inv_l = 1.f / l_run;
        const bool valid = q0 + r < a.n_q;
        uint16_t* orow = a.o + static_cast<int64_t>(it.b * a.S + a.q_row0 + q0 + r) * a.ldo + it.h * HD;
#pragma unroll
        for (int c0 = 0; c0 < HD; c0 += 16) {
          uint32_t ov[16];
          tmem_ld16(o_col + c0, ov);
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
          a.lse[(static_cast<int64_t>(it.b) * a.Nh + it.h) * a.S + a.q_row0 + q0 + r] =
              (m_ref + log2f(l_run)) * kLn2_4;
        tc_fence_before();
      }
      base += n;
    }
  }
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int HD>
static cudaError_t launch_attn4_t(const PrefillAttnArgs& a, cudaStream_t stream) {
  using C = Attn4Cfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attn4_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  const int n_qt = (a.n_q + C::BM - 1) / C::BM;
  const int n_items = (n_qt + 1) / 2 * a.Nh * a.B;
  dim3 grid(std::min(n_items, num_sms()));  // persistent: the kernel deals the items to the CTAs
  prof_mark(stream, true, kProfAttnPrefill);
  cudaError_t e = launch_k(prefill_attn4_kernel<HD>, grid, dim3(352), C::SMEM, stream, g_pdl, tq, tk, tv, a);
  prof_mark(stream, false, kProfAttnPrefill);
  if (e != cudaSuccess) return e;
  ++g_launches;
  return cudaGetLastError();
}

bool prefill_attention_v4_supported(int rk) {
  return rk == 16 || rk == 32 || rk == 48 || rk == 64 || rk == 80 || rk == 96;
}

cudaError_t launch_prefill_attention_v4(const PrefillAttnArgs& a, cudaStream_t stream) {
  switch (a.rk) {
    case 16: return launch_attn4_t<16>(a, stream);
    case 32: return launch_attn4_t<32>(a, stream);
    case 48: return launch_attn4_t<48>(a, stream);
    case 64: return launch_attn4_t<64>(a, stream);
    case 80: return launch_attn4_t<80>(a, stream);
    case 96: return launch_attn4_t<96>(a, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace zdc
