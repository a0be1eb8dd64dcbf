// decode_attn3.cu — a3 for token generation over the compressed cache, v3: byte-balanced flat
// split (s_tj = Q'_t . K'_j / sqrt(d_h), P = softmax(s), O'_t = sum_j P_tj V'_j,
// P:249-260 Eqs. 2-3; with a token split, unimportant keys carry only their first r^u dims and the
// rest read as zero, P:776 DEL / P:1442).
//
// Why: v2 (decode_attn2.cu) gives every (split, KV head, sequence) its own CTA.  At c3 (B = 32,
// 40 KV heads, two pools) that is 1280 + 1280 CTAs over 296 resident slots: 4.3 waves per pool,
// each CTA paying a pipeline ramp and a merge, and the last wave a third full.  Here the
// work is ONE list -- for each (sequence b, KV head g) pair its pool-0 rows, then its pool-1 rows
// -- and each of the W resident warps of the grid takes an equal share of its BYTES (row cost
// r + r for K'+V'), so every warp streams the same amount, across pair and pool boundaries,
// through its own ring of bulk copies without a wave tail.  A warp's share covers ~1-3 pairs; a
// pair covered by several warps is merged by the last of them (LSE merge of the pieces).
//
// Per warp: a 2-stage ring of 32-row tiles {K' rows, V' rows, q of the pair}; lane 0 issues the
// tile two ahead; lane j scores row j for the G query heads of the group; online softmax in the
// log2 domain; P rounded to bf16 before PV, l from the unrounded P (DESIGN.md §4.3 rounding
// points); lane owns output columns lane + 32 i.
#include "attn_mma.cuh"
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace zdc {

namespace {

constexpr int kW3 = 8;     // warps per CTA (one CTA per SM)
constexpr int kTR3 = 32;   // rows per tile
constexpr int kMaxP3 = 128;  // pieces per pair (partial slots per head)
constexpr float kLog2e3 = 1.4426950408889634f;

template <int RK>
struct DA3 {
  static constexpr uint32_t KT = kTR3 * RK * 2;           // one K' (or V') tile of pool 0
  static constexpr uint32_t QB = 8 * RK * 2;              // q of the pair's G <= 8 heads (bf16)
  static constexpr uint32_t STAGE = (2 * KT + QB + 127) / 128 * 128;
  static constexpr int NST = 2;
  static constexpr uint32_t WARP_BYTES = NST * STAGE;
};

__device__ __forceinline__ int64_t cdiv64(int64_t a, int64_t b) { return a <= 0 ? 0 : (a + b - 1) / b; }
__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
// One warp's walk over its tiles: pairs p = b * Nkv + g in order; in a pair, pool-0 rows then
// pool-1 rows; only the rows whose cost start lies in [lo, hi).
struct Walk {
  int64_t lo, hi;
  int p, pool, r, r_end;  // current pair / pool / next row / end row of this pool in the range
  bool done;
};

}  // namespace

template <int RK, int RK1>
__global__ void __launch_bounds__(kW3 * 32, 1) decode_attn3_kernel(const DecodeAttnArgs a, int w_launch, int q_once) {
  using C = DA3<RK>;
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ int64_t s_pb[129];  // cost prefix over sequences (B <= 128)
  __shared__ int s_n0[128], s_n1[128];
  __shared__ int64_t s_weff;
  __shared__ uint64_t bars[kW3][C::NST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kW3 + warp;
  uint8_t* ring = dsm + warp * C::WARP_BYTES;
  uint64_t* wbar = bars[warp];
  if (lane == 0) {
    for (int s = 0; s < C::NST; ++s) mbar_init(&wbar[s], 1);
    fence_barrier_init();
  }
  pdl_trigger();
  pdl_wait();  // the row counts (and the new rows) come from the predecessor

  const int B = a.B, Nkv = a.Nkv, G = a.Nh / a.Nkv, rk1 = RK1;
  const int64_t w0 = RK, w1 = rk1;  // cost of one row of each pool (K' + V' bytes / 4)
  if (threadIdx.x < 32) {
    // per-sequence row counts and the cost prefix (one warp; B <= 128)
    int64_t run = 0, cmax = 0;
    for (int b0 = 0; b0 < B; b0 += 32) {
      const int b = b0 + lane;
      int n0 = 0, n1 = 0;
      if (b < B) {
        if (a.n0_ptr) {
          n0 = a.n0_ptr[b];
          n1 = a.k1 ? a.n1_ptr[b] : 0;
        } else {
          n0 = a.len_ptr ? min(*a.len_ptr + 1, a.S_cap) : a.len;
        }
        s_n0[b] = n0;
        s_n1[b] = n1;
      }
      const int64_t cb = static_cast<int64_t>(n0) * w0 + static_cast<int64_t>(n1) * w1;
      int64_t x = cb;  // inclusive scan over the lanes
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      if (b < B) s_pb[b + 1] = run + x;
      run += __shfl_sync(0xffffffffu, x, 31);
      int64_t m = cb;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) m = max64(m, __shfl_xor_sync(0xffffffffu, m, off));
      cmax = max64(cmax, m);
    }
    if (lane == 0) {
      s_pb[0] = 0;
      // effective warp count: every warp range must hold a row start of each pair it crosses
      // (rows are at most max(w0, w1) apart) and no pair may need more than kMaxP3 pieces
      const int64_t total = run * Nkv;
      int64_t weff = w_launch;
      if (total > 0) {
        weff = min64(weff, total / max64(w0, w1));
        if (cmax > 0) weff = min64(weff, (kMaxP3 - 2) * total / cmax);
      }
      s_weff = max64(weff, 1);
    }
  }
  __syncthreads();
  const int64_t total = s_pb[B] * Nkv;
  const int64_t W = s_weff;
  if (gw >= W || total <= 0) return;

  auto pair_base = [&](int p) {  // cost of the pair's first row
    const int b = p / Nkv, g = p - b * Nkv;
    const int64_t cb = s_pb[b + 1] - s_pb[b];
    return s_pb[b] * Nkv + g * cb;
  };
  auto warp_of = [&](int64_t x) { return static_cast<int>((x * W) / total); };
  // the walk's pool ranges for pair p (false when this warp owns no row of it)
  auto enter_pair = [&](Walk& k) -> bool {
    const int b = k.p / Nkv;
    const int64_t P = pair_base(k.p);
    const int n0 = s_n0[b], n1 = s_n1[b];
    const int i0 = static_cast<int>(min64(n0, cdiv64(k.lo - P, w0)));
    const int i1 = static_cast<int>(min64(n0, cdiv64(k.hi - P, w0)));
    if (i1 > i0) {
      k.pool = 0;
      k.r = i0;
      k.r_end = i1;
      return true;
    }
    if (n1 > 0 && w1 > 0) {
      const int64_t P1 = P + static_cast<int64_t>(n0) * w0;
      const int j0 = static_cast<int>(min64(n1, cdiv64(k.lo - P1, w1)));
      const int j1 = static_cast<int>(min64(n1, cdiv64(k.hi - P1, w1)));
      if (j1 > j0) {
        k.pool = 1;
        k.r = j0;
        k.r_end = j1;
        return true;
      }
    }
    return false;
  };
  auto start_walk = [&](Walk& k) {
    k.lo = cdiv64(static_cast<int64_t>(gw) * total, W);
    k.hi = cdiv64(static_cast<int64_t>(gw + 1) * total, W);
    k.done = false;
    // the pair holding cost lo: the last sequence b with prefix <= lo, then g
    int lo_b = 0, hi_b = B - 1;
    while (lo_b < hi_b) {
      const int mid = (lo_b + hi_b + 1) >> 1;
      if (s_pb[mid] * Nkv <= k.lo) lo_b = mid; else hi_b = mid - 1;
    }
    const int64_t cb = s_pb[lo_b + 1] - s_pb[lo_b];
    int g = cb > 0 ? static_cast<int>((k.lo - s_pb[lo_b] * Nkv) / cb) : 0;
    if (g >= Nkv) g = Nkv - 1;
    k.p = lo_b * Nkv + g;
    while (k.p < B * Nkv && pair_base(k.p) < k.hi) {
      if (enter_pair(k)) return;
      ++k.p;
    }
    k.done = true;
  };
  // move to the next tile's start: rest of this pool, the pool-1 rows, the next pairs
  auto advance = [&](Walk& k, int nr) {
    k.r += nr;
    if (k.r < k.r_end) return;
    const int b = k.p / Nkv;
    if (k.pool == 0 && s_n1[b] > 0 && w1 > 0) {
      const int64_t P1 = pair_base(k.p) + static_cast<int64_t>(s_n0[b]) * w0;
      const int n1 = s_n1[b];
      const int j0 = static_cast<int>(min64(n1, cdiv64(k.lo - P1, w1)));
      const int j1 = static_cast<int>(min64(n1, cdiv64(k.hi - P1, w1)));
      if (j1 > j0) {
        k.pool = 1;
        k.r = j0;
        k.r_end = j1;
        return;
      }
    }
    for (++k.p; k.p < B * Nkv && pair_base(k.p) < k.hi; ++k.p)
      if (enter_pair(k)) return;
    k.done = true;
  };

  const float scl = a.scale * kLog2e3;
  // rows per tile: 32 of pool 0; as many 32-row passes of the narrower pool 1 as fill the same
  // bytes (c3: 96 rows of r^u = 32), so the bytes in flight per warp stay the same in both pools
  constexpr int tr1 = RK1 > 0 ? kTR3 * (RK / RK1 > 0 ? RK / RK1 : 1) : kTR3;
  auto tile_rows = [&](const Walk& k) { return min(k.pool == 0 ? kTR3 : tr1, k.r_end - k.r); };
  // issue side (lane 0): the tile at walk ki into stage st
  int last_p = -1;  // issue side: pair of the previous tile (q is copied with a piece's first tile only)
  auto issue = [&](const Walk& k, int st) {
    const int b = k.p / Nkv, g = k.p - b * Nkv;
    const int nr = tile_rows(k);
    const int width = k.pool == 0 ? RK : rk1;
    const uint16_t* kp = k.pool == 0 ? a.k : a.k1;
    const uint16_t* vp = k.pool == 0 ? a.v : a.v1;
    const int64_t row = (static_cast<int64_t>(b) * Nkv + g) * a.S_cap + k.r;
    const uint32_t rb = static_cast<uint32_t>(nr) * width * 2u;
    uint8_t* dst = ring + st * C::STAGE;
    const bool with_q = !q_once || k.p != last_p;
    last_p = k.p;
    const uint32_t qb = with_q ? static_cast<uint32_t>(G * RK * 2) : 0u;
    mbar_arrive_expect_tx(&wbar[st], 2 * rb + qb);
    bulk_g2s(dst, kp + row * width, rb, &wbar[st]);
    bulk_g2s(dst + C::KT, vp + row * width, rb, &wbar[st]);
    if (with_q) bulk_g2s(dst + 2 * C::KT, a.q + b * a.ldq + static_cast<int64_t>(g) * G * a.rk, qb, &wbar[st]);
  };

  Walk wi, wc;  // issue-side and compute-side walks
  start_walk(wi);
  wc = wi;
  if (wi.done) return;
  if (lane == 0)
    for (int s = 0; s < C::NST && !wi.done; ++s) {
      issue(wi, s);
      advance(wi, tile_rows(wi));
    }

  // ---- tensor-core formulation (attn3_pass): mma.sync m16n8k16, bf16 in, f32 accumulate
  constexpr int KS = RK / 16;   // k-steps of a pool-0 row
  constexpr int NT = RK / 8;    // output n-tiles
  const int g = lane >> 2, tq = lane & 3;
  float m = -INFINITY, l = 0.f;  // running max (log2 domain) / sum of row g
  float oacc[NT][4];
  uint32_t qa[KS][2];           // q fragments of the current piece (rows g < G; rows g + 8 are zero)
  auto reset = [&]() {
    m = -INFINITY;
    l = 0.f;
#pragma unroll
    for (int j = 0; j < NT; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
  };
  reset();
  bool new_piece = true;
  const int RVO = a.rv;
  const uint32_t ring_s = smem_u32(ring);
  for (int t = 0; !wc.done; ++t) {
    const int st = t % C::NST;
    mbar_wait(&wbar[st], (t / C::NST) & 1);
    const int p = wc.p, pool = wc.pool, nr = tile_rows(wc);
    if (new_piece) {  // q of this pair (bf16 in the stage) -> A fragments
      const uint16_t* Qt = reinterpret_cast<const uint16_t*>(ring + st * C::STAGE + 2 * C::KT);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        qa[ks][0] = g < G ? *reinterpret_cast<const uint32_t*>(Qt + g * RK + ks * 16 + 2 * tq) : 0u;
        qa[ks][1] = g < G ? *reinterpret_cast<const uint32_t*>(Qt + g * RK + ks * 16 + 8 + 2 * tq) : 0u;
      }
      new_piece = false;
    }
    const int width = pool == 0 ? RK : RK1;
    for (int j0 = 0; j0 < nr; j0 += kTR3) {  // 32-key passes
      const int np = min(kTR3, nr - j0);
      const uint32_t kb = ring_s + st * C::STAGE + static_cast<uint32_t>(j0 * width * 2);
      const uint32_t vb = kb + C::KT;
      if (np < kTR3) {
        // rows np.. of the stage hold stale bytes: zero those V' rows (P is 0 there, 0 * NaN is not)
        uint16_t* Vz = reinterpret_cast<uint16_t*>(ring + st * C::STAGE + C::KT) + j0 * width;
        for (int i = np * width + lane * 8; i < kTR3 * width; i += 256)
          *reinterpret_cast<uint4*>(Vz + i) = make_uint4(0, 0, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the stage's next bulk copy
        __syncwarp();
      }
      if constexpr (RK1 > 0) {
        if (pool == 1) {
          attn3_pass<RK1, NT, KS>(kb, vb, np, lane, qa, scl, m, l, oacc);
          continue;
        }
      }
      attn3_pass<RK, NT, KS>(kb, vb, np, lane, qa, scl, m, l, oacc);
    }
    __syncwarp();
    // refill this stage with the tile NST ahead
    if (lane == 0 && !wi.done) {
      issue(wi, st);
      advance(wi, tile_rows(wi));
    }
    advance(wc, nr);
    if (!wc.done && wc.p == p) continue;  // the piece of this pair goes on
    // ---- end of this warp's piece of pair p (row g = head g < G of the group)
    const int b = p / Nkv, gg = p - b * Nkv;
    const int64_t P = pair_base(p);
    const int n0 = s_n0[b], n1 = s_n1[b];
    const int64_t last = n1 > 0 && w1 > 0 ? P + static_cast<int64_t>(n0) * w0 + static_cast<int64_t>(n1 - 1) * w1
                                          : P + static_cast<int64_t>(n0 - 1) * w0;
    const int wf = warp_of(P), wl = warp_of(last);
    const int pieces = wl - wf + 1;
    if (pieces == 1) {  // the whole pair: O' and LSE directly
      if (g < G) {
        const float inv = 1.f / l;
        uint16_t* orow = a.o + b * a.ldo + (gg * G + g) * RVO;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int col = 8 * j + 2 * tq;
          if (col < RVO) *reinterpret_cast<uint32_t*>(orow + col) = pack_bf16x2(oacc[j][0] * inv, oacc[j][1] * inv);
        }
        if (tq == 0 && a.lse) a.lse[b * a.Nh + gg * G + g] = (m + log2f(l)) / kLog2e3;
      }
    } else {
      const int piece = gw - wf;
      if (g < G) {
        float* dst = a.part + ((static_cast<int64_t>(b) * a.Nh + gg * G + g) * kMaxP3 + piece) * (RVO + 2);
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int col = 8 * j + 2 * tq;
          if (col < RVO) *reinterpret_cast<float2*>(dst + col) = make_float2(oacc[j][0], oacc[j][1]);
        }
        if (tq == 0) {
          dst[RVO] = m;
          dst[RVO + 1] = l;
        }
      }
      __syncwarp();
      int lastw = 0;
      if (lane == 0) {
        __threadfence();
        lastw = atomicAdd(&a.counters[p], 1) == pieces - 1;
      }
      lastw = __shfl_sync(0xffffffffu, lastw, 0);
      if (lastw) {
        __threadfence();
        // LSE merge of the pieces, lane-parallel over pieces: lane q holds piece q's (m, l) and
        // weight 2^(m_q - M) (chunks of 32 pieces), broadcast by shuffle into the column sums
        for (int gi = 0; gi < G; ++gi) {
          const float* hp = a.part + (static_cast<int64_t>(b) * a.Nh + gg * G + gi) * kMaxP3 * (RVO + 2);
          float M = -INFINITY;
          for (int q = lane; q < pieces; q += 32) M = fmaxf(M, __ldcg(hp + q * (RVO + 2) + RVO));
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
          float L = 0.f;
          for (int q = lane; q < pieces; q += 32) {
            const float ms = __ldcg(hp + q * (RVO + 2) + RVO);
            L += (ms == -INFINITY ? 0.f : exp2f(ms - M)) * __ldcg(hp + q * (RVO + 2) + RVO + 1);
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
          const float inv = 1.f / L;
          for (int col = lane; col < RVO; col += 32) {
            float O = 0.f;
            for (int q0 = 0; q0 < pieces; q0 += 32) {
              const int q = q0 + lane;
              const float ms = q < pieces ? __ldcg(hp + q * (RVO + 2) + RVO) : -INFINITY;
              const float fq = ms == -INFINITY ? 0.f : exp2f(ms - M);  // lane q's weight
              const int nq = min(32, pieces - q0);
#pragma unroll 8
              for (int u = 0; u < nq; ++u)
                O = fmaf(__shfl_sync(0xffffffffu, fq, u), __ldcg(hp + (q0 + u) * (RVO + 2) + col), O);
            }
            a.o[b * a.ldo + (gg * G + gi) * RVO + col] = f32_to_bf16_bits(O * inv);
          }
          if (lane == 0 && a.lse) a.lse[b * a.Nh + gg * G + gi] = (M + log2f(L)) / kLog2e3;
        }
        if (lane == 0) a.counters[p] = 0;
      }
    }
    reset();
    new_piece = true;
  }
}

// ------------------------------------------------------------------ host
template <int RK, int RK1>
static cudaError_t launch3_t(const DecodeAttnArgs& a, cudaStream_t stream) {
  using C = DA3<RK>;
  const size_t smem = static_cast<size_t>(kW3) * C::WARP_BYTES;
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_attn3_kernel<RK, RK1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // as many warps as fit one per SM, but no more than 64 per (sequence, KV head) pair
  const int pairs = a.B * a.Nkv;
  int grid = num_sms();
  const int64_t wmax = static_cast<int64_t>(pairs) * 64;
  if (static_cast<int64_t>(grid) * kW3 > wmax) grid = static_cast<int>((wmax + kW3 - 1) / kW3);
  prof_mark(stream, true, kProfAttnDecode);
  static const int q_once = knob("ZDC_V3_QONCE", 1);  // q copied with a piece's first tile only
  cudaError_t e = launch_k(decode_attn3_kernel<RK, RK1>, dim3(grid), dim3(kW3 * 32), smem, stream, g_pdl, a, grid * kW3,
                           q_once);
  prof_mark(stream, false, kProfAttnDecode);
  ++g_launches;
  return e;
}

template <int RK>
static cudaError_t launch3_r1(const DecodeAttnArgs& a, cudaStream_t s) {
  const int r1 = a.k1 ? a.rk1 : 0;
  switch (r1) {
    case 0: return launch3_t<RK, 0>(a, s);
    case 16: return launch3_t<RK, 16>(a, s);
    case 32: if constexpr (RK >= 32) return launch3_t<RK, 32>(a, s); else return cudaErrorNotSupported;
    case 64: if constexpr (RK >= 64) return launch3_t<RK, 64>(a, s); else return cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
  }
}

bool decode3_supported(const DecodeAttnArgs& a) {
  const int G = a.Nkv > 0 ? a.Nh / a.Nkv : 0;
  if (a.kv_fp8 || !a.counters || !a.part || a.B < 1 || a.B > 128) return false;
  if (G < 1 || G > 8 || a.Nh % a.Nkv != 0) return false;
  if (a.rk != a.rv || (a.rk != 32 && a.rk != 64 && a.rk != 96)) return false;
  if (a.k1 && (a.rk1 != a.rv1 || (a.rk1 != 16 && a.rk1 != 32 && a.rk1 != 64) || a.rk1 > a.rk)) return false;
  if (a.ldq % 8 != 0) return false;
  return true;
}

cudaError_t launch_decode_attention3(const DecodeAttnArgs& a, cudaStream_t s) {
  if (!decode3_supported(a)) return cudaErrorNotSupported;
  switch (a.rk) {
    case 32: return launch3_r1<32>(a, s);
    case 64: return launch3_r1<64>(a, s);
    case 96: return launch3_r1<96>(a, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace zdc
