// decode_cluster.cuh — the decode layer-step (SURVEY.md §8(a) a1, a2, a3, a5 for one new token per
// sequence) as ONE kernel with one thread-block CLUSTER per KV group and no grid barrier.
//
// Why: the persistent kernel of decode_fused.cuh splits the layer by rows across all SMs, so the
// attention of a head needs Q' rows computed anywhere on the chip (grid barrier 1) and the output
// projection needs every head's O' (grid barrier 2), and its CUDA-core GEMVs cap each SM at
// ~45 GB/s of weights (profiles/r01/NOTES.md).  Everything a KV group g needs, however, is local
// to g: its G query heads' Q' come from G·r rows of W_QKV, its new K'/V' from 2r rows (Eq. 1 on
// the folded weights), its attention reads only g's cached rows (Eqs. 2-3), and its
// share of y = Σ_h O'^h W_O^{R,h} (Eq. 4) needs only its own heads' O'.  So one cluster of
// C CTAs per group does the whole layer for that group, and both projections run on the tensor
// cores (tcgen05.mma, M = 128 weight rows, N = 16 >= B sequences, FP32 accumulators in TMEM):
//
//   phase 1  a1 + a2   split-K: CTA `rank` multiplies all (G+2)·r of the group's W_QKV rows by
//                      x[:, rank·d/C : (rank+1)·d/C]; the FP32 partial sums go to every CTA of
//                      the cluster (st.async into DSMEM, completing bytes on their mbarrier); each
//                      CTA adds the C partials in rank order -> Q'/K'/V' (bf16); rank 0 appends
//                      the new K'/V' row to the cache at position len
//   phase 2  a3        each CTA: 1/C of the cached rows (the last rank adds the new row), online
//                      softmax on CUDA cores; its unnormalised partial (m, l, o) per query head is
//                      sent to every CTA of the cluster
//   phase 3  a5        each CTA LSE-merges the C partials -> O' (bf16, the MMA's B operand), then
//                      M-tiles of 128 output rows n: y[n] += Σ_{h in g} W_O^{R,h}[:, n] · O'^h from
//                      the group-major decode copy of W_O (contiguous 16 KB tiles); the FP32 sums
//                      over the N_kv groups meet in a global accumulator (red.add) and the last
//                      group to finish a slice of rows writes the bf16 y and re-zeroes it
//
// Warp roles: warps 0-7 consumers (x / O' operand staging, TMEM read-back, attention, merges),
// warp 8 lane 0 the producer (every byte the CTA reads, TMA / bulk copies into a ring of slots in
// consumption order; the weight stream starts before the programmatic-dependent-launch wait),
// warp 9 lane 0 the MMA issuer (TMEM allocated / freed by warp 9).
//
// Rounding points: Q'/K'/V' to bf16 after phase 1; P = exp(s - m) to bf16 before
// PV with l from the unrounded P; O' to bf16 after the merge; y to bf16 (the FP32 sum over the
// groups is accumulated in an order-dependent way: rounding of the f32 sum only).
#pragma once
#include "decode_fused.cuh"

namespace zdc {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
// shared::cta address -> the same offset in CTA `rank` of this cluster (shared::cluster window)
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// 4-byte store into a (possibly remote) CTA's shared memory, completing 4 transaction bytes on
// that CTA's mbarrier
__device__ __forceinline__ void st_async_f32(uint32_t raddr, float v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
               "r"(__float_as_uint(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred P;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, "
      "0, P;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {
  }
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Byte offset of element (row, k) in a K-major operand tile with `swb`-byte swizzle (128 / 64 /
// 32: the row width in bytes of the swizzle atom, 8 rows per atom; CUTLASS Swizzle<3|2|1,4,3>:
// 16-byte unit index XOR the address bits [7, 10)); the tile base is 1024-byte aligned.
__device__ __forceinline__ uint32_t kmajor_off(int row, int k, int swb) {
  const uint32_t byte = static_cast<uint32_t>(row) * swb + static_cast<uint32_t>(k) * 2;
  return byte ^ (((byte >> 7) & (swb / 16 - 1)) << 4);
}
__host__ __device__ constexpr uint32_t sw_layout(int swb) { return swb == 128 ? kSw128 : swb == 64 ? kSw64 : kSw32; }

// compile-time geometry of one instance
template <int RK, int G>
struct CG {
  static constexpr int K3 = G * RK;                    // a5 reduction length (the group's O' dims)
  static constexpr int NV1 = (G + 2) * RK;             // projection rows of the group (Q' | K' | V')
  static constexpr int NMT1 = (NV1 + 127) / 128;       // phase-1 M-tiles
  static constexpr int ST1 = NV1 * 128;                // phase-1 stage: NV1 rows x 64 K (SW128)
  static constexpr int OVR1 = NMT1 * 128 * 128 - ST1;  // the last M-tile's MMA reads past the stage
  static constexpr int KB3 = K3 >= 64 ? 64 : K3;       // phase-3 k-block width (elements)
  static constexpr int NKB3 = K3 / KB3;
  static constexpr int SW3 = KB3 * 2;                  // its swizzle width (bytes): 128 / 64 / 32
  static constexpr int ST3 = 128 * KB3 * 2;            // phase-3 stage: 128 rows x KB3
  static constexpr int KV = 4 * 32 * RK;               // 32 cached K' + V' rows
  static constexpr int MX = ST1 > ST3 ? ST1 : ST3;
  static constexpr int SB = ((MX > KV ? MX : KV) + 1023) / 1024 * 1024;
  static constexpr int RPS = SB / (4 * RK) / 32 * 32;  // cached K'/V' rows per slot
};

// shared-memory layout (offsets from the 1024-aligned base), used by host and device
struct ClusterSmem {
  size_t xt, ot, xq, pq, wst, pxs, nrow, bars, total;
};
__host__ __device__ __forceinline__ size_t align_to(size_t v, size_t a) { return (v + a - 1) / a * a; }
template <int NB, int RK, int G>
__host__ __device__ __forceinline__ ClusterSmem cluster_smem(int C, int KC, int nslot) {
  using Q = CG<RK, G>;
  ClusterSmem m;
  m.xt = align_to(static_cast<size_t>(nslot) * Q::SB + Q::OVR1, 1024);       // x operand [16][KC]
  m.ot = align_to(m.xt + static_cast<size_t>(KC) * 32, 1024);                 // O' operand [16][K3]
  m.xq = align_to(m.ot + static_cast<size_t>(Q::K3) * 32, 16);                // [NB][NV1] Q'|K'|V'
  m.pq = m.xq + align_to(static_cast<size_t>(NB) * Q::NV1 * 4, 16);           // [C][NB][NV1] partials
  m.wst = m.pq + align_to(static_cast<size_t>(C) * NB * Q::NV1 * 4, 16);      // [kNW][G][RK+2]
  m.pxs = m.wst + align_to(static_cast<size_t>(kNW) * G * (RK + 2) * 4, 16);  // [C][NB][G][RK+2]
  m.nrow = m.pxs + align_to(static_cast<size_t>(C) * NB * G * (RK + 2) * 4, 16);
  m.bars = m.nrow + align_to(static_cast<size_t>(2) * RK * 2, 16);
  m.total = m.bars + (2 * static_cast<size_t>(nslot) + 8) * 8 + 16;
  return m;
}

// virtual projection row i of group g -> row of W_QKV^T: [0, G r) the group's query heads,
// [G r, (G+1) r) its K' dims, [(G+1) r, (G+2) r) its V' dims
template <int RK, int G>
__device__ __forceinline__ int qkv_row(const DecClusterArgs& a, int g, int i) {
  if (i < G * RK) return g * G * RK + i;
  if (i < (G + 1) * RK) return a.nq + g * RK + (i - G * RK);
  return a.nq + a.nk + g * RK + (i - (G + 1) * RK);
}

static constexpr int kClusterThreads = kNC + 64;

// bulk L2 prefetch of [p, p + bytes) in 32 KB requests (16-byte granules)
__device__ __forceinline__ void l2_prefetch_range(const void* p, int64_t bytes) {
  const uint8_t* c = static_cast<const uint8_t*>(p);
  for (int64_t o = 0; o < bytes; o += 32768) {
    const int64_t n = bytes - o < 32768 ? bytes - o : 32768;
    l2_prefetch(c + o, static_cast<uint32_t>(n & ~static_cast<int64_t>(15)));
  }
}

// attn_rows over up to 32 R key rows with R independent row sets per lane (lane j holds rows
// j, 32 + j, ...): R dot products, one max / sum pass over all of them and R interleaved PV
// chains, so a warp keeps R times more independent work in flight than attn_rows.
template <int RK, int G, int R>
__device__ __forceinline__ void attn_rows_r(const uint16_t* Ks, const uint16_t* Vs, int np, const float* qf, float scl,
                                            float (&m)[G], float (&l)[G], float (&o)[G][Dims2<RK>::DPL], int lane) {
  constexpr int UK = RK / 8, DPL = Dims2<RK>::DPL;
  float s[R][G];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int gi = 0; gi < G; ++gi) s[i][gi] = 0.f;
  const int rot = lane % UK;  // rotated chunk order: the 32 rows of a set hit distinct banks
#pragma unroll
  for (int kk = 0; kk < UK; ++kk) {
    int kc = kk + rot;
    if (kc >= UK) kc -= UK;
    float kf[R][8];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int row = i * 32 + lane;
      if (row < np)
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(Ks + row * RK + kc * 8), kf[i]);
      else
#pragma unroll
        for (int e = 0; e < 8; ++e) kf[i][e] = 0.f;
    }
#pragma unroll
    for (int gi = 0; gi < G; ++gi) {
      const float4 q0 = *reinterpret_cast<const float4*>(qf + gi * RK + kc * 8);
      const float4 q1 = *reinterpret_cast<const float4*>(qf + gi * RK + kc * 8 + 4);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        float x = s[i][gi];
        x = fmaf(q0.x, kf[i][0], x);
        x = fmaf(q0.y, kf[i][1], x);
        x = fmaf(q0.z, kf[i][2], x);
        x = fmaf(q0.w, kf[i][3], x);
        x = fmaf(q1.x, kf[i][4], x);
        x = fmaf(q1.y, kf[i][5], x);
        x = fmaf(q1.z, kf[i][6], x);
        x = fmaf(q1.w, kf[i][7], x);
        s[i][gi] = x;
      }
    }
  }
  float pb[R][G];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      s[i][gi] = i * 32 + lane < np ? s[i][gi] * scl : -INFINITY;
      mx = fmaxf(mx, s[i][gi]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float mn = fmaxf(m[gi], mx);  // finite: np >= 1
    const float alpha = exp2f(m[gi] - mn);
    float ps = 0.f;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const float p = i * 32 + lane < np ? exp2f(s[i][gi] - mn) : 0.f;
      ps += p;
      pb[i][gi] = __bfloat162float(__float2bfloat16_rn(p));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
    l[gi] = l[gi] * alpha + ps;
    m[gi] = mn;
#pragma unroll
    for (int e = 0; e < DPL; ++e) o[gi][e] *= alpha;
  }
  // o += P V' (lane-owned dims); row sets are independent FMA chains
  const int full_sets = np >> 5;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    if (i < full_sets) {
#pragma unroll 8
      for (int j = 0; j < 32; ++j) pv_row<RK, G>(Vs + i * 32 * RK, j, lane, pb[i], o);
    } else if (i * 32 < np) {
      for (int j = 0; j < np - i * 32; ++j) pv_row<RK, G>(Vs + i * 32 * RK, j, lane, pb[i], o);
    }
  }
}  // 8 consumer warps, producer warp, MMA warp

template <int NB, int RK, int G>
__global__ void __launch_bounds__(kClusterThreads, 1)
    decode_cluster_kernel(const __grid_constant__ CUtensorMap tm_wo, const DecClusterArgs a) {
  using Q = CG<RK, G>;
  constexpr int DPL = Dims2<RK>::DPL;
  constexpr int K3 = Q::K3, NV1 = Q::NV1, SB = Q::SB, RPS = Q::RPS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nslot = a.nslot, C = a.C, d = a.d, KC = d / C, NKB1 = KC / 64, WA = a.attn_warps;
  const ClusterSmem L0 = cluster_smem<NB, RK, G>(C, KC, nslot);
  uint8_t* ring = smem;
  uint8_t* xt = smem + L0.xt;
  uint8_t* ot = smem + L0.ot;
  float* xq = reinterpret_cast<float*>(smem + L0.xq);
  float* pq = reinterpret_cast<float*>(smem + L0.pq);
  float* wst = reinterpret_cast<float*>(smem + L0.wst);
  float* pxs = reinterpret_cast<float*>(smem + L0.pxs);
  uint16_t* nrow = reinterpret_cast<uint16_t*>(smem + L0.nrow);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L0.bars);
  uint64_t* empty = full + nslot;
  uint64_t* lenbar = empty + nslot;
  uint64_t* xbar1 = lenbar + 1;   // phase-1 partial sums of every CTA arrived
  uint64_t* xbar2 = xbar1 + 1;    // phase-2 attention partials of every CTA arrived
  uint64_t* xready = xbar2 + 1;   // x operand staged
  uint64_t* oready = xready + 1;  // O' operand staged
  uint64_t* mma1 = oready + 1;    // phase-1 accumulators complete
  uint64_t* mma3 = mma1 + 1;      // phase-3 accumulators complete
  int* s_len = reinterpret_cast<int*>(mma3 + 2);
  int* s_flag = s_len + 1;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_len + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int rank = static_cast<int>(cluster_ctarank());
  const int g = blockIdx.x / C;  // KV group of this cluster
  // phase 3 rows [n0, n1) of this CTA: 128-row tiles
  int per3 = (d + C - 1) / C;
  per3 = (per3 + 127) / 128 * 128;
  const int n0 = min(d, rank * per3), n1 = min(d, n0 + per3);
  const int nmt3 = (n1 - n0 + 127) / 128;

  if (tid == kNC) {
    for (int s = 0; s < nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(lenbar, 1);
    mbar_init(xbar1, 1);
    mbar_init(xbar2, 1);
    mbar_init(xready, 1);
    mbar_init(oready, 1);
    mbar_init(mma1, 1);
    mbar_init(mma3, 1);
    fence_barrier_init();
  }
  if (warp == kNW + 1) tmem_alloc(s_tmem, a.tmem_cols);
  tc_fence_before();
  // every CTA's mbarriers exist before any CTA of the cluster writes into its shared memory
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  if (tid == 0) ZDC_STAMP(0);

  if (warp == kNW) {
    // ================= producer: every byte this CTA reads, in consumption order
    if (lane == 0) {
      tma_prefetch_desc(&tm_wo);
      uint32_t k = 0;
      auto take = [&](uint32_t bytes) -> int {
        const int s = static_cast<int>(k % nslot);
        if (k >= static_cast<uint32_t>(nslot)) mbar_wait(&empty[s], ((k / nslot) & 1) ^ 1);
        ++k;
        mbar_arrive_expect_tx(&full[s], bytes);
        return s;
      };
      // phase 1: k-blocks [rank NKB1, (rank+1) NKB1) of the group's pre-swizzled W_QKV tiles
      // (NV1 rows x 64 K each, contiguous: one bulk copy per stage; static weights)
      const uint8_t* wq = reinterpret_cast<const uint8_t*>(a.wqd) +
                          (static_cast<int64_t>(g) * (d / 64) + rank * NKB1) * Q::ST1;
      // Everything past the first ring-full is also requested into L2 up front (bulk prefetch):
      // HBM then streams this CTA's whole working set at full rate while the ring refills from L2,
      // instead of idling whenever the ring holds data the consumers cannot use yet (the cached
      // rows wait for the phase-1 exchange, W_O for the attention merge).
      const int pf = a.l2_prefetch;
      for (int kb = 0; kb < NKB1; ++kb) {
        const int s = take(Q::ST1);
        bulk_g2s(ring + static_cast<size_t>(s) * SB, wq + static_cast<int64_t>(kb) * Q::ST1, Q::ST1, &full[s]);
        if (kb + 1 == min(nslot, NKB1) && (pf & 1) && NKB1 > nslot)
          l2_prefetch_range(wq + static_cast<int64_t>(nslot) * Q::ST1, static_cast<int64_t>(NKB1 - nslot) * Q::ST1);
      }
      ZDC_STAMP(8);
      mbar_wait(lenbar, 0);  // the cache length, read by a consumer after the PDL wait
      const int L = *s_len;
      const int chunk = ((L + C - 1) / C + 31) / 32 * 32;
      const int s0 = min(L, rank * chunk), e0 = min(L, s0 + chunk);
      // issued once the last phase-1 stage is in flight: the rest of the stream queues behind it
      if (pf & 2)
        for (int b = 0; b < a.B && e0 > s0; ++b) {
          const int64_t row0 = (static_cast<int64_t>(b) * a.Nkv + g) * a.S_cap + s0;
          l2_prefetch_range(a.kc + row0 * RK, static_cast<int64_t>(e0 - s0) * RK * 2);
          l2_prefetch_range(a.vc + row0 * RK, static_cast<int64_t>(e0 - s0) * RK * 2);
        }
      if (pf & 4)
        l2_prefetch_range(a.wod + (static_cast<int64_t>(g) * d + n0) * K3, static_cast<int64_t>(n1 - n0) * K3 * 2);
      for (int b = 0; b < a.B; ++b) {  // phase 2: this CTA's cached K'/V' rows
        const int64_t row0 = (static_cast<int64_t>(b) * a.Nkv + g) * a.S_cap;
        for (int p = s0; p < e0; p += RPS) {
          const int np = min(RPS, e0 - p);
          const uint32_t bytes = static_cast<uint32_t>(np) * RK * 2u;
          const int s = take(2 * bytes);
          uint8_t* dst = ring + static_cast<size_t>(s) * SB;
          bulk_g2s(dst, a.kc + (row0 + p) * RK, bytes, &full[s]);
          bulk_g2s(dst + RPS * RK * 2, a.vc + (row0 + p) * RK, bytes, &full[s]);
        }
      }
      ZDC_STAMP(9);
      for (int mt = 0; mt < nmt3; ++mt)  // phase 3: W_O decode copy, 128 rows x KB3 per stage
        for (int kb = 0; kb < Q::NKB3; ++kb) {
          const int s = take(Q::ST3);
          tma_load_2d(ring + static_cast<size_t>(s) * SB, &tm_wo, &full[s], kb * Q::KB3, g * d + n0 + mt * 128);
        }
      ZDC_STAMP(10);
    }
  } else if (warp == kNW + 1) {
    // ================= MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, 16, 0, 0);
      uint32_t k = 0;
      mbar_wait(xready, 0);
      tc_fence_after();
      for (int kb = 0; kb < NKB1; ++kb) {
        const int s = static_cast<int>(k % nslot);
        mbar_wait(&full[s], (k / nslot) & 1);
        ++k;
        tc_fence_after();
        const uint32_t a0 = smem_u32(ring + static_cast<size_t>(s) * SB), b0 = smem_u32(xt + kb * 2048);
#pragma unroll
        for (int mt = 0; mt < Q::NMT1; ++mt)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_ss(tmem + mt * 16, make_sdesc(a0 + mt * 16384 + kk * 32, 16, 1024, kSw128),
                         make_sdesc(b0 + kk * 32, 16, 1024, kSw128), idesc, (kb | kk) != 0 ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(mma1);
      // skip the attention slots (consumed by the consumer warps)
      mbar_wait(lenbar, 0);
      const int L = *s_len;
      const int chunk = ((L + C - 1) / C + 31) / 32 * 32;
      const int s0 = min(L, rank * chunk), e0 = min(L, s0 + chunk);
      k += static_cast<uint32_t>(a.B * ((e0 - s0 + RPS - 1) / RPS));
      mbar_wait(oready, 0);
      tc_fence_after();
      const uint32_t ob = smem_u32(ot);
      for (int mt = 0; mt < nmt3; ++mt)
        for (int kb = 0; kb < Q::NKB3; ++kb) {
          const int s = static_cast<int>(k % nslot);
          mbar_wait(&full[s], (k / nslot) & 1);
          ++k;
          tc_fence_after();
          const uint32_t a0 = smem_u32(ring + static_cast<size_t>(s) * SB);
#pragma unroll
          for (int kk = 0; kk < Q::KB3 / 16; ++kk)
            umma_bf16_ss(tmem + mt * 16, make_sdesc(a0 + kk * 32, 16, 8 * Q::SW3, sw_layout(Q::SW3)),
                         make_sdesc(ob + kb * 16 * Q::SW3 + kk * 32, 16, 8 * Q::SW3, sw_layout(Q::SW3)), idesc,
                         (kb | kk) != 0 ? 1u : 0u);
          umma_commit(&empty[s]);
        }
      umma_commit(mma3);
    }
  } else {
    // ================= consumers (warps 0..kNW-1)
    pdl_wait();
    pdl_trigger();
    if (tid == 0) {
      ZDC_STAMP(14);
      const int L0 = *a.len_ptr;
      *s_len = min(L0, a.S_cap - 1);  // a full cache rewrites its last row (flagged)
      if (L0 >= a.S_cap && a.err) *a.err = 1;
      mbar_arrive(lenbar);
      mbar_arrive_expect_tx(xbar1, static_cast<uint32_t>(C * a.B * NV1 * 4));
      mbar_arrive_expect_tx(xbar2, static_cast<uint32_t>(C * a.B * G * (RK + 2) * 4));
    }
    {  // x[:, rank KC : (rank+1) KC] -> the phase-1 B operand [16][KC] (K-major, SW128), zero rows >= B
      const int u8 = KC >> 3;
      for (int i = tid; i < 16 * u8; i += kNC) {
        const int b = i / u8, u = i - b * u8, kk = u * 8;
        const uint4 v = b < a.B ? __ldcg(reinterpret_cast<const uint4*>(a.x + b * a.ldx + rank * KC) + u)
                                : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(xt + (kk >> 6) * 2048 + kmajor_off(b, kk & 63, 128)) = v;
      }
    }
    fence_proxy_async_smem();
    consumer_sync();
    if (tid == 0) {
      mbar_arrive(xready);
      ZDC_STAMP(1);
    }
    const int L = *s_len;
    const uint32_t pq_s = smem_u32(pq), xbar1_s = smem_u32(xbar1);
    const uint32_t pxs_s = smem_u32(pxs), xbar2_s = smem_u32(xbar2);

    // ---- phase 1 read-back: this CTA's partial sums -> every CTA's pq[rank]
    mbar_wait(mma1, 0);
    tc_fence_after();
    for (int mt = warp >> 2; mt < Q::NMT1; mt += 2) {
      uint32_t r[16];
      tmem_ld16(tmem + ((static_cast<uint32_t>(warp & 3) * 32) << 16) + mt * 16, r);
      tc_wait_ld();
      const int row = mt * 128 + (warp & 3) * 32 + lane;
      if (row < NV1) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (b < a.B) {
            const uint32_t off = static_cast<uint32_t>(((rank * NB + b) * NV1 + row) * 4);
            for (int rr = 0; rr < C; ++rr)
              st_async_f32(mapa_rank(pq_s + off, rr), __uint_as_float(r[b]), mapa_rank(xbar1_s, rr));
          }
      }
    }
    tc_fence_before();
    if (tid == 0) ZDC_STAMP(2);
    mbar_wait_cluster(xbar1, 0);
    if (tid == 0) ZDC_STAMP(3);
    // Q'/K'/V' = bf16(sum of the C partials in rank order); rank 0 appends K'/V' (a2)
    for (int i = tid; i < a.B * NV1; i += kNC) {
      const int b = i / NV1, j = i - b * NV1;
      float v = 0.f;
      for (int rr = 0; rr < C; ++rr) v += pq[(rr * NB + b) * NV1 + j];
      const uint16_t h = f32_to_bf16_bits(v);
      xq[b * NV1 + j] = __uint_as_float(static_cast<uint32_t>(h) << 16);
      if (rank == 0 && j >= G * RK) {
        const int c = (j - G * RK) % RK;
        uint16_t* dst = j < (G + 1) * RK ? a.kc : a.vc;
        dst[((static_cast<int64_t>(b) * a.Nkv + g) * a.S_cap + L) * RK + c] = h;
      }
    }
    consumer_sync();

    // ---- phase 2: a3 partial over this CTA's chunk of cached rows (+ the new row on the last rank)
    uint32_t k = static_cast<uint32_t>(NKB1);  // ring sequence number of the first attention slot
    const float scl = a.scale * kLog2eF;
    const int chunk = ((L + C - 1) / C + 31) / 32 * 32;
    const int s0 = min(L, rank * chunk), e0 = min(L, s0 + chunk);
    const int ns = (e0 - s0 + RPS - 1) / RPS;
    const bool has_new = rank == C - 1;
    for (int b = 0; b < a.B; ++b) {
      const float* qf = xq + b * NV1;  // this sequence's G query heads (bf16 values in f32)
      if (has_new && warp == 0) {
        for (int c = lane; c < RK; c += 32) {
          nrow[c] = f32_to_bf16_bits(qf[G * RK + c]);
          nrow[RK + c] = f32_to_bf16_bits(qf[(G + 1) * RK + c]);
        }
        __syncwarp();
      }
      float m[G], l[G], o[G][DPL];
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        m[gi] = -INFINITY;
        l[gi] = 0.f;
#pragma unroll
        for (int i = 0; i < DPL; ++i) o[gi][i] = 0.f;
      }
      if (warp < WA) {
        // slot k + t is consumed by warp t % WA (WA divides the slot count: every wait is for the
        // use right after the one this warp observed on that slot)
        for (int t = warp; t < ns; t += WA) {
          const uint32_t kk = k + t;
          const int s = static_cast<int>(kk % nslot);
          mbar_wait(&full[s], (kk / nslot) & 1);
          const uint16_t* Ks = reinterpret_cast<const uint16_t*>(ring + static_cast<size_t>(s) * SB);
          const int nr = min(RPS, e0 - (s0 + t * RPS));
          constexpr int R3 = RPS >= 96 ? 3 : RPS >= 64 ? 2 : 1;
          for (int j = 0; j < nr; j += 32 * R3)
            attn_rows_r<RK, G, R3>(Ks + j * RK, Ks + (RPS + j) * RK, min(32 * R3, nr - j), qf, scl, m, l, o, lane);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
      }
      k += ns;
      if (has_new && warp == 0) attn_rows<RK, G>(nrow, nrow + RK, 1, qf, scl, m, l, o, lane);
      float* ws = wst + warp * G * (RK + 2);
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          const int c = RK >= 32 ? lane * DPL + i : lane;
          if (c < RK) ws[gi * (RK + 2) + c] = o[gi][i];
        }
        if (lane == 0) {
          ws[gi * (RK + 2) + RK] = m[gi];
          ws[gi * (RK + 2) + RK + 1] = l[gi];
        }
      }
      consumer_sync();
      // CTA merge of the warp states -> this CTA's partial of (b, gi) -> every CTA's pxs[rank][b]
      for (int i = tid; i < G * (RK + 2); i += kNC) {
        const int gi = i / (RK + 2), c = i - gi * (RK + 2);
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kNW; ++w) M = fmaxf(M, wst[(w * G + gi) * (RK + 2) + RK]);
        float v = c == RK ? M : 0.f;
        if (c != RK && M != -INFINITY) {
#pragma unroll
          for (int w = 0; w < kNW; ++w) {
            const float* e = wst + (w * G + gi) * (RK + 2);
            v = fmaf(e[c], exp2f(e[RK] - M), v);  // c == RK + 1: the row sum l
          }
        }
        const uint32_t off = static_cast<uint32_t>((((rank * NB + b) * G + gi) * (RK + 2) + c) * 4);
        for (int rr = 0; rr < C; ++rr) st_async_f32(mapa_rank(pxs_s + off, rr), v, mapa_rank(xbar2_s, rr));
      }
      consumer_sync();  // wst and nrow are reused by the next sequence
    }
    if (tid == 0) ZDC_STAMP(4);
    mbar_wait_cluster(xbar2, 0);
    if (tid == 0) ZDC_STAMP(5);

    // ---- LSE merge of the C partials -> O' (bf16) = the phase-3 B operand [16][K3] (K-major)
    for (int i = tid; i < 16 * K3; i += kNC) {
      const int b = i / K3, j = i - b * K3, gi = j / RK, c = j - gi * RK;
      float v = 0.f;
      if (b < a.B) {
        float M = -INFINITY;
        for (int rr = 0; rr < C; ++rr) M = fmaxf(M, pxs[((rr * NB + b) * G + gi) * (RK + 2) + RK]);
        float O = 0.f, Ls = 0.f;
        for (int rr = 0; rr < C; ++rr) {
          const float* e = pxs + ((rr * NB + b) * G + gi) * (RK + 2);
          const float f = e[RK] == -INFINITY ? 0.f : exp2f(e[RK] - M);
          O = fmaf(f, e[c], O);
          Ls = fmaf(f, e[RK + 1], Ls);
        }
        v = O / Ls;
        if (c == 0 && rank == 0 && a.lse) a.lse[b * a.Nh + g * G + gi] = (M + log2f(Ls)) / kLog2eF;
      }
      *reinterpret_cast<uint16_t*>(ot + (j / Q::KB3) * 16 * Q::SW3 + kmajor_off(b, j % Q::KB3, Q::SW3)) =
          f32_to_bf16_bits(v);
    }
    fence_proxy_async_smem();
    consumer_sync();
    if (tid == 0) {
      mbar_arrive(oready);
      ZDC_STAMP(6);
    }

    // ---- phase 3 read-back: y partial of this group -> the f32 accumulator
    mbar_wait(mma3, 0);
    tc_fence_after();
    for (int mt = warp >> 2; mt < nmt3; mt += 2) {
      uint32_t r[16];
      tmem_ld16(tmem + ((static_cast<uint32_t>(warp & 3) * 32) << 16) + mt * 16, r);
      tc_wait_ld();
      const int n = n0 + mt * 128 + (warp & 3) * 32 + lane;
      if (n < n1) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (b < a.B) atomicAdd(a.ybuf + static_cast<int64_t>(b) * d + n, __uint_as_float(r[b]));
      }
    }
    tc_fence_before();
    __threadfence();
    consumer_sync();
    if (tid == 0) {
      ZDC_STAMP(11);
      *s_flag = atomic_add_acq_rel(a.ycnt + rank, 1) == a.Nkv - 1;
    }
    consumer_sync();
    if (*s_flag) {
      // the last group to finish rows [n0, n1): y = bf16(sum), accumulator back to zero
      for (int i = tid; i < a.B * (n1 - n0); i += kNC) {
        const int b = i / (n1 - n0), n = n0 + (i - b * (n1 - n0));
        float* p = a.ybuf + static_cast<int64_t>(b) * d + n;
        a.y[b * a.ldy + n] = f32_to_bf16_bits(__ldcg(p));
        __stcg(p, 0.f);
      }
      if (tid == 0) {
        a.ycnt[rank] = 0;
        // every CTA of the grid has read the length: each group's rank-`rank` CTA passed both exchanges
        if (rank == 0) *a.len_ptr = L + 1;
      }
    }
    if (tid == 0) ZDC_STAMP(7);
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
  if (warp == kNW + 1) {
    tc_fence_after();
    tmem_dealloc(tmem, a.tmem_cols);
  }
}

// ------------------------------------------------------------------ host
template <int NB, int RK, int G>
inline bool cluster_config_t(DecClusterArgs& a, size_t* smem_out) {
  using Q = CG<RK, G>;
  constexpr size_t kSmemMax = 227 * 1024;
  if (a.C < 1 || a.d % (64 * a.C) != 0) return false;
  const int KC = a.d / a.C;
  const size_t fixed = cluster_smem<NB, RK, G>(a.C, KC, 0).total + 1024;  // + base alignment slack
  const int nslot = static_cast<int>((kSmemMax - std::min(fixed, kSmemMax)) / (Q::SB + 16));
  if (nslot < 2) return false;
  a.nslot = nslot;
  int wa = kNW;
  while (nslot % wa != 0) --wa;
  a.attn_warps = wa;
  int per3 = (a.d + a.C - 1) / a.C;
  per3 = (per3 + 127) / 128 * 128;
  const int cols = std::max(Q::NMT1, per3 / 128) * 16;
  int tc = 32;
  while (tc < cols) tc *= 2;
  if (tc > 512) return false;
  a.tmem_cols = tc;
  *smem_out = cluster_smem<NB, RK, G>(a.C, KC, nslot).total + 1024;
  return *smem_out <= kSmemMax;
}

template <int NB, int RK, int G>
inline cudaError_t launch_cluster_t(DecClusterArgs a, cudaStream_t stream) {
  using Q = CG<RK, G>;
  size_t smem = 0;
  if (!cluster_config_t<NB, RK, G>(a, &smem)) return cudaErrorNotSupported;
  CUtensorMap tw;
  if (!cluster_wo_tmap(&tw, a.wod, a.Nkv, a.d, Q::K3, Q::KB3)) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_cluster_kernel<NB, RK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.Nkv * a.C);
  cfg.blockDim = dim3(kClusterThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = a.C;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = g_pdl ? 2 : 1;
  prof_mark(stream, true, g_prof_class);
  cudaError_t e = cudaLaunchKernelEx(&cfg, decode_cluster_kernel<NB, RK, G>, tw, a);
  prof_mark(stream, false, g_prof_class);
  ++g_launches;
  return e;
}

// the number of clusters of C CTAs that fit at once (the cluster kernel needs all N_kv resident)
template <int NB, int RK, int G>
inline int cluster_capacity_t(const DecClusterArgs& a0, int C) {
  DecClusterArgs a = a0;
  a.C = C;
  size_t smem = 0;
  if (!cluster_config_t<NB, RK, G>(a, &smem)) return 0;
  if (cudaFuncSetAttribute(decode_cluster_kernel<NB, RK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
      cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * a.Nkv);
  cfg.blockDim = dim3(kClusterThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, decode_cluster_kernel<NB, RK, G>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

template <int NB, int RK, int G>
inline cudaError_t dispatch_cluster_t(const DecClusterArgs& a, int* cap_out, int C, cudaStream_t s) {
  if (cap_out) {
    *cap_out = cluster_capacity_t<NB, RK, G>(a, C);
    return cudaSuccess;
  }
  return launch_cluster_t<NB, RK, G>(a, s);
}

template <int NB, int RK>
inline cudaError_t dispatch_cluster_g(const DecClusterArgs& a, int* cap, int C, int G, cudaStream_t s) {
  switch (G) {
    case 1: return dispatch_cluster_t<NB, RK, 1>(a, cap, C, s);
    case 2: return dispatch_cluster_t<NB, RK, 2>(a, cap, C, s);
    case 4:
      if constexpr (RK * 4 <= 256) return dispatch_cluster_t<NB, RK, 4>(a, cap, C, s);
      return cudaErrorNotSupported;
    case 8:
      if constexpr (RK * 8 <= 256) return dispatch_cluster_t<NB, RK, 8>(a, cap, C, s);
      return cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
  }
}

template <int NB>
inline cudaError_t dispatch_cluster_r(const DecClusterArgs& a, int* cap, int C, int RK, int G, cudaStream_t s) {
  switch (RK) {
    case 16: return dispatch_cluster_g<NB, 16>(a, cap, C, G, s);
    case 32: return dispatch_cluster_g<NB, 32>(a, cap, C, G, s);
    case 64: return dispatch_cluster_g<NB, 64>(a, cap, C, G, s);
    case 128: return dispatch_cluster_g<NB, 128>(a, cap, C, G, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace zdc
