// attn_mma.cuh — decode attention on the legacy warp MMA (mma.sync m16n8k16, bf16 in, f32
// accumulate) for the HBM-bound decode kernels (decode_attn3.cu, the fused layer-step): the tensor
// cores only take the score / PV dot products off the issue slots.  Queries sit on M (G <= 8 heads
// of a KV group in rows 0..G-1, rows 8..15 zero), keys / value columns on N, so
//   S^T[16][8 keys] = Q[16][16 k] . K'^T[16 k][8 keys],   O[16][8 cols] += P[16][16 keys] . V'[16 keys][8 cols]
// (Eqs. 2-3: s = Q'.K'/sqrt(d_h), online softmax, P rounded to bf16
// before PV with l from the unrounded P -- the faithful rounding points of DESIGN.md §4.3).
#pragma once
#include "common.cuh"

namespace zdc {

// d += A . B, m16n8k16, bf16 inputs, f32 accumulators
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
               "{%0, %1, %2, %3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// One 32-key pass of a warp over a tile of width W (a pool-0 row: RK, a pool-1 row: r^u):
//   S^T[16 (heads g < G, rest zero)][8 keys] = Q[16][16 k] . K'^T[16 k][8 keys]  per n-tile, k-step
//   O  [16][8 cols]                 += P[16][16 keys] . V'[16 keys][8 cols]
// lane = 4 g + t holds row g of every accumulator (columns 2t, 2t + 1 of each 8-wide n-tile); the
// S accumulators of two key n-tiles, rounded to bf16, are the P fragment of one PV k-step.  K' /
// V' fragments come straight from the row-major tiles with ldmatrix (V' transposed).
template <int W, int NT, int KSQ>
__device__ __forceinline__ void attn3_pass(uint32_t kb, uint32_t vb, int np, int lane, const uint32_t (&qa)[KSQ][2],
                                           float scl, float& m, float& l, float (&oacc)[NT][4]) {
  constexpr int KS = W / 16, NTW = W / 8;
  const int tq = lane & 3;
  float sacc[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
  // lane's ldmatrix row / column offsets (bytes) of the K' fragments: n-tile 2jp + (lane >> 4)
  const uint32_t krow = static_cast<uint32_t>((8 * (lane >> 4) + (lane & 7)) * W * 2 + ((lane >> 3) & 1) * 16);
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
    for (int jp = 0; jp < 2; ++jp) {
      uint32_t b0, b1, b2, b3;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                   : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                   : "r"(kb + krow + static_cast<uint32_t>(jp * 16 * W * 2 + ks * 32)));
      mma_bf16_16816(sacc[2 * jp], qa[ks][0], 0u, qa[ks][1], 0u, b0, b1);
      mma_bf16_16816(sacc[2 * jp + 1], qa[ks][0], 0u, qa[ks][1], 0u, b2, b3);
    }
  }
  // online softmax of row g over the 32 keys (4 lanes per row), log2 domain
  float x[4][2];
  float tm = -INFINITY;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      x[j][e] = 8 * j + 2 * tq + e < np ? sacc[j][e] * scl : -INFINITY;
      tm = fmaxf(tm, x[j][e]);
    }
  tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 1));
  tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 2));
  const float mn = fmaxf(m, tm);
  const float alpha = exp2f(m - mn);  // 0 on the first pass of a piece
  float ps = 0.f;
  uint32_t pa[2][2];  // P fragments of the two 16-key k-steps (row g; rows g + 8 zero)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float p0 = exp2f(x[j][0] - mn), p1 = exp2f(x[j][1] - mn);
    ps += p0 + p1;
    pa[j >> 1][j & 1] = pack_bf16x2(p0, p1);  // P rounded to bf16 before PV (l from the unrounded P)
  }
  ps += __shfl_xor_sync(0xffffffffu, ps, 1);
  ps += __shfl_xor_sync(0xffffffffu, ps, 2);
  l = l * alpha + ps;
  m = mn;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    oacc[j][0] *= alpha;
    oacc[j][1] *= alpha;
  }
  // PV over the first W / 8 output n-tiles (a pool-1 row adds to its first r^u dims only)
  const uint32_t vrow = static_cast<uint32_t>((lane & 15) * W * 2 + (lane >> 4) * 16);
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
    for (int jn = 0; jn < NTW; jn += 2) {
      uint32_t b0, b1, b2, b3;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                   : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                   : "r"(vb + vrow + static_cast<uint32_t>(kk * 16 * W * 2 + jn * 16)));
      mma_bf16_16816(oacc[jn], pa[kk][0], 0u, pa[kk][1], 0u, b0, b1);
      mma_bf16_16816(oacc[jn + 1], pa[kk][0], 0u, pa[kk][1], 0u, b2, b3);
    }
  }
}

}  // namespace zdc
