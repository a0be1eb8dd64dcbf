// decode_fused.cuh — the whole decode layer-step (SURVEY.md §8(a) a1, a2, a3, a5 for one new token
// per sequence, "Q^h is obtained from the input token, while K^h and V^h of all previous
// tokens are retrieved from the KVC") as ONE persistent kernel, one CTA per SM:
//
//   phase 1  a1 + a2   [Q'|K'|V'] = x W_QKV^R (Eq. 1 on the folded, truncated weights); Q' to
//                      staging, K'/V' of the new token straight into the cache at position len
//   grid barrier
//   phase 2  a3        split-K attention over the cached rows and the new row at head dim r
//                      (Eqs. 2-3, scale 1/sqrt(d_h)); one unnormalised partial (m, l, o) per
//                      (sequence, KV head, chunk) item; the last CTA to finish a chunk of a
//                      (sequence, KV head) LSE-merges its chunks -> O' (bf16) and the row LSE
//   grid barrier
//   phase 3  a5        y = O' W_O^R (Eq. 4 with the folded W_L), O' staged in shared memory
//
// Why one kernel: at B <= 8 a decode layer reads ~85 MB (c2) and the three separate kernels are
// each latency-bound at their start and tail.  Here a single producer thread per CTA streams
// every byte the CTA will read — its W_QKV rows, its K'/V' chunk rows, its W_O rows — through one
// ring of shared-memory slots with cp.async.bulk, in consumption order.  It never waits for the
// grid barriers (weights and cached rows do not depend on them), so HBM stays busy across the
// phase boundaries; only the consumers wait.
//
// Consumers: warps 0..kNW-1; ring slot sequence number k is consumed by warp k % kNW, which owns
// its own sub-ring of slots (ProducerCursor / ConsumerCursor) (every mbarrier wait is for the phase right after the last one
// the waiter observed; see profiles/r01/NOTES.md on parity aliasing).
//
// Rounding points (DESIGN.md §4 faithful mode): Q'/K'/V' to bf16 in phase 1; P = exp(s - m)
// rounded to bf16 before PV with l taken from the unrounded P; O' to bf16 after the merge; y to bf16.
#pragma once
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>

namespace zdc {

static constexpr float kLog2eF = 1.4426950408889634f;

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Grid barrier on a monotonic 64-bit arrival counter, called by ONE thread per CTA after a
// CTA-level barrier (the release is cumulative over the CTA's writes ordered by it, as in
// CUTLASS's generic barrier).  The arrival is a fire-and-forget red.release; the thread then
// polls with ld.acquire until the counter reaches `target` = base + k * n for the k-th barrier of
// this launch, where base (a multiple of n) is read after the PDL wait (every earlier launch has
// completed, and no CTA of this launch can have passed barrier 1 yet).  No reset is needed.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// The poll spins on relaxed loads and acquires once at the end: ld.acquire compiles to a strong
// load + CCTL.IVALL (an L1 invalidate), which in a spin loop would run once per iteration.
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned long long target) {
  asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
  while (ld_relaxed_u64(bar) < target) {
  }
  (void)ld_acquire_u64(bar);
}

__device__ __forceinline__ int atomic_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define ZDC_STAMP(i)                                                        \
  do {                                                                      \
    if (a.trace) a.trace[static_cast<int64_t>(blockIdx.x) * 32 + (i)] = globaltimer(); \
  } while (0)

// consumer warps per CTA (one more warp is the producer)
static constexpr int kNW = 8;
static constexpr int kNC = kNW * 32;  // consumer threads

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kNC) : "memory"); }

// Ring geometry: sequence number k is consumed by warp w = k % kNW, which owns a sub-ring of
// spw slots, plus one more when w < ex (so the ring can use every slot the shared memory holds).
// Both sides walk the sequence incrementally (no integer division on the issue path: the single
// producer thread issues every slot of the CTA, so its per-slot cost is on the critical path).
struct ProducerCursor {
  int w = 0, u = 0;        // k = u * kNW + w
  int pa = 0, fa = 0;      // position / phase in the sub-rings of spw + 1 slots
  int pb = 0, fb = 0;      // ... of spw slots
  __device__ __forceinline__ int slot(int spw, int ex) const { return w * spw + min(w, ex) + (w < ex ? pa : pb); }
  __device__ __forceinline__ uint32_t phase(int ex) const { return w < ex ? fa : fb; }
  __device__ __forceinline__ bool reuse(int spw, int ex) const { return u >= spw + (w < ex ? 1 : 0); }
  __device__ __forceinline__ void next(int spw) {
    if (++w == kNW) {
      w = 0;
      ++u;
      if (++pa == spw + 1) { pa = 0; fa ^= 1; }
      if (++pb == spw) { pb = 0; fb ^= 1; }
    }
  }
};
struct ConsumerCursor {  // warp w's slots, visited in sequence order
  int base, n, pos = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ ConsumerCursor(int w, int spw, int ex) : base(w * spw + min(w, ex)), n(spw + (w < ex ? 1 : 0)) {}
  __device__ __forceinline__ int slot() const { return base + pos; }
  __device__ __forceinline__ void next() {
    if (++pos == n) { pos = 0; ph ^= 1; }
  }
};

template <int RK>
struct Dims2 {
  // V'/O' dims a lane owns: RK >= 32: [lane*DPL, lane*DPL + DPL); RK == 16: dim lane (lanes < 16)
  static constexpr int DPL = RK >= 32 ? RK / 32 : 1;
};

// o[gi][:] += P[j][gi] V'[j][lane-owned dims] (P broadcast from lane j)
template <int RK, int G>
__device__ __forceinline__ void pv_row(const uint16_t* Vs, int j, int lane, const float (&pb)[G],
                                       float (&o)[G][Dims2<RK>::DPL]) {
  constexpr int DPL = Dims2<RK>::DPL;
  {
    float v[DPL];
    if constexpr (RK >= 32) {
      const uint16_t* vr = Vs + j * RK + lane * DPL;
      if constexpr (DPL == 4) {
        const uint2 u = *reinterpret_cast<const uint2*>(vr);
        v[0] = __uint_as_float(u.x << 16);
        v[1] = __uint_as_float(u.x & 0xFFFF0000u);
        v[2] = __uint_as_float(u.y << 16);
        v[3] = __uint_as_float(u.y & 0xFFFF0000u);
      } else if constexpr (DPL == 2) {
        const uint32_t u = *reinterpret_cast<const uint32_t*>(vr);
        v[0] = __uint_as_float(u << 16);
        v[1] = __uint_as_float(u & 0xFFFF0000u);
      } else {
#pragma unroll
        for (int i = 0; i < DPL; ++i) v[i] = __uint_as_float(static_cast<uint32_t>(vr[i]) << 16);
      }
    } else {
      v[0] = lane < RK ? __uint_as_float(static_cast<uint32_t>(Vs[j * RK + lane]) << 16) : 0.f;
    }
#pragma unroll
    for (int gi = 0; gi < G; ++gi) {
      const float pj = __shfl_sync(0xffffffffu, pb[gi], j);
#pragma unroll
      for (int i = 0; i < DPL; ++i) o[gi][i] = fmaf(pj, v[i], o[gi][i]);
    }
  }
}

// One warp folds up to 32 key rows (lane j = row j) into its running softmax state for the G
// query heads of the KV group: s = q.k * scale * log2(e); m, l, o rescaled online.
template <int RK, int G>
__device__ __forceinline__ void attn_rows(const uint16_t* Ks, const uint16_t* Vs, int np, const float* qf, float scl,
                                          float (&m)[G], float (&l)[G], float (&o)[G][Dims2<RK>::DPL], int lane) {
  constexpr int UK = RK / 8, DPL = Dims2<RK>::DPL;
  float s[G], s2[G];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) s[gi] = s2[gi] = 0.f;
  if (lane < np) {
    const int rot = lane % UK;  // rotated chunk order: the 32 rows of a warp hit distinct banks
#pragma unroll
    for (int kk = 0; kk < UK; ++kk) {
      int kc = kk + rot;
      if (kc >= UK) kc -= UK;
      float kf[8];
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(Ks + lane * RK + kc * 8), kf);
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        const float4 q0 = *reinterpret_cast<const float4*>(qf + gi * RK + kc * 8);
        const float4 q1 = *reinterpret_cast<const float4*>(qf + gi * RK + kc * 8 + 4);
        float x0 = s[gi], x1 = s2[gi];  // two independent FMA chains
        x0 = fmaf(q0.x, kf[0], x0);
        x1 = fmaf(q0.y, kf[1], x1);
        x0 = fmaf(q0.z, kf[2], x0);
        x1 = fmaf(q0.w, kf[3], x1);
        x0 = fmaf(q1.x, kf[4], x0);
        x1 = fmaf(q1.y, kf[5], x1);
        x0 = fmaf(q1.z, kf[6], x0);
        x1 = fmaf(q1.w, kf[7], x1);
        s[gi] = x0;
        s2[gi] = x1;
      }
    }
  }
#pragma unroll
  for (int gi = 0; gi < G; ++gi) s[gi] += s2[gi];
  float pb[G];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    const float sv = lane < np ? s[gi] * scl : -INFINITY;
    float mx = sv;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float mn = fmaxf(m[gi], mx);  // finite: np >= 1
    const float alpha = exp2f(m[gi] - mn);
    const float p = lane < np ? exp2f(sv - mn) : 0.f;
    float ps = p;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
    l[gi] = l[gi] * alpha + ps;
    m[gi] = mn;
    pb[gi] = __bfloat162float(__float2bfloat16_rn(p));
#pragma unroll
    for (int i = 0; i < DPL; ++i) o[gi][i] *= alpha;
  }
  // o += P V' (lane-owned dims); full slots take the unrolled path
  if (np == 32) {
#pragma unroll 8
    for (int j = 0; j < 32; ++j) pv_row<RK, G>(Vs, j, lane, pb, o);
    return;
  }
  for (int j = 0; j < np; ++j) pv_row<RK, G>(Vs, j, lane, pb, o);
}

// GEMV of R consecutive rows of one ring slot against NB input rows (x converted once per
// chunk and shared by the R rows): acc[r][b] = W[r0 + r] . xs[b]
template <int NB, int R>
__device__ __forceinline__ void gemv_rows(const uint8_t* slot, int K, const uint4* xs4, int xw8, int lane,
                                          float (&acc)[R][NB], int r0) {
  const int kc = K >> 3;
  const uint4* w = reinterpret_cast<const uint4*>(slot) + static_cast<size_t>(r0) * kc;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[r][b] = 0.f;
#pragma unroll 2
  for (int c = lane; c < kc; c += 32) {
    uint4 wv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) wv[r] = w[r * kc + c];
    float xf[NB][8];
#pragma unroll
    for (int b = 0; b < NB; ++b) bf16x8_to_f32(xs4[b * xw8 + c], xf[b]);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float wf[8];
      bf16x8_to_f32(wv[r], wf);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float x0 = 0.f, x1 = 0.f;  // two short chains per chunk
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          x0 = fmaf(wf[e], xf[b][e], x0);
          x1 = fmaf(wf[e + 1], xf[b][e + 1], x1);
        }
        acc[r][b] += x0 + x1;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[r][b] += __shfl_xor_sync(0xffffffffu, acc[r][b], off);
    }
}

template <int NB, int RK, int G>
__global__ void __launch_bounds__(kNC + 32, 1) decode_fused_kernel(const DecFusedArgs a) {
  constexpr int DPL = Dims2<RK>::DPL;
  extern __shared__ __align__(128) uint8_t smem[];
  const int SB = a.slot_bytes, spw = a.spw, ex = a.ring_extra, nslot = kNW * spw + ex;
  const int xw = a.xw, xw8 = xw >> 3;
  uint8_t* ring = smem;
  uint16_t* xs = reinterpret_cast<uint16_t*>(smem + static_cast<size_t>(nslot) * SB);  // [NB][xw]
  float* qf = reinterpret_cast<float*>(xs + NB * xw);                                  // [G][RK]
  float* wst = qf + G * RK;                                                            // [kNW][G][RK+2]
  uint16_t* nrow = reinterpret_cast<uint16_t*>(wst + kNW * G * (RK + 2));             // [2][RK]
  float* pst = reinterpret_cast<float*>(nrow + 2 * RK);  // staged partials [B*Nh][splits][RK+2] (stage_part)
  uint64_t* full = reinterpret_cast<uint64_t*>(pst + a.pst_floats);
  uint64_t* empty = full + nslot;
  uint64_t* lenbar = empty + nslot;
  uint64_t* pbar = lenbar + 1;
  unsigned long long* s_base = reinterpret_cast<unsigned long long*>(pbar + 1);
  int* s_flag = reinterpret_cast<int*>(s_base + 1);
  int* s_lens = s_flag + 1;  // [nl] cache lengths at entry

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int cta = blockIdx.x, ncta = gridDim.x;
  if (tid == kNC) {
    for (int s = 0; s < nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(lenbar, 1);
    mbar_init(pbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) ZDC_STAMP(0);

  // ---- static work split, identical for every layer of the run (and in producer and consumers)
  const int d = a.d, ko = a.ko_p;
  const int per1 = (a.n_qkv + ncta - 1) / ncta;
  const int r1a = min(a.n_qkv, cta * per1), r1b = min(a.n_qkv, r1a + per1);
  const int rps1 = SB / (d * 2);
  const int n1 = (r1b - r1a + rps1 - 1) / rps1;
  const int per3 = (d + ncta - 1) / ncta;
  const int r3a = min(d, cta * per3), r3b = min(d, r3a + per3);
  const int rps3 = SB / (ko * 2);
  const int n3 = (r3b - r3a + rps3 - 1) / rps3;
  const int nitems = a.B * a.Nkv * a.splits;
  const int RPS = a.rps;  // K'/V' rows per slot (a multiple of 32): [RPS][RK] K' then [RPS][RK] V'
  const int tl = a.nl > 1 ? 1 : 0;  // layer whose timeline the trace records

  if (warp == kNW) {
    pdl_trigger();  // every thread of the CTA triggers: the dependent launch may become resident now
    // ================= producer (one thread): every HBM byte of this CTA, in consumption order,
    // layer after layer: while the consumers finish layer l, the ring fills with layer l+1's W_QKV
    if (lane == 0) {
      ProducerCursor pc;
      bool have_lens = false;
      for (int li = 0; li < a.nl; ++li) {
        const DecLayer Ly = a.layers[li];
        for (int r = r1a; r < r1b; r += rps1) {  // phase 1 weights (static: no dependency wait)
          const int nr = min(rps1, r1b - r);
          const int s = pc.slot(spw, ex);
          if (pc.reuse(spw, ex)) mbar_wait(&empty[s], pc.phase(ex) ^ 1);
          pc.next(spw);
          const uint32_t bytes = static_cast<uint32_t>(nr) * d * 2u;
          mbar_arrive_expect_tx(&full[s], bytes);
          bulk_g2s(ring + static_cast<size_t>(s) * SB, Ly.wqkv + static_cast<int64_t>(r) * d, bytes, &full[s]);
        }
        if (li == tl) ZDC_STAMP(8);
        if (!have_lens) {  // lengths are read by a consumer after the PDL wait
          mbar_wait(lenbar, 0);
          have_lens = true;
        }
        const int L = s_lens[li], L1 = L + 1;
        const int chunk = (L1 + a.splits - 1) / a.splits;
        for (int it = cta; it < nitems; it += ncta) {
          const int sp = it % a.splits, g = (it / a.splits) % a.Nkv, b = it / (a.splits * a.Nkv);
          const int s0 = sp * chunk, e0 = min(min(L1, s0 + chunk), L);  // cached rows only
          const int64_t row0 = (static_cast<int64_t>(b) * a.Nkv + g) * a.S_cap;
          for (int p = s0; p < e0; p += RPS) {
            const int np = min(RPS, e0 - p);
            const int s = pc.slot(spw, ex);
            if (pc.reuse(spw, ex)) mbar_wait(&empty[s], pc.phase(ex) ^ 1);
            pc.next(spw);
            const uint32_t bytes = static_cast<uint32_t>(np) * RK * 2u;
            mbar_arrive_expect_tx(&full[s], 2 * bytes);
            uint8_t* dst = ring + static_cast<size_t>(s) * SB;
            bulk_g2s(dst, Ly.kc + (row0 + p) * RK, bytes, &full[s]);
            bulk_g2s(dst + RPS * RK * 2, Ly.vc + (row0 + p) * RK, bytes, &full[s]);
          }
        }
        if (li == tl) ZDC_STAMP(9);
        for (int r = r3a; r < r3b; r += rps3) {  // phase 3 weights
          const int nr = min(rps3, r3b - r);
          const int s = pc.slot(spw, ex);
          if (pc.reuse(spw, ex)) mbar_wait(&empty[s], pc.phase(ex) ^ 1);
          pc.next(spw);
          const uint32_t bytes = static_cast<uint32_t>(nr) * ko * 2u;
          mbar_arrive_expect_tx(&full[s], bytes);
          bulk_g2s(ring + static_cast<size_t>(s) * SB, Ly.wo + static_cast<int64_t>(r) * ko, bytes, &full[s]);
        }
        if (li == tl) ZDC_STAMP(10);
      }
    }
    return;
  }

  // ================= consumers (warps 0..kNW-1)
  pdl_wait();
  pdl_trigger();
  if (tid == 0) {
    for (int li = 0; li < a.nl; ++li) {
      const int L0 = *a.layers[li].len_ptr;
      // a full cache (graph replays past max_seq) rewrites its last row instead of writing past it
      s_lens[li] = min(L0, a.S_cap - 1);
      if (L0 >= a.S_cap && cta == 0 && a.err) *a.err = 1;
    }
    *s_base = ld_acquire_u64(a.gbar) / ncta * ncta;
    mbar_arrive(lenbar);
  }
  ConsumerCursor cc(warp, spw, ex);
  const uint4* xs4 = reinterpret_cast<const uint4*>(xs);
  const float scl = a.scale * kLog2eF;
  unsigned long long nbar = 0;  // grid barriers passed in this launch
  int kb = 0;                   // ring sequence number of the current phase's first slot

  for (int li = 0; li < a.nl; ++li) {
    const DecLayer Ly = a.layers[li];
    if (tid == 0 && li == tl) ZDC_STAMP(13);
    // ---- stage this layer's input: x for the first layer, the previous layer's y after
    {
      const uint16_t* xin = li == 0 ? a.x : a.y;
      const int64_t ld = li == 0 ? a.ldx : a.ldy;
      const int kcx = d >> 3;
      uint4* xw4 = reinterpret_cast<uint4*>(xs);
      for (int i = tid; i < NB * kcx; i += kNC) {
        const int b = i / kcx, c = i - b * kcx;
        xw4[b * xw8 + c] = b < a.B ? __ldcg(reinterpret_cast<const uint4*>(xin + b * ld) + c) : make_uint4(0, 0, 0, 0);
      }
    }
    consumer_sync();
    if (tid == 0 && li == tl) ZDC_STAMP(1);
    const int L = s_lens[li], L1 = L + 1;

    // ---- phase 1: a1 + a2
    for (int t = (warp - kb % kNW + kNW) % kNW; t < n1; t += kNW) {
      const int s = cc.slot();
      mbar_wait(&full[s], cc.ph);
      cc.next();
      const int rb = r1a + t * rps1, nr = min(rps1, r1b - rb);
      for (int r = 0; r < nr; ++r) {
        float acc[1][NB];
        gemv_rows<NB, 1>(ring + static_cast<size_t>(s) * SB, d, xs4, xw8, lane, acc, r);
        const int n = rb + r;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (lane == b && b < a.B) {
            const uint16_t v = f32_to_bf16_bits(acc[0][b]);
            if (n < a.nq) {
              a.q[b * a.ldq + n] = v;
            } else if (n < a.nq + a.nk) {
              const int nn = n - a.nq, g = nn / RK, c = nn - g * RK;
              Ly.kc[((static_cast<int64_t>(b) * a.Nkv + g) * a.S_cap + L) * RK + c] = v;
            } else {
              const int nn = n - a.nq - a.nk, g = nn / RK, c = nn - g * RK;
              Ly.vc[((static_cast<int64_t>(b) * a.Nkv + g) * a.S_cap + L) * RK + c] = v;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    kb += n1;
    consumer_sync();
    if (tid == 0) {
      if (li == tl) ZDC_STAMP(2);
      grid_barrier(a.gbar, *s_base + (++nbar) * ncta);
      if (li == tl) ZDC_STAMP(3);
    }
    if (tid != 0) ++nbar;
    consumer_sync();

    // ---- phase 2: a3 partials
    const int chunk = (L1 + a.splits - 1) / a.splits;
    for (int it = cta; it < nitems; it += ncta) {
      const int sp = it % a.splits, g = (it / a.splits) % a.Nkv, b = it / (a.splits * a.Nkv);
      const int s0 = sp * chunk, s1 = min(L1, s0 + chunk), e0 = min(s1, L);
      const int ns = e0 > s0 ? (e0 - s0 + RPS - 1) / RPS : 0;
      const bool has_new = s0 <= L && L < s1;
      for (int i = tid; i < G * RK; i += kNC) {
        const int gi = i / RK, c = i - gi * RK;
        const uint16_t u = __ldcg(reinterpret_cast<const unsigned short*>(a.q) + b * a.ldq + (g * G + gi) * RK + c);
        qf[i] = __uint_as_float(static_cast<uint32_t>(u) << 16);
      }
      if (has_new && warp == 0) {
        const int64_t row = ((static_cast<int64_t>(b) * a.Nkv + g) * a.S_cap + L) * RK;
        for (int c = lane; c < RK; c += 32) {
          nrow[c] = __ldcg(reinterpret_cast<const unsigned short*>(Ly.kc) + row + c);
          nrow[RK + c] = __ldcg(reinterpret_cast<const unsigned short*>(Ly.vc) + row + c);
        }
      }
      consumer_sync();
      float m[G], l[G], o[G][DPL];
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        m[gi] = -INFINITY;
        l[gi] = 0.f;
#pragma unroll
        for (int i = 0; i < DPL; ++i) o[gi][i] = 0.f;
      }
      for (int t = (warp - kb % kNW + kNW) % kNW; t < ns; t += kNW) {
        const int s = cc.slot();
        mbar_wait(&full[s], cc.ph);
        if (tid == 0 && li == tl && it == cta && t < kNW) ZDC_STAMP(14);
        cc.next();
        const uint16_t* Ks = reinterpret_cast<const uint16_t*>(ring + static_cast<size_t>(s) * SB);
        const int nr = min(RPS, e0 - (s0 + t * RPS));
        for (int j = 0; j < nr; j += 32)
          attn_rows<RK, G>(Ks + j * RK, Ks + (RPS + j) * RK, min(32, nr - j), qf, scl, m, l, o, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      if (has_new && warp == 0) attn_rows<RK, G>(nrow, nrow + RK, 1, qf, scl, m, l, o, lane);
      // warp states -> shared memory, then the CTA merges them into this item's partial
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
      if (tid == 0 && li == tl) ZDC_STAMP(11);
      for (int i = tid; i < G * RK; i += kNC) {
        const int gi = i / RK, c = i - gi * RK;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kNW; ++w) M = fmaxf(M, wst[(w * G + gi) * (RK + 2) + RK]);
        float O = 0.f, Ls = 0.f;
        if (M != -INFINITY) {
#pragma unroll
          for (int w = 0; w < kNW; ++w) {
            const float* e = wst + (w * G + gi) * (RK + 2);
            const float f = exp2f(e[RK] - M);  // 0 for warps without rows (m = -inf)
            O = fmaf(e[c], f, O);
            Ls = fmaf(e[RK + 1], f, Ls);
          }
        }
        float* dst = a.part + ((static_cast<int64_t>(b) * a.Nh + g * G + gi) * a.splits + sp) * (RK + 2);
        dst[c] = O;
        if (c == 0) {
          dst[RK] = M;
          dst[RK + 1] = Ls;
        }
      }
      // without staging (large partial sets) the last CTA to finish a chunk of (b, g) merges them:
      // O' = sum_s o_s 2^(m_s - M) / sum_s l_s 2^(m_s - M), LSE = (M + log2 L) ln 2
      consumer_sync();
      if (!a.stage_part && tid == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        *s_flag = atomic_add_acq_rel(a.counters + b * a.Nkv + g, 1) == a.splits - 1;
      }
      consumer_sync();
      if (!a.stage_part && *s_flag) {
        for (int i = tid; i < G * RK; i += kNC) {
          const int gi = i / RK, c = i - gi * RK;
          const float* hp = a.part + (static_cast<int64_t>(b) * a.Nh + g * G + gi) * a.splits * (RK + 2);
          float M = -INFINITY;
          for (int s2 = 0; s2 < a.splits; ++s2) M = fmaxf(M, __ldcg(hp + s2 * (RK + 2) + RK));
          float O = 0.f, Ls = 0.f;
          for (int s2 = 0; s2 < a.splits; ++s2) {
            const float ms = __ldcg(hp + s2 * (RK + 2) + RK);
            const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
            O = fmaf(f, __ldcg(hp + s2 * (RK + 2) + c), O);
            Ls = fmaf(f, __ldcg(hp + s2 * (RK + 2) + RK + 1), Ls);
          }
          a.o[b * ko + (g * G + gi) * RK + c] = f32_to_bf16_bits(O / Ls);
          if (c == 0 && a.lse) a.lse[b * a.Nh + g * G + gi] = (M + log2f(Ls)) / kLog2eF;
        }
        if (tid == 0) a.counters[b * a.Nkv + g] = 0;
      }
      consumer_sync();
      kb += ns;
    }
    consumer_sync();
    if (tid == 0) {
      if (li == tl) ZDC_STAMP(4);
      grid_barrier(a.gbar, *s_base + (++nbar) * ncta);
      if (li == tl) ZDC_STAMP(5);
    }
    if (tid != 0) ++nbar;
    consumer_sync();
    if (cta == 0 && tid == 0) *Ly.len_ptr = L1;  // every reader of this length has passed barrier 1

    if (a.stage_part) {
      // ---- every CTA merges all heads from ONE bulk copy of the partials (one round trip
      // instead of the atomic + merge + reload chain): the same LSE merge as above
      if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> async-proxy reads
        mbar_arrive_expect_tx(pbar, static_cast<uint32_t>(a.pst_bytes));
        bulk_g2s(pst, a.part, static_cast<uint32_t>(a.pst_bytes), pbar);
      }
      mbar_wait(pbar, static_cast<uint32_t>(li & 1));
      if (tid == 0 && li == tl) ZDC_STAMP(12);
      const int S2 = a.splits;
      // O' chunks of 8 columns (one head never straddles a chunk: RK % 16 == 0); each thread
      // merges its head's splits in one pass: M = max m_s, L = sum 2^(m_s-M) l_s, O' = sum 2^(m_s-M) o_s / L
      const int ko8 = ko >> 3, hk8 = (a.Nh * RK) >> 3;
      uint4* xo = reinterpret_cast<uint4*>(xs);
      for (int i = tid; i < NB * ko8; i += kNC) {
        const int b = i / ko8, c8 = i - b * ko8;
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = 0.f;
        if (b < a.B && c8 < hk8) {
          const int h = (c8 * 8) / RK, cc8 = c8 * 8 - h * RK;
          const int bh = b * a.Nh + h;
          const float* hp = pst + bh * S2 * (RK + 2);
          float M = -INFINITY;
          for (int s2 = 0; s2 < S2; ++s2) M = fmaxf(M, hp[s2 * (RK + 2) + RK]);
          float Ls = 0.f;
          for (int s2 = 0; s2 < S2; ++s2) {
            const float* e2 = hp + s2 * (RK + 2);
            const float ms = e2[RK];
            const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
            Ls = fmaf(f, e2[RK + 1], Ls);
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const float2 o2 = *reinterpret_cast<const float2*>(e2 + cc8 + e);  // 8-byte aligned
              v[e] = fmaf(f, o2.x, v[e]);
              v[e + 1] = fmaf(f, o2.y, v[e + 1]);
            }
          }
          const float inv = 1.f / Ls;
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] *= inv;
          if (cc8 == 0 && cta == 0 && a.lse) a.lse[bh] = (M + log2f(Ls)) / kLog2eF;
        }
        xo[b * xw8 + c8] = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                                      pack_bf16x2(v[6], v[7]));
      }
    } else {
      // ---- O' (merged by the last CTA of each (b, g), published by barrier 2) -> shared memory
      const int ko8 = ko >> 3, hk8 = (a.Nh * RK) >> 3;
      uint4* xo = reinterpret_cast<uint4*>(xs);
      for (int i = tid; i < NB * ko8; i += kNC) {
        const int b = i / ko8, c = i - b * ko8;
        xo[b * xw8 + c] = b < a.B && c < hk8 ? __ldcg(reinterpret_cast<const uint4*>(a.o + b * ko) + c)
                                             : make_uint4(0, 0, 0, 0);
      }
    }
    consumer_sync();
    if (tid == 0 && li == tl) ZDC_STAMP(6);

    // ---- phase 3: a5
    for (int t = (warp - kb % kNW + kNW) % kNW; t < n3; t += kNW) {
      const int s = cc.slot();
      mbar_wait(&full[s], cc.ph);
      if (tid == 0 && li == tl && t < kNW) ZDC_STAMP(15);
      cc.next();
      const int rb = r3a + t * rps3, nr = min(rps3, r3b - rb);
      int r = 0;
      for (; r + 2 <= nr; r += 2) {  // row pairs: two independent dot products per lane
        float acc[2][NB];
        gemv_rows<NB, 2>(ring + static_cast<size_t>(s) * SB, ko, xs4, xw8, lane, acc, r);
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (lane == b && b < a.B) {
            a.y[b * a.ldy + rb + r] = f32_to_bf16_bits(acc[0][b]);
            a.y[b * a.ldy + rb + r + 1] = f32_to_bf16_bits(acc[1][b]);
          }
      }
      if (r < nr) {
        float acc[1][NB];
        gemv_rows<NB, 1>(ring + static_cast<size_t>(s) * SB, ko, xs4, xw8, lane, acc, r);
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (lane == b && b < a.B) a.y[b * a.ldy + rb + r] = f32_to_bf16_bits(acc[0][b]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    kb += n3;
    if (li + 1 < a.nl) {
      // y of this layer is the next layer's input
      consumer_sync();
      if (tid == 0) grid_barrier(a.gbar, *s_base + (++nbar) * ncta);
      if (tid != 0) ++nbar;
      consumer_sync();
    }
  }
  if (a.trace) {
    consumer_sync();
    if (tid == 0) ZDC_STAMP(7);
  }
}

// ------------------------------------------------------------------ host
// ring cap (ZDC_FUSED_RING_KB); the launcher fits as many slots as the 227 KB of shared memory allow
static const int kFusedRingBytes = knob("ZDC_FUSED_RING_KB", 224) * 1024;

template <int NB, int RK, int G>
inline cudaError_t launch_fused_t(DecFusedArgs a, cudaStream_t stream) {
  // slot: a multiple of the a1 row, of 32 K'+V' rows and of the a5 row; larger slots (fewer, bigger
  // bulk copies in flight) stream faster from HBM (tools/stream_probe.cu)
  int slot = std::max(std::max(a.d * 2, 4 * 32 * RK), a.ko_p * 2);
  static const int slot_kb = knob("ZDC_FUSED_SLOT_KB", 0);
  if (slot_kb * 1024 > slot) {
    const int unit = std::max(std::max(a.d * 2, a.ko_p * 2), 4 * 32 * RK);
    slot = std::max(slot, slot_kb * 1024 / unit * unit);
  }
  a.rps = slot / (4 * RK) / 32 * 32;
  a.slot_bytes = slot;
  a.xw = std::max(a.d, a.ko_p);
  constexpr size_t kSmemMax = 227 * 1024;
  const size_t fixed = static_cast<size_t>(NB) * a.xw * 2 + G * RK * 4 + kNW * G * (RK + 2) * 4 + 2 * RK * 2 + 48 +
                       static_cast<size_t>(a.nl) * 4;
  // the partials of every head staged by one bulk copy after barrier 2 when they fit (<= 48 KB)
  const int64_t pbytes = (static_cast<int64_t>(a.B) * a.Nh * a.splits * (RK + 2) * 4 + 15) / 16 * 16;
  const size_t per_slot = static_cast<size_t>(slot) + 16;  // slot + its two mbarriers
  a.stage_part = pbytes <= 48 * 1024 && fixed + pbytes + kNW * per_slot <= kSmemMax ? 1 : 0;
  a.pst_floats = a.stage_part ? pbytes / 4 : 0;
  a.pst_bytes = a.stage_part ? pbytes : 0;
  const size_t base = fixed + static_cast<size_t>(a.pst_floats) * 4;
  const int nslot = static_cast<int>(std::min<size_t>(kFusedRingBytes / slot, (kSmemMax - std::min(base, kSmemMax)) / per_slot));
  if (nslot < kNW) return cudaErrorNotSupported;
  a.spw = nslot / kNW;
  a.ring_extra = nslot % kNW;
  const size_t smem = base + static_cast<size_t>(nslot) * per_slot;
  if (smem > kSmemMax) return cudaErrorNotSupported;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_fused_kernel<NB, RK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // the grid barriers need every CTA resident at once: one per SM (num_sms() CTAs).  Checked once
  // per shared-memory size with the occupancy API; otherwise the caller runs the separate kernels.
  static size_t checked_smem = 0;
  if (checked_smem != smem) {
    int per_sm = 0;
    cudaError_t eo = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_fused_kernel<NB, RK, G>, kNC + 32, smem);
    if (eo != cudaSuccess) return eo;
    if (per_sm < 1) return cudaErrorNotSupported;
    checked_smem = smem;
  }
  prof_mark(stream, true, g_prof_class);
  cudaError_t e = launch_k(decode_fused_kernel<NB, RK, G>, dim3(num_sms()), dim3(kNC + 32), smem, stream, g_pdl, a);
  prof_mark(stream, false, g_prof_class);
  ++g_launches;
  return e;
}

template <int NB, int RK>
inline cudaError_t launch_fused_g(const DecFusedArgs& a, int G, cudaStream_t s) {
  switch (G) {
    case 1: return launch_fused_t<NB, RK, 1>(a, s);
    case 2: return launch_fused_t<NB, RK, 2>(a, s);
    case 4: return launch_fused_t<NB, RK, 4>(a, s);
    case 8: return launch_fused_t<NB, RK, 8>(a, s);
    default: return cudaErrorNotSupported;
  }
}

template <int NB>
inline cudaError_t launch_fused_r(const DecFusedArgs& a, int RK, int G, cudaStream_t s) {
  switch (RK) {
    case 16: return launch_fused_g<NB, 16>(a, G, s);
    case 32: return launch_fused_g<NB, 32>(a, G, s);
    case 64: return launch_fused_g<NB, 64>(a, G, s);
    case 96: return launch_fused_g<NB, 96>(a, G, s);
    case 128: return launch_fused_g<NB, 128>(a, G, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace zdc
