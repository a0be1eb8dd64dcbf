// gemm.cu — the a1 / a5 projection engine: D[M][N] = A[M][K] * B[N][K]^T.
//
// a1 (Eq. 1, with the folded, pre-truncated W^R of P:1206 / P:1218): A = x [B*S][d],
//    B = packed W_QKV^R transposed [N_h r_k + N_kv (r_k + r_v)][d]; the epilogue scatters Q' to
//    a staging matrix and K'/V' straight into the compressed KV cache (a2 fused).
// a5 (Eq. 4, folded W_O of P:1219-1221): A = O' [B*S][N_h r_v], B = W_O^R transposed.
//
// sm_100a design: persistent CTAs (one per SM), warp-specialised:
//   warp 0   TMA producer   (cp.async.bulk.tensor, 128B swizzle, STAGES-deep mbarrier ring)
//   warp 1   MMA issuer     (one elected thread, tcgen05.mma kind::f16 M=128 N=BN K=16)
//   warp 2   TMEM allocator (2 x BN f32 columns: double-buffered accumulators)
//   warps 4-7 epilogue     (tcgen05.ld 32x32b -> bf16 RNE -> global), overlapping the next
//                           tile's mainloop through the accumulator double buffer.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

namespace zdc {

int64_t g_launches = 0;
bool g_pdl = knob("ZDC_NO_PDL", 0) == 0;  // A/B switch for programmatic dependent launch
// which decode kernels launch with PDL: bit 0 projections (GEMV), bit 1 attention
int g_pdl_mask = knob("ZDC_PDL_MASK", 3);
int g_prof_class = kProfOther;

// ------------------------------------------------------------------ host: per-class event timing
struct ProfState {
  bool on = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  cudaEvent_t pending = nullptr;
  std::vector<cudaEvent_t> pool;
};
static ProfState g_prof;

bool prof_enabled() { return g_prof.on; }

static cudaEvent_t prof_event() {
  if (!g_prof.pool.empty()) {
    cudaEvent_t e = g_prof.pool.back();
    g_prof.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_mark(cudaStream_t s, bool begin, int cls) {
  if (!g_prof.on) return;
  cudaEvent_t e = prof_event();
  cudaEventRecord(e, s);
  if (begin) {
    g_prof.pending = e;
  } else {
    g_prof.marks.push_back({cls, {g_prof.pending, e}});
    g_prof.pending = nullptr;
  }
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }
cudaError_t launch_set_int(int* p, int v, cudaStream_t s) {
  set_int_kernel<<<1, 1, 0, s>>>(p, v);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ host: tensor maps
typedef CUresult (*PFN_tmapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                        CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                        CUtensorMapFloatOOBfill);

static PFN_tmapEncodeTiled get_encode_fn() {
  static PFN_tmapEncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_tmapEncodeTiled>(p);
  });
  return fn;
}

bool make_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner_elems, uint64_t outer_rows,
                  uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  PFN_tmapEncodeTiled fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner_elems, outer_rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = kNumSMsB200;
  }
  return n;
}

// ------------------------------------------------------------------ device: epilogue store
// Store 8 consecutive output columns [n, n+8) of row m (already packed to bf16x2 x 4).
__device__ __forceinline__ void store_unit(const Epilogue& e, int m, int n, uint4 val) {
  uint16_t* dst;
  if (e.mode == 0) {
    dst = e.d + static_cast<int64_t>(m) * e.ldd + n;
  } else if (e.mode == 2) {
    const UlyssesDest& u = e.uly;
    int q, c;
    if (n < u.nq) {
      q = n / u.hq;
      c = n - q * u.hq;
    } else if (n < u.nq + u.nk) {
      const int nn = n - u.nq;
      q = nn / u.kq;
      c = u.hq + nn - q * u.kq;
    } else {
      const int nn = n - u.nq - u.nk;
      q = nn / u.vq;
      c = u.hq + u.kq + nn - q * u.vq;
    }
    dst = u.send + (static_cast<int64_t>(q) * u.rows + m) * u.cols + c;
  } else {
    const QkvDest& q = e.qkv;
    if (n < q.nq) {
      dst = q.q + static_cast<int64_t>(m) * q.ldq + n;
    } else {
      const int b = m / q.S, t = m - (m / q.S) * q.S;
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
  *reinterpret_cast<uint4*>(dst) = val;
}

// ------------------------------------------------------------------ device: the GEMM
// AR < 128 (skinny decode GEMMs, M <= AR): a stage loads only AR rows of A (the activations), so
// the ring holds more stages of weight (B) tiles -- the bytes in flight per SM set the HBM stream
// rate of these HBM-bound GEMMs.  The MMA still runs M = 128: rows >= AR of its A operand read the
// next stage's bytes (in-bounds shared memory) and only produce accumulator rows >= M, which the
// epilogue never stores.
template <int BN, int AR = 128>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr uint32_t A_TILE = AR * BK * 2, B_TILE = BN * BK * 2;
  static constexpr uint32_t A_BYTES = A_TILE, B_BYTES = B_TILE, STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = AR == 128 ? (BN == 256 ? 4 : 6) : static_cast<int>((200u * 1024u) / STAGE_BYTES);
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  // (the last A stage's 128-row view reaches into the B stages that follow it: still in bounds)
  static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

// Output tile -> (M-block, N-block).  band == 0: M fastest.  band > 0: grouped raster -- bands of
// `band` N-blocks, each swept over every M-block with the band's N fastest, so concurrent CTAs share
// A rows (read once per band) while the band's weight tiles stay L2-resident.
__device__ __forceinline__ void tile_coords(int tile, int m_tiles, int n_tiles, int band, int& mb, int& nb) {
  if (band <= 0) {
    mb = tile % m_tiles;
    nb = tile / m_tiles;
    return;
  }
  const int per_band = m_tiles * band;
  const int bi = tile / per_band, n0 = bi * band;
  const int w = min(band, n_tiles - n0);  // the last band may be narrower
  const int idx = tile - bi * per_band;
  mb = idx / w;
  nb = n0 + idx % w;
}

template <int BN, int AR>
__global__ void __launch_bounds__(256, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, int M,
                        int N, int K, const Epilogue epi) {
  using C = GemmCfg<BN, AR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);

  const int m_tiles = (M + C::BM - 1) / C::BM;
  const int n_tiles = (N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int k_blocks = K / C::BK;
  // work item w: output tile w % num_tiles, k-split w / num_tiles (k-blocks [kb0, kb1))
  const int ks = epi.k_splits;
  const int num_work = num_tiles * ks;
  const int kpb = (k_blocks + ks - 1) / ks;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma_a);
    tma_prefetch_desc(&tma_b);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Launched with programmatic dependent launch (decode): everything that reads the predecessor's
  // output waits for it; the producer first requests the weight (B) tiles of the ring's first
  // stages, which do not depend on it (griddepcontrol.wait is a no-op without PDL).
  if (warp != 0) pdl_wait();
  if (epi.len_inc && blockIdx.x == 0 && threadIdx.x == 4 * 32) advance_len(epi);
  if (warp == 0) {
    // ---------------- TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int issued = 0;
      bool waited = false;
      const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
      for (int w = blockIdx.x; w < num_work; w += gridDim.x) {
        const int tile = w % num_tiles, sp = w / num_tiles;
        int mb, nb;
        tile_coords(tile, m_tiles, n_tiles, epi.raster_n, mb, nb);
        const int kb1 = min(k_blocks, (sp + 1) * kpb);
        if (!waited && w == static_cast<int>(blockIdx.x)) {
          // prologue: B of the first stages, then the dependency wait, then their A
          const int n0 = max(0, min(C::STAGES, kb1 - sp * kpb));
          for (int i = 0; i < n0; ++i) {
            mbar_arrive_expect_tx(&full[i], C::STAGE_BYTES);
            tma_load_2d(sB + i * C::B_BYTES, &tma_b, &full[i], (sp * kpb + i) * C::BK, nb * BN);
          }
          pdl_wait();
          pdl_trigger();
          for (int i = 0; i < n0; ++i)
            tma_load_2d(sA + i * C::A_BYTES, &tma_a, &full[i], (sp * kpb + i) * C::BK, mb * C::BM);
          issued = n0;
          waited = true;
          stage = n0 % C::STAGES;
          phase = n0 == C::STAGES ? 1u : 0u;
        }
        for (int kb = sp * kpb + issued; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          if (epi.raster_n) {  // A streams through L2 once; B (the weights) stays resident
            tma_load_2d_hint(sA + stage * C::A_BYTES, &tma_a, &full[stage], kb * C::BK, mb * C::BM, pol_first);
            tma_load_2d_hint(sB + stage * C::B_BYTES, &tma_b, &full[stage], kb * C::BK, nb * BN, pol_last);
          } else {
            tma_load_2d(sA + stage * C::A_BYTES, &tma_a, &full[stage], kb * C::BK, mb * C::BM);
            tma_load_2d(sB + stage * C::B_BYTES, &tma_b, &full[stage], kb * C::BK, nb * BN);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        issued = 0;
      }
      if (!waited) pdl_wait();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc_bf16(C::BM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int w = blockIdx.x; w < num_work; w += gridDim.x) {
        const int sp = w / num_tiles, kb0 = sp * kpb, kb1 = min(k_blocks, kb0 + kpb);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < C::BK / 16; ++kk) {
            const uint64_t ad = make_sdesc(a_addr + kk * 32, 16, 1024, kSw128);
            const uint64_t bd = make_sdesc(b_addr + kk * 32, 16, 1024, kSw128);
            umma_bf16_ss(d_tmem, ad, bd, idesc, (kb != kb0 || kk != 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);  // frees the smem slot once these MMAs have read it
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> bf16 -> global
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int w = blockIdx.x; w < num_work; w += gridDim.x) {
      const int tile = w % num_tiles;
      int mb, nb;
      tile_coords(tile, m_tiles, n_tiles, epi.raster_n, mb, nb);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = mb * C::BM + q * 32 + lane;
      if (ks > 1) {
        // split-K: this split's partial tile into the f32 workspace (vector reductions at L2)
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tmem_ld32(tmem_base + ((q * 32) << 16) + acc * BN + c, r);
          tc_wait_ld();
          const int n0 = nb * BN + c;
          if (row < M && n0 < N) {
            float* wrow = epi.ws + static_cast<int64_t>(row) * N;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int n = n0 + u * 4;
              if (n + 4 <= N)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(wrow + n), "f"(__uint_as_float(r[u * 4])),
                             "f"(__uint_as_float(r[u * 4 + 1])), "f"(__uint_as_float(r[u * 4 + 2])),
                             "f"(__uint_as_float(r[u * 4 + 3]))
                             : "memory");
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        __threadfence();
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (warp == 4 && lane == 0) *s_last = atomicAdd(epi.ws_cnt + tile, 1) == ks - 1;
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (*s_last) {  // the last split: summed tile -> bf16 -> the epilogue's destination; reset
          __threadfence();
          // 8-column units of the tile's valid rows, spread over the 128 epilogue threads with four
          // independent L2 round trips in flight per thread (a row per thread serialises ~BN/8 of them)
          const int et = (warp - 4) * 32 + lane;
          const int r0 = mb * C::BM, rows = min(C::BM, M - r0);
          const int c0 = nb * BN, cols = min(BN, N - c0) / 8;
          const int units = rows * cols;
          for (int u0 = 0; u0 < units; u0 += 4 * 128) {
            float4 v[4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int u = u0 + i * 128 + et;
              if (u < units) {
                const float* src = epi.ws + static_cast<int64_t>(r0 + u / cols) * N + c0 + (u % cols) * 8;
                v[i][0] = __ldcg(reinterpret_cast<const float4*>(src));
                v[i][1] = __ldcg(reinterpret_cast<const float4*>(src + 4));
              }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int u = u0 + i * 128 + et;
              if (u < units) {
                const int rr = r0 + u / cols, n = c0 + (u % cols) * 8;
                uint4 val;
                val.x = pack_bf16x2(v[i][0].x, v[i][0].y);
                val.y = pack_bf16x2(v[i][0].z, v[i][0].w);
                val.z = pack_bf16x2(v[i][1].x, v[i][1].y);
                val.w = pack_bf16x2(v[i][1].z, v[i][1].w);
                store_unit(epi, rr, n, val);
                float* dst = epi.ws + static_cast<int64_t>(rr) * N + n;
                __stcg(reinterpret_cast<float4*>(dst), make_float4(0.f, 0.f, 0.f, 0.f));
                __stcg(reinterpret_cast<float4*>(dst + 4), make_float4(0.f, 0.f, 0.f, 0.f));
              }
            }
          }
          if (warp == 4 && lane == 0) epi.ws_cnt[tile] = 0;
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");  // s_last is rewritten by the next item
        continue;
      }
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((q * 32) << 16) + acc * BN + c, r);
        tc_wait_ld();
        const int n0 = nb * BN + c;
        if (row < M && n0 < N) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int n = n0 + u * 8;
            if (n + 8 <= N) {
              uint4 val;
              val.x = pack_bf16x2(__uint_as_float(r[u * 8 + 0]), __uint_as_float(r[u * 8 + 1]));
              val.y = pack_bf16x2(__uint_as_float(r[u * 8 + 2]), __uint_as_float(r[u * 8 + 3]));
              val.z = pack_bf16x2(__uint_as_float(r[u * 8 + 4]), __uint_as_float(r[u * 8 + 5]));
              val.w = pack_bf16x2(__uint_as_float(r[u * 8 + 6]), __uint_as_float(r[u * 8 + 7]));
              store_unit(epi, row, n, val);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

template <int BN, int AR = 128>
static cudaError_t launch_gemm_bn(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                                  const Epilogue& epi, cudaStream_t stream) {
  using C = GemmCfg<BN, AR>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tc_kernel<BN, AR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::SMEM));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((M + C::BM - 1) / C::BM) * ((N + BN - 1) / BN) * epi.k_splits;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  prof_mark(stream, true, g_prof_class);
  cudaError_t e = launch_k(gemm_bf16_tc_kernel<BN, AR>, dim3(grid), dim3(256), C::SMEM, stream,
                           epi.pdl && g_pdl && (g_pdl_mask & 1), ta, tb, M, N, K, epi);
  prof_mark(stream, false, g_prof_class);
  if (e != cudaSuccess) return e;
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_gemm(const uint16_t* A, int64_t lda, const uint16_t* B, int64_t ldb, int M, int N, int K,
                        const Epilogue& epi, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (K % 64 != 0) return cudaErrorInvalidValue;
  int BN = N > 128 ? 256 : 128;
  Epilogue ep = epi;
  ep.k_splits = 1;
  // skinny M (decode, B > 8): BN = 128 (c4 layer-step 4 % faster than 256-wide tiles; c3 a1, 45
  // tiles of 256, 111.6 vs 114.8 us per layer-step); ZDC_SKINNY_BN=256 forces 256 (diagnostic builds)
  static const int skinny_bn = knob("ZDC_SKINNY_BN", 0);
  static const int skinny_ar = knob("ZDC_SKINNY_AR", 0);  // 128 = load full 128-row A tiles (round 1)
  const bool skinny = epi.ws && epi.ws_cnt && M <= 128 && N % 8 == 0;
  if (skinny && N > 128) BN = skinny_bn == 256 ? 256 : 128;
  // A rows per stage: the batch rounded up to 32 / 64 (more weight stages in flight), else 128
  const int AR = !skinny || skinny_ar == 128 ? 128 : M <= 32 ? 32 : M <= 64 ? 64 : 128;
  if (skinny) {
    // split K so the weight stream spreads over the SMs (>= 4 stage blocks per split): the split
    // count of best wave efficiency items / (rounds x SMs), items = tiles x sk, sk <= 4 (ties: fewer
    // splits) -- c3 a1 (90 tiles of 128) 3, c3 a5 / c4 a1 (40) 3, c4 a5 (64) 2
    const int tiles = (N + BN - 1) / BN, kbs = K / 64;
    int sk = 1;
    double best = 0.0;
    for (int c = 1; c <= 4; ++c) {
      const int items = tiles * c, rounds = (items + num_sms() - 1) / num_sms();
      const double eff = static_cast<double>(items) / (static_cast<double>(rounds) * num_sms());
      if (eff > best + 1e-9) {
        best = eff;
        sk = c;
      }
    }
    if (sk > kbs / 4) sk = kbs / 4;
    if (sk > 1) {
      const int kpb = (kbs + sk - 1) / sk;
      ep.k_splits = (kbs + kpb - 1) / kpb;  // every split keeps >= 1 k-block
    }
  }
  // N-fastest raster for a large A: concurrent CTAs share A rows (read once from HBM) while the
  // weights B stay L2-resident; the default M-fastest order re-reads A once per N-tile (c4 prefill
  // a1: 174 GB of DRAM reads for 8.7 GB of operands, ncu).  ZDC_GEMM_RASTER=0/1 forces it.
  static const int raster_env = knob("ZDC_GEMM_RASTER", -1);
  const double a_bytes = static_cast<double>(M) * K * 2;
  // band: the N-blocks whose weight tiles fit ~40 MB of L2 (ZDC_GEMM_RASTER=0 keeps M-fastest,
  // = n forces a band of n)
  const int n_tiles_all = (N + BN - 1) / BN;
  int band = std::max(1, static_cast<int>(40e6 / (static_cast<double>(BN) * K * 2)));
  if (band > n_tiles_all) band = n_tiles_all;
  ep.raster_n = raster_env >= 0 ? raster_env : (a_bytes > 128e6 && N > BN ? band : 0);
  CUtensorMap ta, tb;
  if (!make_tmap_2d(&ta, A, K, M, lda * 2, 64, AR, 128)) return cudaErrorInvalidValue;
  if (!make_tmap_2d(&tb, B, K, N, ldb * 2, 64, BN, 128)) return cudaErrorInvalidValue;
  if (AR == 32)
    return BN == 256 ? launch_gemm_bn<256, 32>(ta, tb, M, N, K, ep, stream)
                     : launch_gemm_bn<128, 32>(ta, tb, M, N, K, ep, stream);
  if (AR == 64)
    return BN == 256 ? launch_gemm_bn<256, 64>(ta, tb, M, N, K, ep, stream)
                     : launch_gemm_bn<128, 64>(ta, tb, M, N, K, ep, stream);
  return BN == 256 ? launch_gemm_bn<256>(ta, tb, M, N, K, ep, stream)
                   : launch_gemm_bn<128>(ta, tb, M, N, K, ep, stream);
}

}  // namespace zdc

extern "C" {
// zdc_profile(1) starts per-kernel-class event timing (eager launches only: zdc_decode bypasses
// its CUDA graphs while profiling); zdc_profile_read synchronises and returns, per class, the
// summed milliseconds and launch counts since the last read, then clears them.
void zdc_profile(int enable) { zdc::g_prof.on = enable != 0; }
int zdc_profile_read(float* ms, int64_t* count, int n) {
  using namespace zdc;
  for (int i = 0; i < n; ++i) {
    if (ms) ms[i] = 0.f;
    if (count) count[i] = 0;
  }
  for (auto& m : g_prof.marks) {
    cudaEventSynchronize(m.second.second);
    float t = 0.f;
    cudaEventElapsedTime(&t, m.second.first, m.second.second);
    if (m.first < n) {
      if (ms) ms[m.first] += t;
      if (count) count[m.first] += 1;
    }
    g_prof.pool.push_back(m.second.first);
    g_prof.pool.push_back(m.second.second);
  }
  g_prof.marks.clear();
  return kProfClasses;
}
}
