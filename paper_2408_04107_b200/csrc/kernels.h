// kernels.h — host-side launch interface of the ZDC sm_100a kernels (internal to libzdc.so).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "knobs.h"

namespace zdc {

// Where the a1 projection writes its outputs: Q' to a staging matrix,
// K'/V' straight into the compressed KV cache (the append of a2 fused into the epilogue).
// Output column n of the packed [Q'|K'|V'] row: n < nq -> Q' col n; n < nq+nk -> K' of KV head
// (n-nq)/rk, dim (n-nq)%rk; else V' of head (n-nq-nk)/rv, dim (n-nq-nk)%rv.
// Token row m = b*S + t is written at cache position posmap ? posmap[t] : pos0 + t.
struct QkvDest {
  uint16_t* q = nullptr;
  int64_t ldq = 0;
  int nq = 0, nk = 0;
  uint16_t* k = nullptr;
  uint16_t* v = nullptr;
  int rk = 0, rv = 0;
  int S = 1;
  int64_t kb = 0, kg = 0, vb = 0, vg = 0;  // element strides per sequence / per KV head
  int pos0 = 0;
  const int* pos_ptr = nullptr;  // if set, pos0 is read from device memory (graph-replayable decode)
  int pos_cap = 0;               // with pos_ptr: rows per (sequence, KV head); *pos_ptr is clamped to pos_cap - 1
  const int* posmap = nullptr;
};

// Ulysses SP send layout (comm.cpp, zdc_sp_prefill_ulysses): column n of a local token row goes to
// the slab of the rank that owns its head: send[q][m][cols], cols = hq (Q' of the rank's N_h/P
// heads) + kq (K' of its N_kv/P groups) + vq (V').  hq, kq, vq are multiples of 8.
struct UlyssesDest {
  uint16_t* send = nullptr;
  int nq = 0, nk = 0;          // Q' / K' columns of the full projection row
  int hq = 0, kq = 0, vq = 0, cols = 0;
  int64_t rows = 0;            // rows per slab (B * n_local)
};

struct Epilogue {
  int mode = 0;  // 0 = plain bf16 D[M][ldd]; 1 = QKV scatter (QkvDest); 2 = Ulysses send slabs (UlyssesDest)
  uint16_t* d = nullptr;
  int64_t ldd = 0;
  QkvDest qkv;
  UlyssesDest uly;
  int* len_inc = nullptr;  // if set, the kernel increments *len_inc once (decode: advances the layer length)
  int len_cap = 0;         // ... saturating at len_cap: a step with *len_inc >= len_cap sets *err instead
  int* err = nullptr;      // device overflow flag (reported by zdc_cache_sync)
  // split-K for skinny M (M <= 128, few output tiles: decode at B > 8): fp32 workspace [M][N] and
  // per-tile arrival counters, both zero between launches; the last split of a tile applies the
  // epilogue above to the summed tile.  k_splits is chosen by launch_gemm when ws is set.
  float* ws = nullptr;
  int* ws_cnt = nullptr;
  int k_splits = 1;
  int pdl = 0;  // launch with programmatic dependent launch (decode chains)
  int raster_n = 0;  // tile order: 0 M-fastest; n > 0 bands of n N-blocks, N fastest (launch_gemm, large A)
};

#ifdef __CUDACC__
// SP layouts: global position of local row t of rank q (0 contiguous, 1 zigzag: chunks q, 2P-1-q)
__device__ __forceinline__ int sp_global_pos(int S, int P, int q, int layout, int t) {
  const int n = S / P;
  if (layout == 0) return q * n + t;
  const int c = S / (2 * P);
  return t < c ? q * c + t : (2 * P - 1 - q) * c + (t - c);
}

// Decode length advance (one thread, after every reader of the old length): saturates at len_cap;
// a step that found the cache full sets the overflow flag instead (zdc_cache_sync reports it).
__device__ __forceinline__ void advance_len(const Epilogue& e) {
  const int v = *e.len_inc;
  if (e.len_cap > 0 && v >= e.len_cap) {
    if (e.err) *e.err = 1;
  } else {
    *e.len_inc = v + 1;
  }
}
#endif

// ---- tensor maps (driver entry point resolved at runtime; no -lcuda link)
bool make_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner_elems, uint64_t outer_rows,
                  uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes);

int num_sms();

// ---- a1 / a5 projection GEMM: D[M][N] = A[M][K] * B[N][K]^T (tcgen05, TMA, TMEM)
cudaError_t launch_gemm(const uint16_t* A, int64_t lda, const uint16_t* B, int64_t ldb, int M, int N, int K,
                        const Epilogue& epi, cudaStream_t stream);

// ---- decode: skinny projection (B <= 8 rows), weights streamed once from HBM
bool gemv_supported(int B, int K);  // else the tcgen05 GEMM takes the projection
cudaError_t launch_gemv(const uint16_t* W, const uint16_t* x, int64_t ldx, int B, int N, int K,
                        const Epilogue& epi, cudaStream_t stream);

// ---- a3 prefill attention (tcgen05 flash attention at head dim r, causal, LSE out)
struct PrefillAttnArgs {
  const uint16_t* q;   // Q' staging [B*S][ldq]; head h at cols h*rk
  int64_t ldq;
  const uint16_t* k;   // K' cache rows: sequence b, KV head g, position p at ((b*Nkv+g)*S_cap + p)*rk
  const uint16_t* v;   // V' likewise with rv
  int S_cap;           // row capacity per (b, g) of the K/V buffers
  uint16_t* o;         // O' [B*S][ldo]; head h at cols h*rv
  int64_t ldo;
  float* lse;          // [B][Nh][S] (natural log of the Eq. 3 denominator), may be null
  int B, S, Nh, Nkv, rk, rv;
  float scale;         // 1/sqrt(d_h) (reading c2)
  int q_pos0;          // global position of query row t is q_pos0 + t (SP chunks)
  int q_row0;          // first row of this chunk inside the Q'/O' matrices
  int n_q;             // number of query rows of this launch (per sequence)
  // key addressing: kv_mode 0 = position-ordered rows (above); 1 = SP gather buffer
  // [P][K|V][B][Nkv][sp_n_local][r]: key position -> (owner rank, local row) by the layout;
  // 2 = zigzag half-major gather buffer [2][P][K|V][B][Nkv][sp_chunk][r] (overlapped exchange)
  int kv_mode = 0;
  int sp_P = 1, sp_n_local = 0, sp_chunk = 0, sp_zigzag = 0;
  int64_t v_row_off = 0;      // V row = K row + v_row_off (kv_mode 1: both maps share the base)
  int64_t kv_rows_total = 0;  // rows of the K/V tensor maps (0 = B * Nkv * S_cap)
};
cudaError_t launch_prefill_attention(const PrefillAttnArgs& a, cudaStream_t stream);

// ---- SP x token split (sp_split.cu, NEXT-2): the global top-g selection across ranks
// scores of this rank's local query rows (global positions for the mean-mode adjustment) into its
// slot out[B][n_local]; lse [B][Nh][n_local]
cudaError_t launch_sp_importance(const float* lse, int n_local, int Nh, int B, int mode, int S, int P, int p,
                                 int layout, float* out, cudaStream_t s);
// gathered score slots [P][B][n_local] -> scores [B][ld] in global position order
cudaError_t launch_sp_scores_global(const float* slots, int P, int B, int n_local, int S, int layout, float* scores,
                                    int64_t ld, cudaStream_t s);
// zero dims [r_u, w) of the rows of unimportant tokens in gather-buffer slots [q0, q1) of
// [P][K|V][B][Nkv][n_local][w] (class of (b, position) at cls[b ld + position])
cudaError_t launch_sp_truncate(uint16_t* gbuf, int q0, int q1, int P, int layout, int S, int B, int Nkv, int n_local,
                               int w, int r_u, const uint8_t* cls, int64_t ld_cls, cudaStream_t s);

// SP decode partial merge: {O'_p bf16 [B][ldo], LSE_p [B][Nh]} -> f32 slot [B][Nh][rv+1]; slots
// [P][...] -> O' (bf16) and LSE merged over the ranks
cudaError_t launch_sp_decode_pack(const uint16_t* o, int64_t ldo, const float* lse, int B, int Nh, int rv, float* slot,
                                  cudaStream_t s);
cudaError_t launch_sp_decode_merge(const float* slots, int P, int B, int Nh, int rv, uint16_t* o, int64_t ldo,
                                   float* lse, cudaStream_t s);

// ---- Ulysses SP re-layouts (sp_ulysses.cu).  Global position of local row t of rank q:
// layout 0 contiguous (q n + t), 1 zigzag (chunks q and 2P-1-q of 2P).
// recv[src][B][n_local][cols] (this rank's heads, from every rank) -> Q' [B*S][hq] and the K'/V'
// cache of this rank's groups [B][nkv_loc][S_cap][rk] / [rv], in global position order
cudaError_t launch_ulysses_unpack_qkv(const uint16_t* recv, int P, int B, int n_local, int S, int layout, int hq, int kq,
                                      int vq, int rk, int rv, uint16_t* q, uint16_t* kc, uint16_t* vc, int S_cap,
                                      cudaStream_t s);
// O' [B*S][ho] (this rank's heads, position order) -> send[dst][B][n_local][ho] (dst's tokens)
cudaError_t launch_ulysses_pack_o(const uint16_t* o, int P, int B, int n_local, int S, int layout, int ho,
                                  uint16_t* send, cudaStream_t s);
// recv[src][B][n_local][ho] (src's heads for this rank's tokens) -> O'_local [B*n_local][ko_p]
// (head-major columns: src * ho + c; padding columns >= P * ho zeroed)
cudaError_t launch_ulysses_unpack_o(const uint16_t* recv, int P, int B, int n_local, int ho, uint16_t* o, int ko_p,
                                    cudaStream_t s);
cudaError_t launch_prefill_attention_v3(const PrefillAttnArgs& a, cudaStream_t stream);
cudaError_t launch_prefill_attention_v4(const PrefillAttnArgs& a, cudaStream_t stream);
bool prefill_attention_v4_supported(int rk);

// ---- a3 decode attention: split-K over the context (one or two pools) + LSE-merge combine
struct DecodeAttnArgs {
  const uint16_t* q = nullptr;  // Q' [B][ldq]; head h at cols h*rk
  int64_t ldq = 0;
  // pool 0 (important rows, or every row without a token split): row i of (b, g) at
  // ((b*Nkv+g)*S_cap + i) * width
  const uint16_t* k = nullptr;
  const uint16_t* v = nullptr;
  int rk = 0, rv = 0;
  // pool 1 (unimportant rows, truncated width; token split only)
  const uint16_t* k1 = nullptr;
  const uint16_t* v1 = nullptr;
  int rk1 = 0, rv1 = 0;
  int S_cap = 0;
  int len = 0;                   // upper bound on any pool's rows (fixes the split count)
  const int* len_ptr = nullptr;  // uniform cache: pool-0 rows = *len_ptr + 1
  int kv_fp8 = 0;                // FP8 cache rows (NEXT-4): launch_decode_attention -> launch_decode2_f8
  const int* n0_ptr = nullptr;   // token split: per-sequence rows of pool 0 / pool 1 [B]
  const int* n1_ptr = nullptr;
  uint16_t* o = nullptr;  // O' [B][ldo]
  int64_t ldo = 0;
  float* lse = nullptr;   // [B][Nh]
  float* part = nullptr;  // scratch [B][Nh][2 * splits][rv + 2]
  int* counters = nullptr;  // scratch [B][Nkv] zero-initialised; the last CTA per (b, g) merges
  int prefetch_before_wait = 1;  // stage cached rows before the PDL dependency wait
  // weights of the next kernels (a5 of this layer, a1 of the next) pulled into L2 while this
  // latency-bound kernel leaves HBM bandwidth idle; split evenly over the CTAs
  const void* pf_ptr[2] = {nullptr, nullptr};
  int64_t pf_bytes[2] = {0, 0};
  int B = 0, Nh = 0, Nkv = 0;
  float scale = 0.f;
  int splits = 1;
};
cudaError_t launch_decode_attention(const DecodeAttnArgs& a, cudaStream_t stream);
// v3 (decode_attn3.cu): byte-balanced flat split of every (sequence, KV head) pair's pool-0 and
// pool-1 rows over one resident warp set; partials [B][Nh][128][rv+2], counters [B][Nkv]
bool decode3_supported(const DecodeAttnArgs& a);
cudaError_t launch_decode_attention3(const DecodeAttnArgs& a, cudaStream_t stream);
// tcgen05 decode attention for grouped-query layers (decode_attn_tc.cu): uniform rank r in
// {64, 128}, G in {2, 4, 8, 16}, device-side length (len_ptr); a.splits from decode_tc_splits
bool decode_attention_tc_supported(int rk, int rv, int G);
int decode_tc_splits(int B, int Nkv, int len);
cudaError_t launch_decode_attention_tc(const DecodeAttnArgs& a, cudaStream_t stream);
cudaError_t launch_decode2_partial(const DecodeAttnArgs& a, int width, const uint16_t* kp, const uint16_t* vp,
                                   int pool, int slot0, int nslots, cudaStream_t s);
int decode2_splits(int B, int Nkv, int len, int width, int G);
// NEXT-4: decode attention over the FP8 cache (decode_attn2.cu; uniform rank, one pool)
cudaError_t launch_decode2_f8(const DecodeAttnArgs& a, cudaStream_t s);
// NEXT-4 (kv_quant.cu): bf16 rows -> FP8 E4M3 rows (r codes, f32 scale, 12 pad bytes), reading c23.
// Rows (bg, t) for bg < n_bg, t in [t0, t0 + T): src at (bg * src_bg + t) * w elements (bf16), dst
// at (bg * S_cap + pos) * (w + 16) bytes with pos = (pos_ptr ? min(*pos_ptr, S_cap - 1) : 0) + t.
cudaError_t launch_quantize_kv(const uint16_t* src, int64_t src_bg, uint8_t* dst, int S_cap, int n_bg, int t0, int T,
                               int w, const int* pos_ptr, cudaStream_t s);
int decode_splits(int B, int Nkv, int len);

// ---- the fused decode layer-step (decode_fused.cuh): a1 + a2 + a3 + a5 of a run of consecutive
// layers in one persistent kernel, for B <= 8 on uniform-rank layers (width RK = r_k = r_v padded)
struct DecLayer {                  // per-layer pointers (device-resident table, written at bind)
  const uint16_t* wqkv;            // [n_qkv][d]
  const uint16_t* wo;              // [d][ko_p]
  uint16_t* kc;                    // K'/V' cache: row (b, g, p) at ((b*Nkv+g)*S_cap + p)*RK
  uint16_t* vc;
  int* len_ptr;                    // cached rows before this step; advanced by the kernel
};
struct DecFusedArgs {
  const DecLayer* layers = nullptr;  // [nl] layers of the run, chained: y of layer i feeds layer i+1
  int nl = 1;
  const uint16_t* x = nullptr;     // [B][ldx] input of the first layer
  int64_t ldx = 0;
  uint16_t* y = nullptr;           // [B][ldy] output of every layer (the last one is the result)
  int64_t ldy = 0;
  uint16_t* q = nullptr;           // Q' staging [B][ldq]
  int64_t ldq = 0;
  float* part = nullptr;           // [B][Nh][splits][RK+2]
  float* lse = nullptr;            // [B][Nh]
  uint16_t* o = nullptr;           // O' [B][ko_p] (bf16), written by the last CTA of each (b, g)
  int* counters = nullptr;         // [B][Nkv] arrival counters, zero between launches
  unsigned long long* gbar = nullptr;  // grid barrier arrival counter (monotonic), zero-initialised
  unsigned long long* trace = nullptr;  // optional [ncta][16] globaltimer stamps (ZDC_FUSED_TRACE)
  int B = 0, d = 0, n_qkv = 0, nq = 0, nk = 0, Nh = 0, Nkv = 0, S_cap = 0, splits = 1, ko_p = 0;
  float scale = 0.f;
  // ring geometry (set by the launcher)
  int slot_bytes = 0, spw = 0, ring_extra = 0, xw = 0, rps = 32;
  int stage_part = 0, pst_floats = 0;
  int64_t pst_bytes = 0;
  int* err = nullptr;                   // device overflow flag: a step found *len_ptr >= S_cap
};
bool decode_fused_supported(int B, int RK, int G);
int decode_fused_splits(int B, int Nkv);
cudaError_t launch_decode_fused(const DecFusedArgs& a, int RK, cudaStream_t s);
unsigned long long* fused_trace_buffer();  // null unless ZDC_FUSED_TRACE is set

// ---- the cluster decode layer-step (decode_cluster.cuh): one thread-block cluster of C CTAs per
// KV group does a1 + a2 + a3 + a5 of ONE layer for that group (tcgen05 projections, DSMEM
// exchanges); the groups meet only in the fp32 y accumulator (B <= 8, uniform rank RK = r_k = r_v
// padded, RK in {16, 32, 64, 128}, G * RK <= 256, d % (64 C) == 0)
struct DecClusterArgs {
  const uint16_t* wqd = nullptr;   // W_QKV decode copy: [Nkv][d/64] tiles of (G+2)*RK rows x 64 K,
                                   // each the SW128 K-major shared-memory image (pack_qkv_decode)
  const uint16_t* wod = nullptr;   // W_O decode copy, group-major [Nkv][d][G*RK] (pack_wo_decode)
  uint16_t* kc = nullptr;          // K'/V' cache: row (b, g, p) at ((b*Nkv+g)*S_cap + p)*RK
  uint16_t* vc = nullptr;
  int* len_ptr = nullptr;          // cached rows before this step; advanced by the kernel
  int* err = nullptr;              // device overflow flag: a step found *len_ptr >= S_cap
  const uint16_t* x = nullptr;     // [B][ldx]
  int64_t ldx = 0;
  uint16_t* y = nullptr;           // [B][ldy]
  int64_t ldy = 0;
  float* ybuf = nullptr;           // [8][d] fp32 accumulator, zero between launches
  int* ycnt = nullptr;             // [C] arrival counters, zero between launches
  float* lse = nullptr;            // [B][Nh]
  unsigned long long* trace = nullptr;  // optional [ncta][16] globaltimer stamps (ZDC_FUSED_TRACE)
  int B = 0, d = 0, nq = 0, nk = 0, Nh = 0, Nkv = 0, S_cap = 0;
  int C = 0;                       // cluster size (CTAs per KV group)
  int l2_prefetch = 7;             // bulk L2 prefetch of: 1 phase-1 weights past the ring, 2 cached rows, 4 W_O
  float scale = 0.f;
  // geometry (set by the launcher)
  int nslot = 0, attn_warps = 0, tmem_cols = 0;
};
bool decode_cluster_supported(int B, int RK, int G);
bool decode_cluster_layer_ok(int RK, int G);  // the layer gets a W_O decode copy
// cluster size for N_kv groups (0 = the cluster kernel cannot hold every group at once)
int decode_cluster_size(int B, int RK, int G, int Nkv, int d);
cudaError_t launch_decode_cluster(const DecClusterArgs& a, int RK, cudaStream_t s);
// tensor map of the W_O decode copy [Nkv*d][K3] in boxes of KB3 x 128 rows (swizzle = KB3 * 2 bytes)
bool cluster_wo_tmap(CUtensorMap* tw, const uint16_t* wod, int Nkv, int d, int K3, int KB3);
// W_QKV^T [n_qkv][d] -> the decode copy wqd (tiles of group g, k-block kb: rows (Q'_g | K'_g | V'_g)
// x 64 K in the 128-byte-swizzled K-major image the tcgen05 A operand reads)
cudaError_t launch_pack_qkv_decode(const uint16_t* wqkv_t, uint16_t* wqd, int d, int nq, int nk, int Nkv, int G,
                                   int RK, cudaStream_t s);
// W_O^T [d][ko_p] -> the group-major decode copy wod[g][n][j] = wo_t[n][g*K3 + j]
cudaError_t launch_pack_wo_decode(const uint16_t* wo_t, uint16_t* wod, int d, int ko_p, int Nkv, int K3,
                                  cudaStream_t s);

// ---- weight packing (load time): f32/bf16 full-rank folded -> truncated, padded, bf16
cudaError_t launch_pack_weights_bf16(const uint16_t* wq, const uint16_t* wk, const uint16_t* wv,
                                     const uint16_t* wo, uint16_t* wqkv_t, uint16_t* wo_t, int d, int Nh,
                                     int Nkv, int dh, int rk, int rv, int rk_p, int rv_p, int ko_p,
                                     cudaStream_t stream);

// ---- a4 selection + class-aware packing (select.cu)
cudaError_t launch_importance(const float* lse, int T, int Nh, int B, int t0, int mode, float* scores, int64_t ld,
                              float* out_copy, int64_t ld_copy, const int* pos_ptr, cudaStream_t s);
// eviction (H2O-ZDC, reading c26): after a non-representative layer's decode attention, the new token
// (the last pool_I row) leaves pool_I when its representative classed it unimportant
cudaError_t launch_evict_last(const uint8_t* cls, int64_t ld_cls, int* n_i, int* n_u, int* pos_u, int64_t ld_pos,
                              const int* len_ptr, int S_cap, int B, cudaStream_t s);
cudaError_t launch_select(const float* scores, int64_t ld, int S, int g_bp, int B, uint8_t* cls, float* tau,
                          cudaStream_t s, int* nan_flag = nullptr);
cudaError_t launch_truncate(uint16_t* kv, int width, int r_u, int B, int Nkv, int S, int S_cap, const uint8_t* cls,
                            int64_t ld_cls, cudaStream_t s);
cudaError_t launch_rank(const uint8_t* cls, int64_t ld_cls, int S, int B, int* didx, int64_t ld_didx, int* pos_i,
                        int* pos_u, int64_t ld_pos, int* n_i, int* n_u, cudaStream_t s);
cudaError_t launch_pack(const uint16_t* src, int w, uint16_t* pool_i, uint16_t* pool_u, int wu, int r_u, int B, int Nkv,
                        int S, int S_cap, const int* didx, int64_t ld_didx, cudaStream_t s);
cudaError_t launch_append(const uint16_t* knew, const uint16_t* vnew, int w, int Nkv, uint16_t* ki, uint16_t* vi,
                          uint16_t* ku, uint16_t* vu, int wu, int r_u, int S_cap, int* n_i, int* n_u, int* pos_i,
                          int* pos_u, int64_t ld_pos, const int* len_ptr, const uint8_t* rep_cls, int64_t ld_cls,
                          int is_rep, int B, cudaStream_t s);
cudaError_t launch_classify(const float* lse, int Nh, int mode, const float* tau, float* scores, uint8_t* cls,
                            int64_t ld, float* out_copy, int64_t ld_copy, int w, int Nkv, uint16_t* ki, uint16_t* vi,
                            uint16_t* ku, uint16_t* vu, int wu, int r_u, int S_cap, int* n_i, int* n_u, int* pos_i,
                            int* pos_u, const int* len_ptr, int B, cudaStream_t s);

extern int64_t g_launches;  // kernels enqueued by the last API call
extern bool g_pdl;          // launch decode kernels with programmatic stream serialization
extern int g_pdl_mask;      // bit 0: projections, bit 1: attention

// Launch with the programmatic-dependent-launch attribute (when pdl): the kernel may start while
// its predecessor is still running; it must call pdl_wait() before reading the predecessor's output.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? attr : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- per-kernel-class timing (zdc_profile): CUDA events bracket each launch on its stream
enum ProfClass { kProfGemmQkv = 0, kProfAttnPrefill, kProfGemmO, kProfGemvQkv, kProfAttnDecode, kProfAttnCombine,
                 kProfGemvO, kProfOther, kProfDecodeLayer, kProfClasses };
extern int g_prof_class;  // class the next launches belong to (set by the orchestration)
void prof_mark(cudaStream_t s, bool begin, int cls);
bool prof_enabled();
cudaError_t launch_set_int(int* p, int v, cudaStream_t s);

}  // namespace zdc
