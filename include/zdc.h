/*
 * zdc.h — C ABI of the B200-native ZDC hot path (zero-delay QKV compression,
 * arxiv 2408.04107).  "P:<n>" cites /root/reference/PAPER.md line n (section / equation
 * given alongside); DESIGN.md §3 lists every reading of a silent or ambiguous passage.
 *
 * Library: libzdc.so (built in-tree for sm_100a).  Every entry point is extern "C",
 * takes plain pointers and sizes, and never takes ownership of a caller buffer.
 *
 * Conventions
 *   - Status: ZDC_OK (0) or a negative zdc_status.  zdc_last_error() returns the
 *     message of the last failing call on the calling thread.
 *   - Device calls are asynchronous on `stream` (a cudaStream_t passed as void*; NULL =
 *     legacy default stream).  Argument and shape errors are detected synchronously,
 *     before anything is enqueued; asynchronous CUDA / NCCL faults surface on the next
 *     call as ZDC_ERR_CUDA / ZDC_ERR_NCCL.
 *   - Element types: "bf16" = IEEE bfloat16 bit patterns (uint16_t), "f32" = float,
 *     "f64" = double.  Matrices are dense row-major unless stated.
 *   - Ownership: the caller owns every buffer (host and device).  The library owns the
 *     zdc_ctx host metadata and, after zdc_comm_init, the NCCL communicator; both are
 *     released by zdc_ctx_destroy.
 *   - There is no CPU fallback: a call that needs the GPU fails with ZDC_ERR_CUDA when
 *     no sm_100 device is present.
 */
#ifndef ZDC_H
#define ZDC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ZDC_OK = 0,
  ZDC_ERR_INVALID_ARG = -1,     /* null pointer, non-finite input, aliasing, bad enum */
  ZDC_ERR_SHAPE = -2,           /* dimension mismatch; the message names both shapes  */
  ZDC_ERR_NOT_ORTHONORMAL = -3, /* fold produced R with |R^T R - I| > 1e-10            */
  ZDC_ERR_NO_CONVERGENCE = -4,  /* one-sided Jacobi did not converge in 60 sweeps      */
  ZDC_ERR_CAPACITY = -5,        /* len + S > max_seq, B > max_batch                    */
  ZDC_ERR_CUDA = -6,
  ZDC_ERR_NCCL = -7,
  ZDC_ERR_UNSUPPORTED = -8,     /* shape the kernels do not implement (see zdc_ctx_create) */
  ZDC_ERR_STATE = -9            /* call order: unbound ctx, prefill on a non-empty cache,
                                   representative layer has not classified a position  */
} zdc_status;

const char* zdc_last_error(void);
const char* zdc_version(void);

/* Model dimensions (Table tab:symbols): d = d_model, N_h = n_heads,
 * d_h = d_head = d / N_h in the paper; GQA (n_kv_heads < n_heads) is reading c4. */
typedef struct {
  int32_t n_layers, d_model, n_heads, n_kv_heads, d_head;
} zdc_dims;

/* Compression plan {g^l, p_QK^i, p_QK^u, p_VL^i, p_VL^u} (§5.2 Eqs. 5-6),
 * expressed as integer kept ranks (reading c6: r = ceil((1-p) d_h)) and g in basis
 * points (reading c11).  Every array has n_layers entries.
 *   1 <= r_*_unimp[l] <= r_*_imp[l] <= d_head.
 *   g_bp[l] in [0, 10000]; 10000 = no token split at layer l (all tokens important).
 *   group_rep[l] <= l and group_rep[group_rep[l]] == group_rep[l]; g_bp and the four
 *     ranks are equal within a group (reading c15).  The representative classifies the
 *     tokens; the other layers of the group reuse its classes.
 *   importance_mode 0 = raw sum_h sum_{k<=t} exp(s) (default);
 *                   1 = per-key mean (minus log(t+1) per head, reading c10). */
typedef struct {
  const int32_t *r_qk_imp, *r_qk_unimp, *r_vl_imp, *r_vl_unimp;
  const int32_t *g_bp;
  const int32_t *group_rep;
  int32_t importance_mode;
  /* NEXT-4 (GEAR-ZDC, P:1642 DEL: "quantizes each matrix element of the compressed data after ZDC
   * compression and dequantizes them before ZDC decompression"): 1 = the compressed K'/V' cache is
   * stored as FP8 E4M3 codes with one f32 scale per row (token, KV head), reading c23 (scale =
   * max|x| / 448, RNE + satfinite); the prompt attends at full precision, decode attends the
   * quantized cache (its own new row included).  Uniform-rank plans with padded ranks in
   * {32, 64, 96, 128} only (else ZDC_ERR_UNSUPPORTED).  Row layout: r codes, the f32 scale,
   * 12 pad bytes (r + 16 bytes vs 2 r for bf16).  0 = bf16 cache. */
  int32_t kv_fp8;
} zdc_plan;

/* ------------------------------------------------------------------------------------
 * (1) Offline fold of ONE layer — host, fp64, NOT part of the timed hot path.
 *
 * P:977 and P:989-990 (§4.3, "Finding common rotation matrix offline"): per head
 * (here per KV group g, reading c4) stack [Q^h for h in group; K^g] ("concatenate
 * them into a 2 Sigma_S x d_h matrix") and [V^g; (W_O^h)^T for h in group] ((Sigma_S + d) x d_h),
 * with Q^h = X_c W_Q^h etc. (Eq. 1); R = right singular vectors (A = U Sigma R^T,
 * P:300 §2.2), sorted by non-increasing sigma, canonical signs (reading c5: the entry of
 * largest |.| of each column is positive, ties to the lowest row).  Fold (P:1204,
 * P:1218-1219, Lemma 1): W_Q^{R,h} = W_Q^h R_qk, W_K^{R,g} = W_K^g R_qk,
 * W_V^{R,g} = W_V^g R_vl, W_O^{R,h} = R_vl^T W_O^h (reading c1).
 * Algorithm: Householder QR of each stacked block (TSQR), then one-sided Jacobi SVD of
 * the d_h x d_h triangular factor (no Gram matrix, so tiny singular values keep their
 * relative accuracy).
 *
 *   wq [d][N_h d_h], wk [d][N_kv d_h], wv [d][N_kv d_h], wo [N_h d_h][d]: unfolded, f64.
 *   calib_x [n_calib][d]: this layer's inputs (stands in for the pruned, k-meaned history
 *     of P:1154-1167, reading c8).  n_calib (G+1) >= d_h else ZDC_ERR_SHAPE.
 *   r_qk, r_vl [N_kv][d_h][d_h] (column j = j-th right singular vector);
 *   sigma_qk, sigma_vl [N_kv][d_h] non-increasing;
 *   wq_f, wk_f, wv_f, wo_f: full-rank folded weights, same shapes as the inputs.
 * All outputs are caller-owned host buffers.  Non-finite input -> ZDC_ERR_INVALID_ARG.
 * ---------------------------------------------------------------------------------- */
zdc_status zdc_fold_weights(const zdc_dims* dims,
                            const double* wq, const double* wk, const double* wv, const double* wo,
                            const double* calib_x, int64_t n_calib,
                            double* r_qk, double* r_vl, double* sigma_qk, double* sigma_vl,
                            double* wq_f, double* wk_f, double* wv_f, double* wo_f);

/* (1b) NEXT-3: the same fold on the GPU at the paper's calibration scale (§5.1:
 * "we propose employing pruning and K-means clustering ... K-means ... consolidates vectors within
 * each cluster by averaging them into a single vector ... we conduct the K-means clustering on Q,
 * K, and V, respectively"; no K-means for W_L^h).  All pointers are DEVICE fp64, same
 * shapes as zdc_fold_weights; `workspace` is caller-owned device memory of at least
 * zdc_fold_gpu_workspace() bytes.  k_clusters <= 0 or >= n_calib: no consolidation (the plain fold
 * of P:989-990); else kmeans_iters Lloyd rounds per Q^h / K^g / V^g block (reading c21: centroid j
 * starts at row floor(j n / k), nearest by squared distance, ties -> lowest index, empty clusters
 * keep their centroid).  R comes from a Jacobi eigen-decomposition of each stack's Gram matrix
 * (eigenvectors = right singular vectors; sigma = sqrt(eigenvalue); canonical signs, reading c5).
 * d_head must be even and <= 128 (ZDC_ERR_UNSUPPORTED).  Asynchronous on `stream`. */
int64_t zdc_fold_gpu_workspace(const zdc_dims* dims, int64_t n_calib, int32_t k_clusters);
zdc_status zdc_fold_weights_gpu(const zdc_dims* dims, const double* wq, const double* wk, const double* wv,
                                const double* wo, const double* calib_x, int64_t n_calib, int32_t k_clusters,
                                int32_t kmeans_iters, double* r_qk, double* r_vl, double* sigma_qk,
                                double* sigma_vl, double* wq_f, double* wk_f, double* wv_f, double* wo_f,
                                void* workspace, int64_t workspace_bytes, void* stream);

/* NEXT-3 planner step (layers whose important / unimportant token sets repeat with
 * ratio > 95% share one representative).  classes: host uint8 [n_layers][positions] (nonzero =
 * important; every layer classified as its own representative, e.g. by zdc_cache_export after a
 * calibration prefill); positions = B * S.  Consecutive layers: layer l joins the current group when
 * the fraction of positions whose class equals the representative's exceeds threshold_bp / 10000
 * (strict, exact integer arithmetic; reading c22), else it starts a new group.  Writes group_rep
 * [n_layers] (a valid zdc_plan.group_rep). */
zdc_status zdc_layer_groups(const uint8_t* classes, int32_t n_layers, int64_t positions, int32_t threshold_bp,
                            int32_t* group_rep);

/* ------------------------------------------------------------------------------------
 * Context: host metadata only.  Device memory is caller-owned: query the three sizes,
 * allocate (any allocator; 256-byte aligned), bind.  zdc_ctx_bind zeroes the regions;
 * zdc_cache_reset empties the cache by resetting the per-layer lengths (host and device):
 * no kernel reads a cache row at or beyond its layer's length.
 *
 * Supported shapes (else ZDC_ERR_UNSUPPORTED): d_model % 64 == 0; d_head <= 128;
 * n_heads % n_kv_heads in {1,2,4,8} groups; every kept rank is stored zero-padded to a
 * multiple of 16 (zero columns are exact: they add 0 to every dot product); the padded
 * QK and VL ranks of a class must be equal (r_qk_imp ~ r_vl_imp, r_qk_unimp ~ r_vl_unimp).
 * ---------------------------------------------------------------------------------- */
typedef struct zdc_ctx zdc_ctx;

zdc_status zdc_ctx_create(const zdc_dims* dims, const zdc_plan* plan,
                          int32_t max_batch, int32_t max_seq, zdc_ctx** out);
zdc_status zdc_ctx_sizes(const zdc_ctx* ctx, int64_t* weight_bytes, int64_t* cache_bytes,
                         int64_t* scratch_bytes);
zdc_status zdc_ctx_bind(zdc_ctx* ctx, void* d_weights, void* d_cache, void* d_scratch);
void zdc_ctx_destroy(zdc_ctx* ctx);

/* Load ONE layer's full-rank folded weights (from zdc_fold_weights, or any fold):
 * truncate to the plan's important ranks ("drop the right p fraction of
 * columns of W_Q^R"; "discard p x d_h dimensions from each W_L^{R,h} and
 * concatenate"), zero-pad ranks to a multiple of 16, round to bf16 (RNE), and pack into
 * the bound weight region (layout: DESIGN.md §5).  Host f64 inputs; synchronous w.r.t.
 * the host buffers (they may be freed on return).  No compress op ever runs online. */
zdc_status zdc_load_folded(zdc_ctx* ctx, int32_t layer, const double* wq_f, const double* wk_f,
                           const double* wv_f, const double* wo_f, void* stream);
/* Same, from DEVICE bf16 full-rank folded weights (same shapes); asynchronous on stream.
 * Used by the benchmark for layers whose fp64 fold is never computed. */
zdc_status zdc_load_folded_device(zdc_ctx* ctx, int32_t layer, const uint16_t* wq_f,
                                  const uint16_t* wk_f, const uint16_t* wv_f,
                                  const uint16_t* wo_f, void* stream);

/* ------------------------------------------------------------------------------------
 * (2) Prefill (prompt processing) on an EMPTY cache, layers [l0, l1) chained:
 * y of layer l feeds x of layer l+1.  Per layer (§5.1, fig:overview P:938):
 *   a1  [Q'|K'|V'] = x W_QKV^R           (Eq. 1 with folded, truncated weights)
 *   a2  append K'/V' to the compressed KV cache (P:774-776 DEL, P:813 DEL)
 *   a3  O'^h = softmax(Q'^h K'^T / sqrt(d_h)) V'  causal (Eqs. 2-3; scale: reading c2)
 *   a4  (representative layers with g_bp < 10000) importance + top-g selection
 *   a5  y = O' W_O^R                       (Eq. 4 with the folded W_O)
 *   x, y: device bf16 [B][S][d]; must not alias.  B <= max_batch, S <= max_seq.
 *   importance: optional device f32 [n_layers][B][max_seq]; row (l, b) receives the
 *     representative layer l's token scores (log of sum_h sum_{k<=t} exp(s), reading c9).
 * Every sequence of the batch has length S.  Rejects a non-empty cache (ZDC_ERR_STATE).
 * ---------------------------------------------------------------------------------- */
zdc_status zdc_prefill(zdc_ctx* ctx, int32_t l0, int32_t l1, const uint16_t* x, uint16_t* y,
                       int32_t B, int32_t S, float* importance, void* stream);

/* (3) Decode (token generation): one new token per sequence, appended at position
 * len[l] of each layer l in [l0, l1) (each layer tracks its own length; all B sequences
 * share it).  The new token's K'/V' are appended before it attends, so it attends to
 * itself.  With a token split, a representative layer classifies the token as important
 * iff its score > tau (the k-th prompt score, reading c12); a non-representative layer
 * requires its representative to have processed this position (else ZDC_ERR_STATE).
 *   x, y: device bf16 [B][d]; must not alias.  B must equal the prefill batch. */
zdc_status zdc_decode(zdc_ctx* ctx, int32_t l0, int32_t l1, const uint16_t* x, uint16_t* y,
                      int32_t B, void* stream);

/* ------------------------------------------------------------------------------------
 * (4) Sequence-parallel prefill (§5.3 motivates exchanging compressed data;
 * the exchange here is an all-gather of compressed K'/V', reading c17).  Rank p of P
 * holds S_total/P tokens of every sequence:
 *   layout 0 = contiguous (rank p holds [p S/P, (p+1) S/P)),
 *   layout 1 = zigzag (2P chunks of S/(2P); rank p holds chunks p and 2P-1-p),
 *   layout 2 = zigzag with the exchange overlapped: the gather buffer is half-major
 *     [2][P][K|V][B][N_kv][S/(2P)][r]; a1 runs per local chunk and each half (every rank's early /
 *     late chunk) is all-gathered on a library-owned comm stream as soon as it exists -- half 0
 *     overlaps the late chunk's a1, half 1 overlaps the early chunk's attention (which needs keys
 *     of half 0 only); the compute stream waits on events.  Same result rows as layout 1 (bit for
 *     bit); not combinable with a token split or zdc_sp_decode (ZDC_ERR_UNSUPPORTED).
 * Per layer: a1 on local tokens -> all-gather of K'/V' over NCCL (the only data moved;
 * bytes = (P-1)/P * B S N_kv (r_k + r_v) * 2) -> a3 for local queries against all keys at
 * or before their global position -> a5 on local rows.  The result rows equal the
 * zdc_prefill rows of the same tokens.  Token split under SP (NEXT-2): a representative
 * layer's importance scores of the local rows are all-gathered (B S/P f32 per rank) and every rank
 * runs the same top-g selection over the whole sequence (identical classes and tau on every rank,
 * equal to zdc_prefill's); unimportant rows are truncated to r^u in the gather buffer (the
 * representative after classifying, the other layers of its group before their exchange).  zdc_comm_init takes a 128-byte ncclUniqueId.  Each rank keeps the
 * gathered compressed K'/V' of the whole sequence in its cache, in the gather layout
 * [P][K|V][B][N_kv][S/P][r]; zdc_decode on such a layer returns ZDC_ERR_UNSUPPORTED, and
 * zdc_cache_export exports only its classes and tau (k = v = NULL).  Chunks (S/P, or S/(2P) for zigzag) must be
 * multiples of 128 when P > 1.
 *   stats (optional, host): bytes exchanged per rank and the exchange time on the device.
 * ---------------------------------------------------------------------------------- */
zdc_status zdc_comm_unique_id(void* nccl_unique_id_out /*128 B, rank 0 creates, broadcast by the caller*/);
zdc_status zdc_comm_init(zdc_ctx* ctx, const void* nccl_unique_id, int32_t rank, int32_t world);
/* Test transport: instead of ncclAllGather, call fn(user, gather_buf, chunk_bytes, rank, world, stream)
 * where the caller must make gather_buf[q*chunk_bytes, (q+1)*chunk_bytes) equal rank q's slot for every q
 * before returning (used to run P ranks as P processes on ONE GPU in tests).  Replaces zdc_comm_init. */
typedef void (*zdc_exchange_fn)(void* user, void* gather_buf, int64_t chunk_bytes, int32_t rank, int32_t world,
                                void* stream);
zdc_status zdc_sp_set_exchange_hook(zdc_ctx* ctx, zdc_exchange_fn fn, void* user, int32_t rank, int32_t world);
typedef struct {
  int64_t bytes_sent, bytes_recv, bytes_recv_uncompressed;
  float exchange_ms, total_ms;
} zdc_sp_stats;
zdc_status zdc_sp_prefill(zdc_ctx* ctx, int32_t l0, int32_t l1, const uint16_t* x_local,
                          uint16_t* y_local, int32_t B, int32_t S_total, int32_t layout,
                          zdc_sp_stats* stats, void* stream);
/* (4b) Ulysses SP prefill, the paper's own dataflow (§5.3, Fig. bkg:fig:all2all:
 * "the four GPUs execute an all-to-all operation to gather tokens along the sequence dimension and
 * distribute heads ... The resulting tensors undergo a second all-to-all operation to gather heads
 * and sequence partitions"; "transmitting compressed Q, K, and V tensors in the first all-to-all
 * communication significantly reduces communication time").  Same arguments, layouts and result
 * rows as zdc_sp_prefill.  Per layer on rank p: a1 on the local tokens writes the compressed
 * Q'/K'/V' as P per-destination slabs (rank q gets the N_h/P heads h in [q N_h/P, (q+1) N_h/P) and
 * their N_kv/P KV groups) -> all-to-all #1 -> a3 (causal, full sequence) for rank p's heads ->
 * all-to-all #2 of O' back to the token owners -> a5 on the local rows.  Bytes received per rank
 * and layer: (P-1)/P * B S (N_h r_k + N_kv (r_k + r_v)) * 2 (#1) + (P-1)/P * B S N_h r_v * 2 (#2).
 * Requires N_kv % P == 0 (ZDC_ERR_SHAPE); S_total divisible by P (contiguous) or 2P (zigzag); no
 * 128-token chunk condition.  Each rank keeps the K'/V' cache of ITS KV groups for the whole
 * sequence ([B][N_kv/P][max_seq][r] in the layer's cache region); zdc_decode / zdc_cache_export on
 * such a layer return ZDC_ERR_UNSUPPORTED.  The NCCL transport is grouped ncclSend/ncclRecv on the
 * caller's stream (zdc_comm_init); the test transport below replaces it. */
zdc_status zdc_sp_prefill_ulysses(zdc_ctx* ctx, int32_t l0, int32_t l1, const uint16_t* x_local,
                                  uint16_t* y_local, int32_t B, int32_t S_total, int32_t layout,
                                  zdc_sp_stats* stats, void* stream);
/* Test transport of the all-to-all: fn(user, send, recv, chunk_bytes, rank, world, stream) must make
 * recv[q*chunk, (q+1)*chunk) equal rank q's send[rank*chunk, (rank+1)*chunk) for every q before
 * returning (device buffers; P processes on ONE GPU in tests).  Keeps an all-gather hook / comm of
 * the same rank and world. */
typedef void (*zdc_alltoall_fn)(void* user, const void* send, void* recv, int64_t chunk_bytes, int32_t rank,
                                int32_t world, void* stream);
zdc_status zdc_sp_set_alltoall_hook(zdc_ctx* ctx, zdc_alltoall_fn fn, void* user, int32_t rank, int32_t world);
/* (4c) NEXT-2: decode over the sequence-sharded compressed cache an all-gather zdc_sp_prefill left
 * (non-split layers).  One token per sequence on EVERY rank (same x on every rank, replicated a1/a5):
 * decode token j (j = 0, 1, ... after the prompt) is appended by rank j mod P only, into that rank's
 * tail of S/P rows per (sequence, KV head) after the gather buffer (needs max_seq >= S + S/P;
 * ZDC_ERR_CAPACITY past S/P decode tokens per rank).  Each rank attends over ITS keys only (its
 * prompt slot + its decode rows, the split-K kernel with two pools) -> {O'_p, LSE_p}; the ranks
 * all-gather these partials (B N_h (r_v + 1) f32 each) and every rank merges them by LSE (the
 * softmax of P:254-260 over the union of the key sets), then a5.  y rows equal zdc_decode's up to
 * the bf16 rounding of the partial O'_p.  Host-driven (no caller graph capture); B must equal the
 * SP prefill's batch. */
zdc_status zdc_sp_decode(zdc_ctx* ctx, int32_t l0, int32_t l1, const uint16_t* x, uint16_t* y, int32_t B,
                         void* stream);
/* Host helper: the global token positions rank `rank` holds (n = S_total / world). */
zdc_status zdc_sp_positions(int32_t S_total, int32_t world, int32_t rank, int32_t layout,
                            int32_t* positions);

/* ------------------------------------------------------------------------------------
 * Inspection (tests): export one layer's cache as zero-filled f32 at the important
 * widths, in position order: k [B][len][N_kv][r_qk_imp], v [B][len][N_kv][r_vl_imp],
 * is_important u8 [B][len] (all 1 without a split), tau f32 [B] (+inf without a split).
 * Host output buffers; synchronises `stream`.  Any pointer may be NULL to skip it.
 * ---------------------------------------------------------------------------------- */
zdc_status zdc_cache_export(const zdc_ctx* ctx, int32_t layer, float* k, float* v,
                            uint8_t* is_important, float* tau, void* stream);
zdc_status zdc_cache_length(const zdc_ctx* ctx, int32_t layer, int32_t* len);
/* The cache lengths live on the device (decode kernels advance them, so one decode graph serves
 * every position); the host keeps a copy for argument checks and the inspection calls, advanced by
 * each zdc_prefill / zdc_decode call.  A caller that replays zdc_decode calls inside its OWN captured
 * CUDA graph calls zdc_cache_sync afterwards: it copies the device lengths back (synchronises
 * `stream`).  ZDC_ERR_STATE if the ctx is not bound.
 * Capacity: every replayed decode step uses one cache row; only the host-side check at capture time
 * sees max_seq, so the caller bounds its replay count.  A step that finds the cache full does not
 * write outside the layer's rows: it rewrites the last row, the length stays at max_seq and a
 * device overflow flag is set; zdc_cache_sync then returns ZDC_ERR_CAPACITY (the outputs of the
 * overflowing steps are invalid) until zdc_cache_reset clears it. */
zdc_status zdc_cache_sync(zdc_ctx* ctx, void* stream);
/* Importance scores (reading c9: log of sum_h sum_{k<=t} exp(s_k^h), f32 as computed on the GPU)
 * of every cached token of a representative layer of a split group: scores [B][len], host. */
zdc_status zdc_scores_export(const zdc_ctx* ctx, int32_t layer, float* scores, void* stream);
zdc_status zdc_cache_reset(zdc_ctx* ctx, void* stream);

/* Device LSE of the last prefill/decode call of a layer: f32 [B][N_h][T] (T = S for a
 * prefill, 1 for a decode step), log of the Eq. 3 denominator of each query row. */
zdc_status zdc_last_lse(const zdc_ctx* ctx, int32_t layer, float* lse_host, void* stream);

/* ------------------------------------------------------------------------------------
 * Kernel-level entry (tests and roofline measurements): the tcgen05 projection GEMM of
 * a1/a5, D[M][N] = A[M][K] * B[N][K]^T, bf16 in, f32 accumulate, bf16 out (RNE).
 * a, b, d: device; K % 64 == 0; rows 16-byte aligned. */
zdc_status zdc_gemm_bf16(const uint16_t* a, const uint16_t* b, uint16_t* d,
                         int32_t M, int32_t N, int32_t K, void* stream);
/* Kernel-level entries of a3 (tests and roofline measurements), Eqs. 2-3 with the
 * given scale (1/sqrt(d_h), reading c2), bf16 in / out, f32 softmax and accumulation:
 * prefill (causal): q, o [B*S][N_h*r] (head h at cols h*r), k, v [B][N_kv][S][r], lse [B][N_h][S]
 *   (may be NULL); r % 16 == 0, r <= 128.
 * decode (the query attends to positions [0, len)): q, o [B][N_h*r], k, v [B][N_kv][S_cap][r],
 *   lse [B][N_h] (may be NULL); workspace: zdc_decode_attention_workspace(...) bytes, zeroed by the
 *   caller once (the kernel leaves its merge counters at zero). */
zdc_status zdc_prefill_attention_bf16(const uint16_t* q, const uint16_t* k, const uint16_t* v, uint16_t* o,
                                      float* lse, int32_t B, int32_t S, int32_t Nh, int32_t Nkv, int32_t r,
                                      float scale, void* stream);
int64_t zdc_decode_attention_workspace(int32_t B, int32_t Nh, int32_t Nkv, int32_t r);
zdc_status zdc_decode_attention_bf16(const uint16_t* q, const uint16_t* k, const uint16_t* v, uint16_t* o,
                                     float* lse, int32_t B, int32_t Nh, int32_t Nkv, int32_t r, int32_t len,
                                     int32_t S_cap, float scale, void* workspace, void* stream);
/* Kernel-level entry of the decode projection (a1 / a5 for B <= 8 rows, HBM-bound):
 * y[b][n] = sum_k x[b][k] w[n][k]; w [N][K], x [B][K], y [B][N] bf16 (f32 accumulate). */
zdc_status zdc_gemv_bf16(const uint16_t* w, const uint16_t* x, uint16_t* y, int32_t B, int32_t N, int32_t K,
                         void* stream);

/* Decode kernel selection for B <= 8 uniform-rank layers (process-wide, takes effect at the next
 * zdc_decode; cached decode CUDA graphs keep the kernels they captured, so call it before the
 * first decode of a context): 0 = automatic (default: the persistent fused layer-step where
 * supported, else separate kernels), 1 = the persistent fused layer-step (decode_fused.cuh),
 * 2 = the cluster layer-step (decode_cluster.cuh: one cluster of CTAs per KV group, tcgen05
 * projections, DSMEM exchanges, no grid barrier; needs r in {16, 32, 64, 128}, G r <= 256 and
 * d % 64 == 0; falls back to 1 where unsupported), 3 = separate kernels (GEMV / GEMM, split-K
 * attention, GEMV).  Returns the previous mode; -1 for an invalid mode.
 * Mode 2 must be selected before zdc_ctx_create: the cluster kernel streams decode copies of the
 * weights (pre-tiled W_QKV, group-major W_O) that zdc_ctx_sizes then counts and zdc_load_folded
 * fills.  The initial mode is 0 (release builds read no environment variables). */
int zdc_decode_mode(int mode);

/* Number of kernels the last prefill / decode call enqueued (for bench.py's gpu_launches). */
int64_t zdc_kernel_launch_count(void);

/* Per-kernel-class device timing (bench.py's roofline): zdc_profile(1) brackets every launch
 * with CUDA events on its stream (zdc_decode then runs eagerly instead of replaying its CUDA
 * graph); zdc_profile_read synchronises, writes per class the summed milliseconds and launch
 * counts since the previous read, clears them, and returns the number of classes:
 * 0 a1 prefill GEMM, 1 a3 prefill attention, 2 a5 prefill GEMM, 3 a1 decode GEMV,
 * 4 a3 decode attention (partial), 5 a3 decode combine, 6 a5 decode GEMV, 7 other,
 * 8 fused decode layer-step (a1+a2+a3+a5 in one kernel, B <= 8 uniform-rank layers). */
void zdc_profile(int enable);
int zdc_profile_read(float* ms, int64_t* count, int n);
/* Diagnostics (diagnostic builds only, -DZDC_DEBUG_KNOBS, csrc/knobs.h; release builds return 0):
 * with ZDC_FUSED_TRACE set in the environment, the fused decode kernel records
 * per-CTA %globaltimer stamps (ns) of its last launch, [CTA][16]: 0 start, 1 input staged,
 * 2 phase-1 done, 3 after grid barrier 1, 4 phase-2 done, 5 after grid barrier 2, 6 merge done,
 * 7 end, 8/9/10 producer finished issuing phase 1/2/3.  Copies n values (synchronising the
 * device); returns the count copied, 0 when tracing is off, -1 on a CUDA error. */
int zdc_trace_read(unsigned long long* out, int n);

#ifdef __cplusplus
}
#endif
#endif /* ZDC_H */
