// api.cpp — the C ABI of include/zdc.h: context, weight loading, and the per-layer
// orchestration of the hot path (a1 projection -> a2 append -> a3 attention -> a4 selection
// -> a5 output projection).  Host code only; every step of the path runs in the kernels of
// gemm.cu / attn_prefill.cu / decode.cu / select.cu.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "api_util.h"
#include "ctx.h"
#include "kernels.h"
#include "zdc.h"

namespace zdc {

static thread_local std::string t_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_err = buf;
}

zdc_status fail(zdc_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_err = buf;
  return s;
}

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
static inline int pad16(int r) { return (r + 15) / 16 * 16; }

// bf16 round-to-nearest-even of an f64 through f32 (the same two steps the GPU epilogues take
// from their f32 accumulators).
static inline uint16_t f64_to_bf16(double v) {
  float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return static_cast<uint16_t>(u >> 16);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

static zdc_status check_sticky() {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(ZDC_ERR_CUDA, "asynchronous CUDA error from an earlier call: %s", cudaGetErrorString(e));
  }
  return ZDC_OK;
}

void graphs_destroy(zdc_ctx* c) {
  for (auto& kv : c->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  c->graphs.clear();
}

}  // namespace zdc

using namespace zdc;

extern "C" {

const char* zdc_last_error(void) { return t_err.c_str(); }
const char* zdc_version(void) { return "zdc-b200 0.1 (sm_100a tcgen05)"; }
int64_t zdc_kernel_launch_count(void) { return g_launches; }



// ------------------------------------------------------------------ context
static int g_decode_mode = knob("ZDC_DECODE_MODE", 0);
int zdc_decode_mode(int mode) {
  if (mode < 0 || mode > 3) return -1;
  const int old = g_decode_mode;
  g_decode_mode = mode;
  return old;
}

zdc_status zdc_ctx_create(const zdc_dims* dims, const zdc_plan* plan, int32_t max_batch, int32_t max_seq,
                          zdc_ctx** out) {
  if (!dims || !plan || !out) return fail(ZDC_ERR_INVALID_ARG, "zdc_ctx_create: null argument");
  *out = nullptr;
  const zdc_dims& d = *dims;
  if (d.n_layers <= 0 || d.d_model <= 0 || d.n_heads <= 0 || d.n_kv_heads <= 0 || d.d_head <= 0)
    return fail(ZDC_ERR_SHAPE, "zdc_ctx_create: non-positive dims (L=%d d=%d Nh=%d Nkv=%d dh=%d)", d.n_layers,
                d.d_model, d.n_heads, d.n_kv_heads, d.d_head);
  if (d.n_heads % d.n_kv_heads != 0)
    return fail(ZDC_ERR_SHAPE, "zdc_ctx_create: n_heads %d not a multiple of n_kv_heads %d", d.n_heads,
                d.n_kv_heads);
  if (d.d_model % 64 != 0) return fail(ZDC_ERR_UNSUPPORTED, "zdc_ctx_create: d_model %d %% 64 != 0", d.d_model);
  if (d.d_head > 128) return fail(ZDC_ERR_UNSUPPORTED, "zdc_ctx_create: d_head %d > 128", d.d_head);
  const int G = d.n_heads / d.n_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return fail(ZDC_ERR_UNSUPPORTED, "zdc_ctx_create: group size %d not in {1,2,4,8}", G);
  if (max_batch <= 0 || max_seq <= 0)
    return fail(ZDC_ERR_SHAPE, "zdc_ctx_create: max_batch %d / max_seq %d", max_batch, max_seq);
  if (!plan->r_qk_imp || !plan->r_qk_unimp || !plan->r_vl_imp || !plan->r_vl_unimp || !plan->g_bp ||
      !plan->group_rep)
    return fail(ZDC_ERR_INVALID_ARG, "zdc_ctx_create: null plan array");
  if (plan->importance_mode != 0 && plan->importance_mode != 1)
    return fail(ZDC_ERR_INVALID_ARG, "zdc_ctx_create: importance_mode %d", plan->importance_mode);
  if (plan->kv_fp8 != 0 && plan->kv_fp8 != 1)
    return fail(ZDC_ERR_INVALID_ARG, "zdc_ctx_create: kv_fp8 %d", plan->kv_fp8);

  zdc_ctx* c = new zdc_ctx();
  c->dims = d;
  c->G = G;
  c->max_batch = max_batch;
  c->max_seq = max_seq;
  c->importance_mode = plan->importance_mode;
  c->kv_fp8 = plan->kv_fp8;
  c->layers.resize(d.n_layers);
  c->len.assign(d.n_layers, 0);
  c->sp_layer.assign(d.n_layers, 0);
  c->sp_prompt.assign(d.n_layers, 0);
  int64_t woff = 0, coff = 0;
  int max_nq = 0, max_ko = 0, max_rv = 0, max_split_w = 0, max_nqkv = 0;
  bool any_split = false;
  for (int l = 0; l < d.n_layers; ++l) {
    LayerInfo& L = c->layers[l];
    L.rk = plan->r_qk_imp[l];
    L.rku = plan->r_qk_unimp[l];
    L.rv = plan->r_vl_imp[l];
    L.rvu = plan->r_vl_unimp[l];
    L.g_bp = plan->g_bp[l];
    L.rep = plan->group_rep[l];
    // r_unimp = 0 (both pairs) in a split group = eviction of the unimportant tokens (H2O-ZDC, reading c26)
    const bool evict0 = L.rku == 0 && L.rvu == 0 && plan->g_bp[l] < 10000;
    if ((L.rku < 1 && !evict0) || L.rku > L.rk || L.rk < 1 || L.rk > d.d_head || (L.rvu < 1 && !evict0) ||
        L.rvu > L.rv || L.rv < 1 || L.rv > d.d_head) {
      delete c;
      return fail(ZDC_ERR_SHAPE, "layer %d: ranks must satisfy 1 <= r_unimp <= r_imp <= d_head, or r_unimp = 0 in a "
                  "split group (eviction) (qk %d/%d vl %d/%d)", l, L.rk, L.rku, L.rv, L.rvu);
    }
    L.evict = evict0;
    if (L.g_bp < 0 || L.g_bp > 10000 || L.rep < 0 || L.rep > l || plan->group_rep[L.rep] != L.rep) {
      delete c;
      return fail(ZDC_ERR_INVALID_ARG, "layer %d: g_bp %d / group_rep %d invalid", l, L.g_bp, L.rep);
    }
    L.split = L.g_bp < 10000;
    if (L.split) {
      const int r = L.rep;
      if (plan->g_bp[r] != L.g_bp || plan->r_qk_imp[r] != L.rk || plan->r_qk_unimp[r] != L.rku ||
          plan->r_vl_imp[r] != L.rv || plan->r_vl_unimp[r] != L.rvu) {
        delete c;
        return fail(ZDC_ERR_INVALID_ARG, "layer %d: g and ranks must equal those of its representative %d", l, r);
      }
      any_split = true;
    }
    L.rk_p = pad16(L.rk);
    L.rv_p = pad16(L.rv);
    L.rku_p = pad16(L.rku);
    L.rvu_p = pad16(L.rvu);
    if (L.rk_p != L.rv_p || L.rku_p != L.rvu_p) {
      delete c;
      return fail(ZDC_ERR_UNSUPPORTED, "layer %d: padded ranks must satisfy r_qk == r_vl (imp %d/%d, unimp %d/%d)", l,
                  L.rk_p, L.rv_p, L.rku_p, L.rvu_p);
    }
    L.nq = d.n_heads * L.rk_p;
    L.nk = d.n_kv_heads * L.rk_p;
    L.nv = d.n_kv_heads * L.rv_p;
    L.n_qkv = L.nq + L.nk + L.nv;
    L.ko_p = static_cast<int>(align_up(static_cast<int64_t>(d.n_heads) * L.rv_p, 64));
    L.w_qkv = woff;
    woff = align_up(woff + static_cast<int64_t>(L.n_qkv) * d.d_model * 2, 256);
    L.w_o = woff;
    woff = align_up(woff + static_cast<int64_t>(d.d_model) * L.ko_p * 2, 256);
    if (g_decode_mode == 2 && !L.split && decode_cluster_layer_ok(L.rk_p, d.n_heads / d.n_kv_heads)) {
      // the group-major copy of W_O that the cluster decode kernel streams in contiguous tiles
      L.w_od = woff;
      woff = align_up(woff + static_cast<int64_t>(d.n_heads) * L.rv_p * d.d_model * 2, 256);
      if (d.d_model % 64 == 0) {  // and of W_QKV, pre-tiled and pre-swizzled (contiguous per CTA)
        L.w_qd = woff;
        woff = align_up(woff + static_cast<int64_t>(L.n_qkv) * d.d_model * 2, 256);
      }
    }
    const int64_t kv_rows = static_cast<int64_t>(max_batch) * d.n_kv_heads * max_seq;
    if (c->kv_fp8) {
      const bool w_ok = L.rk_p == 32 || L.rk_p == 64 || L.rk_p == 96 || L.rk_p == 128;
      if (L.split || !w_ok || L.rk_p != L.rv_p) {
        delete c;
        return fail(ZDC_ERR_UNSUPPORTED, "zdc_ctx_create: kv_fp8 needs uniform-rank layers with padded ranks in "
                    "{32, 64, 96, 128} (layer %d: split %d, rank %d)", l, L.split ? 1 : 0, L.rk_p);
      }
    }
    // bf16 rows of r, or FP8 rows of r codes + f32 scale + 12 pad bytes (NEXT-4)
    const int64_t krow = c->kv_fp8 ? L.rk_p + 16 : L.rk_p * 2, vrow = c->kv_fp8 ? L.rv_p + 16 : L.rv_p * 2;
    L.k_off = coff;
    coff = align_up(coff + kv_rows * krow, 256);
    L.v_off = coff;
    coff = align_up(coff + kv_rows * vrow, 256);
    if (c->kv_fp8 && L.rk_p > max_split_w) max_split_w = L.rk_p;
    if (L.split) {
      L.ku_off = coff;
      coff = align_up(coff + kv_rows * L.rku_p * 2, 256);
      L.vu_off = coff;
      coff = align_up(coff + kv_rows * L.rvu_p * 2, 256);
      L.posi_off = coff;
      coff = align_up(coff + static_cast<int64_t>(max_batch) * max_seq * 4, 256);
      L.posu_off = coff;
      coff = align_up(coff + static_cast<int64_t>(max_batch) * max_seq * 4, 256);
      L.ni_off = coff;
      coff = align_up(coff + static_cast<int64_t>(max_batch) * 4, 256);
      L.nu_off = coff;
      coff = align_up(coff + static_cast<int64_t>(max_batch) * 4, 256);
      if (L.rk_p > max_split_w) max_split_w = L.rk_p;
    }
    if (L.split && L.rep == l) {
      L.cls_off = coff;
      coff = align_up(coff + static_cast<int64_t>(max_batch) * max_seq, 256);
      L.tau_off = coff;
      coff = align_up(coff + static_cast<int64_t>(max_batch) * 4, 256);
      L.score_off = coff;
      coff = align_up(coff + static_cast<int64_t>(max_batch) * max_seq * 4, 256);
    }
    if (L.nq > max_nq) max_nq = L.nq;
    if (L.ko_p > max_ko) max_ko = L.ko_p;
    if (L.n_qkv > max_nqkv) max_nqkv = L.n_qkv;
    if (L.rv_p > max_rv) max_rv = L.rv_p;
  }
  c->len_dev_off = coff;  // [n_layers] device lengths, the decode overflow flag, the NaN-score flag
  coff = align_up(coff + static_cast<int64_t>(d.n_layers + 2) * 4, 256);
  c->weight_bytes = woff;
  c->cache_bytes = coff;
  const int64_t rows = static_cast<int64_t>(max_batch) * max_seq;
  int64_t s = 0;
  c->s_q = s;
  s = align_up(s + rows * max_nq * 2, 256);
  c->s_o = s;
  s = align_up(s + rows * max_ko * 2, 256);
  c->s_lse = s;
  s = align_up(s + rows * d.n_heads * 4, 256);
  c->s_part = s;
  s = align_up(s + static_cast<int64_t>(max_batch) * d.n_heads * 128 * (max_rv + 2) * 4, 256);
  c->s_cnt = s;  // decode-attention merge counters [max_batch][N_kv], kept at zero between launches
  s = align_up(s + static_cast<int64_t>(max_batch) * d.n_kv_heads * 4, 256);
  c->s_gbar = s;  // fused decode grid barrier, kept self-resetting between launches
  s = align_up(s + 64, 256);
  c->s_ltab = s;  // fused decode layer table (DecLayer per layer), written at bind
  s = align_up(s + static_cast<int64_t>(d.n_layers) * static_cast<int64_t>(sizeof(DecLayer)), 256);
  if (max_batch > 8) {  // split-K decode GEMMs (B > 8): f32 workspace [min(B,128)][max N] + tile counters
    c->s_gsk = s;
    s = align_up(s + static_cast<int64_t>(std::min(max_batch, 128)) * std::max(max_nqkv, d.d_model) * 4 + 1024 * 4,
                 256);
  }
  // Ulysses SP (zdc_sp_prefill_ulysses): all-to-all send and receive slabs, each at most
  // (rows / 2) x n_qkv bf16 (P >= 2 ranks hold at most half of the rows each)
  c->s_sp = s;
  s = align_up(s + rows * max_nqkv * 2, 256);
  c->s_ybuf = s;  // cluster decode: y accumulator [8][d] f32 then 16 arrival counters, zero between launches
  s = align_up(s + static_cast<int64_t>(8) * d.d_model * 4 + 16 * 4, 256);
  if (any_split || c->kv_fp8) {  // staged K'/V' (split: before packing; FP8: before quantizing), indices, new rows
    const int64_t kv_rows = static_cast<int64_t>(max_batch) * d.n_kv_heads * max_seq;
    c->s_ks = s;
    s = align_up(s + kv_rows * max_split_w * 2, 256);
    c->s_vs = s;
    s = align_up(s + kv_rows * max_split_w * 2, 256);
    c->s_didx = s;
    s = align_up(s + rows * 4, 256);
    c->s_new = s;
    s = align_up(s + static_cast<int64_t>(max_batch) * d.n_kv_heads * max_split_w * 2 * 2, 256);
  }
  c->ldq = max_nq;
  c->max_nqkv = max_nqkv;
  c->ldo = max_ko;
  c->scratch_bytes = s;
  *out = c;
  return ZDC_OK;
}

zdc_status zdc_ctx_sizes(const zdc_ctx* c, int64_t* wb, int64_t* cb, int64_t* sb) {
  if (!c) return fail(ZDC_ERR_INVALID_ARG, "zdc_ctx_sizes: null ctx");
  if (wb) *wb = c->weight_bytes;
  if (cb) *cb = c->cache_bytes;
  if (sb) *sb = c->scratch_bytes;
  return ZDC_OK;
}

zdc_status zdc_ctx_bind(zdc_ctx* c, void* w, void* cache, void* scratch) {
  if (!c || !w || !cache || !scratch) return fail(ZDC_ERR_INVALID_ARG, "zdc_ctx_bind: null argument");
  if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(cache) | reinterpret_cast<uintptr_t>(scratch)) &
      255)
    return fail(ZDC_ERR_INVALID_ARG, "zdc_ctx_bind: buffers must be 256-byte aligned");
  graphs_destroy(c);
  c->w = static_cast<uint8_t*>(w);
  c->cache = static_cast<uint8_t*>(cache);
  c->scratch = static_cast<uint8_t*>(scratch);
  ZDC_CUDA_TRY(cudaMemset(c->cache, 0, c->cache_bytes));
  ZDC_CUDA_TRY(cudaMemset(c->scratch, 0, c->scratch_bytes));
  ZDC_CUDA_TRY(cudaMemset(c->w, 0, c->weight_bytes));
  fused_trace_buffer();  // allocated here (if ZDC_FUSED_TRACE is set), never inside a graph capture
  {
    std::vector<DecLayer> tab(c->dims.n_layers);
    for (int l = 0; l < c->dims.n_layers; ++l) {
      const LayerInfo& L = c->layers[l];
      tab[l].wqkv = reinterpret_cast<const uint16_t*>(c->w + L.w_qkv);
      tab[l].wo = reinterpret_cast<const uint16_t*>(c->w + L.w_o);
      tab[l].kc = reinterpret_cast<uint16_t*>(c->cache + L.k_off);
      tab[l].vc = reinterpret_cast<uint16_t*>(c->cache + L.v_off);
      tab[l].len_ptr = c->len_dev() + l;
    }
    ZDC_CUDA_TRY(cudaMemcpy(c->scratch + c->s_ltab, tab.data(), tab.size() * sizeof(DecLayer), cudaMemcpyHostToDevice));
  }
  c->len.assign(c->dims.n_layers, 0);
  c->sp_layer.assign(c->dims.n_layers, 0);
  c->sp_prompt.assign(c->dims.n_layers, 0);
  c->batch = 0;
  return ZDC_OK;
}

void zdc_ctx_destroy(zdc_ctx* c) {
  if (!c) return;
  comm_destroy(c);
  graphs_destroy(c);
  delete c;
}

// ------------------------------------------------------------------ weights
zdc_status zdc_load_folded(zdc_ctx* c, int32_t layer, const double* wq, const double* wk, const double* wv,
                           const double* wo, void* stream) {
  if (!c || !wq || !wk || !wv || !wo) return fail(ZDC_ERR_INVALID_ARG, "zdc_load_folded: null argument");
  if (!c->w) return fail(ZDC_ERR_STATE, "zdc_load_folded: ctx not bound");
  if (layer < 0 || layer >= c->dims.n_layers) return fail(ZDC_ERR_SHAPE, "zdc_load_folded: layer %d", layer);
  const LayerInfo& L = c->layers[layer];
  const int d = c->dims.d_model, Nh = c->dims.n_heads, Nkv = c->dims.n_kv_heads, dh = c->dims.d_head;
  std::vector<uint16_t> qkv(static_cast<size_t>(L.n_qkv) * d, 0), o(static_cast<size_t>(d) * L.ko_p, 0);
  auto finite = [](double v) { return std::isfinite(v); };
  for (int n = 0; n < L.n_qkv; ++n) {
    const double* src;
    int64_t ld, col;
    int c_in;
    if (n < L.nq) {
      c_in = n % L.rk_p;
      if (c_in >= L.rk) continue;
      src = wq, ld = static_cast<int64_t>(Nh) * dh, col = (n / L.rk_p) * dh + c_in;
    } else if (n < L.nq + L.nk) {
      c_in = (n - L.nq) % L.rk_p;
      if (c_in >= L.rk) continue;
      src = wk, ld = static_cast<int64_t>(Nkv) * dh, col = ((n - L.nq) / L.rk_p) * dh + c_in;
    } else {
      c_in = (n - L.nq - L.nk) % L.rv_p;
      if (c_in >= L.rv) continue;
      src = wv, ld = static_cast<int64_t>(Nkv) * dh, col = ((n - L.nq - L.nk) / L.rv_p) * dh + c_in;
    }
    for (int k = 0; k < d; ++k) {
      const double v = src[k * ld + col];
      if (!finite(v)) return fail(ZDC_ERR_INVALID_ARG, "zdc_load_folded: non-finite weight");
      qkv[static_cast<size_t>(n) * d + k] = f64_to_bf16(v);
    }
  }
  for (int h = 0; h < Nh; ++h)
    for (int cc = 0; cc < L.rv; ++cc) {
      const double* row = wo + static_cast<int64_t>(h * dh + cc) * d;
      for (int j = 0; j < d; ++j) {
        if (!finite(row[j])) return fail(ZDC_ERR_INVALID_ARG, "zdc_load_folded: non-finite weight");
        o[static_cast<size_t>(j) * L.ko_p + h * L.rv_p + cc] = f64_to_bf16(row[j]);
      }
    }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ZDC_CUDA_TRY(cudaMemcpyAsync(c->w + L.w_qkv, qkv.data(), qkv.size() * 2, cudaMemcpyHostToDevice, st));
  ZDC_CUDA_TRY(cudaMemcpyAsync(c->w + L.w_o, o.data(), o.size() * 2, cudaMemcpyHostToDevice, st));
  if (L.w_od >= 0)
    ZDC_CUDA_TRY(launch_pack_wo_decode(reinterpret_cast<const uint16_t*>(c->w + L.w_o),
                                       reinterpret_cast<uint16_t*>(c->w + L.w_od), c->dims.d_model, L.ko_p,
                                       c->dims.n_kv_heads, c->G * L.rv_p, st));
  if (L.w_qd >= 0)
    ZDC_CUDA_TRY(launch_pack_qkv_decode(reinterpret_cast<const uint16_t*>(c->w + L.w_qkv),
                                        reinterpret_cast<uint16_t*>(c->w + L.w_qd), c->dims.d_model, L.nq, L.nk,
                                        c->dims.n_kv_heads, c->G, L.rk_p, st));
  ZDC_CUDA_TRY(cudaStreamSynchronize(st));
  return ZDC_OK;
}

zdc_status zdc_load_folded_device(zdc_ctx* c, int32_t layer, const uint16_t* wq, const uint16_t* wk,
                                  const uint16_t* wv, const uint16_t* wo, void* stream) {
  if (!c || !wq || !wk || !wv || !wo) return fail(ZDC_ERR_INVALID_ARG, "zdc_load_folded_device: null argument");
  if (!c->w) return fail(ZDC_ERR_STATE, "zdc_load_folded_device: ctx not bound");
  if (layer < 0 || layer >= c->dims.n_layers) return fail(ZDC_ERR_SHAPE, "zdc_load_folded_device: layer %d", layer);
  const LayerInfo& L = c->layers[layer];
  ZDC_CUDA_TRY(launch_pack_weights_bf16(wq, wk, wv, wo, reinterpret_cast<uint16_t*>(c->w + L.w_qkv),
                                        reinterpret_cast<uint16_t*>(c->w + L.w_o), c->dims.d_model, c->dims.n_heads,
                                        c->dims.n_kv_heads, c->dims.d_head, L.rk, L.rv, L.rk_p, L.rv_p, L.ko_p,
                                        static_cast<cudaStream_t>(stream)));
  if (L.w_od >= 0)
    ZDC_CUDA_TRY(launch_pack_wo_decode(reinterpret_cast<const uint16_t*>(c->w + L.w_o),
                                       reinterpret_cast<uint16_t*>(c->w + L.w_od), c->dims.d_model, L.ko_p,
                                       c->dims.n_kv_heads, c->G * L.rv_p, static_cast<cudaStream_t>(stream)));
  if (L.w_qd >= 0)
    ZDC_CUDA_TRY(launch_pack_qkv_decode(reinterpret_cast<const uint16_t*>(c->w + L.w_qkv),
                                        reinterpret_cast<uint16_t*>(c->w + L.w_qd), c->dims.d_model, L.nq, L.nk,
                                        c->dims.n_kv_heads, c->G, L.rk_p, static_cast<cudaStream_t>(stream)));
  return ZDC_OK;
}

// ------------------------------------------------------------------ hot path
static zdc_status check_run(zdc_ctx* c, int l0, int l1, const void* x, const void* y, const char* who) {
  if (!c) return fail(ZDC_ERR_INVALID_ARG, "%s: null ctx", who);
  if (!c->w) return fail(ZDC_ERR_STATE, "%s: ctx not bound", who);
  if (!x || !y) return fail(ZDC_ERR_INVALID_ARG, "%s: null x / y", who);
  if (x == y) return fail(ZDC_ERR_INVALID_ARG, "%s: x and y alias", who);
  if (l0 < 0 || l1 > c->dims.n_layers || l0 >= l1)
    return fail(ZDC_ERR_SHAPE, "%s: layer range [%d, %d) outside [0, %d)", who, l0, l1, c->dims.n_layers);
  return check_sticky();
}

static QkvDest qkv_dest(zdc_ctx* c, const LayerInfo& L, int S, int pos0, const int* posmap) {
  QkvDest q;
  q.q = reinterpret_cast<uint16_t*>(c->scratch + c->s_q);
  q.ldq = L.nq;
  q.nq = L.nq;
  q.nk = L.nk;
  q.k = reinterpret_cast<uint16_t*>(c->cache + L.k_off);
  q.v = reinterpret_cast<uint16_t*>(c->cache + L.v_off);
  q.rk = L.rk_p;
  q.rv = L.rv_p;
  q.S = S;
  q.kg = static_cast<int64_t>(c->max_seq) * L.rk_p;
  q.kb = q.kg * c->dims.n_kv_heads;
  q.vg = static_cast<int64_t>(c->max_seq) * L.rv_p;
  q.vb = q.vg * c->dims.n_kv_heads;
  q.pos0 = pos0;
  q.posmap = posmap;
  return q;
}

zdc_status zdc_prefill(zdc_ctx* c, int32_t l0, int32_t l1, const uint16_t* x, uint16_t* y, int32_t B, int32_t S,
                       float* importance, void* stream) {
  zdc_status st = check_run(c, l0, l1, x, y, "zdc_prefill");
  if (st != ZDC_OK) return st;
  if (B <= 0 || S <= 0) return fail(ZDC_ERR_SHAPE, "zdc_prefill: B=%d S=%d", B, S);
  {
    const long long nb = 2LL * B * S * c->dims.d_model;
    if (ranges_overlap(x, nb, y, nb)) return fail(ZDC_ERR_INVALID_ARG, "zdc_prefill: x and y overlap");
  }
  if (B > c->max_batch || S > c->max_seq)
    return fail(ZDC_ERR_CAPACITY, "zdc_prefill: B=%d S=%d exceeds max_batch=%d max_seq=%d", B, S, c->max_batch,
                c->max_seq);
  for (int l = l0; l < l1; ++l)
    if (c->len[l] != 0) return fail(ZDC_ERR_STATE, "zdc_prefill: layer %d cache is not empty (len %d)", l, c->len[l]);
  if (c->batch != 0 && c->batch != B) {
    bool all_empty = true;
    for (int l = 0; l < c->dims.n_layers; ++l) all_empty &= c->len[l] == 0;
    if (!all_empty) return fail(ZDC_ERR_SHAPE, "zdc_prefill: batch %d differs from the cache batch %d", B, c->batch);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  g_launches = 0;
  const int d = c->dims.d_model, Nh = c->dims.n_heads, Nkv = c->dims.n_kv_heads;
  const int M = B * S;
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& L = c->layers[l];
    const uint16_t* xin = l == l0 ? x : y;
    const bool is_rep = L.rep == l;
    if (L.split && !is_rep && c->len[L.rep] != S)
      return fail(ZDC_ERR_STATE, "zdc_prefill: layer %d needs its representative layer %d prefilled first", l, L.rep);
    // a1 + a2: [Q'|K'|V'] = x W_QKV^R; K'/V' written into the cache at positions [0, S) (uniform
    // layers) or staged for the class-aware packing (token split)
    Epilogue e1;
    e1.mode = 1;
    e1.qkv = qkv_dest(c, L, S, 0, nullptr);
    uint16_t* ks = reinterpret_cast<uint16_t*>(c->scratch + c->s_ks);
    uint16_t* vs = reinterpret_cast<uint16_t*>(c->scratch + c->s_vs);
    if (L.split || c->kv_fp8) {  // staged: class-aware packing (split) / quantization (FP8, NEXT-4)
      e1.qkv.k = ks;
      e1.qkv.v = vs;
    }
    e1.pdl = 1;  // PDL: the weight tiles of the first stages stream before the dependency wait
    g_prof_class = kProfGemmQkv;
    ZDC_CUDA_TRY(launch_gemm(xin, d, reinterpret_cast<const uint16_t*>(c->w + L.w_qkv), d, M, L.n_qkv, d, e1, s));
    const LayerInfo& R = c->layers[L.rep];
    uint8_t* rep_cls = reinterpret_cast<uint8_t*>(c->cache + R.cls_off);
    g_prof_class = kProfOther;
    if (L.split && !is_rep && !L.evict) {
      // non-representative layer: the group's classes are known; unimportant key/value rows lose
      // dims >= r^u BEFORE attention (P:774-776 DEL; reading c13).  (Eviction: the prompt
      // attends in full; the pack below keeps the important rows only, reading c26.)
      ZDC_CUDA_TRY(launch_truncate(ks, L.rk_p, L.rku, B, Nkv, S, c->max_seq, rep_cls, c->max_seq, s));
      ZDC_CUDA_TRY(launch_truncate(vs, L.rv_p, L.rvu, B, Nkv, S, c->max_seq, rep_cls, c->max_seq, s));
    }
    // a3: causal attention at head dim r, O' and LSE
    PrefillAttnArgs a;
    a.q = reinterpret_cast<const uint16_t*>(c->scratch + c->s_q);
    a.ldq = L.nq;
    a.k = L.split || c->kv_fp8 ? ks : reinterpret_cast<const uint16_t*>(c->cache + L.k_off);
    a.v = L.split || c->kv_fp8 ? vs : reinterpret_cast<const uint16_t*>(c->cache + L.v_off);
    a.S_cap = c->max_seq;
    a.o = reinterpret_cast<uint16_t*>(c->scratch + c->s_o);
    a.ldo = L.ko_p;
    a.lse = reinterpret_cast<float*>(c->scratch + c->s_lse);
    a.B = B;
    a.S = S;
    a.Nh = Nh;
    a.Nkv = Nkv;
    a.rk = L.rk_p;
    a.rv = L.rv_p;
    a.scale = 1.0f / std::sqrt(static_cast<float>(c->dims.d_head));
    a.q_pos0 = 0;
    a.q_row0 = 0;
    a.n_q = S;
    ZDC_CUDA_TRY(launch_prefill_attention(a, s));
    if (c->kv_fp8) {  // NEXT-4: the prompt attended at full precision; the cache keeps FP8 rows
      g_prof_class = kProfOther;
      ZDC_CUDA_TRY(launch_quantize_kv(ks, c->max_seq, c->cache + L.k_off, c->max_seq, B * Nkv, 0, S, L.rk_p, nullptr, s));
      ZDC_CUDA_TRY(launch_quantize_kv(vs, c->max_seq, c->cache + L.v_off, c->max_seq, B * Nkv, 0, S, L.rv_p, nullptr, s));
    }
    if (L.split) {
      g_prof_class = kProfOther;
      if (is_rep) {
        // a4: importance from the reused softmax denominators, then the top-g selection
        float* scores = reinterpret_cast<float*>(c->cache + L.score_off);
        ZDC_CUDA_TRY(launch_importance(a.lse, S, Nh, B, 0, c->importance_mode, scores, c->max_seq,
                                       importance ? importance + static_cast<int64_t>(l) * B * c->max_seq : nullptr,
                                       c->max_seq, nullptr, s));
        ZDC_CUDA_TRY(launch_select(scores, c->max_seq, S, L.g_bp, B, reinterpret_cast<uint8_t*>(c->cache + L.cls_off),
                                   reinterpret_cast<float*>(c->cache + L.tau_off), s, c->len_dev() + c->dims.n_layers + 1));
      }
      // a2 (split): stable class-aware compaction of the staged rows into pool_I / pool_U
      int* didx = reinterpret_cast<int*>(c->scratch + c->s_didx);
      ZDC_CUDA_TRY(launch_rank(rep_cls, c->max_seq, S, B, didx, c->max_seq,
                               reinterpret_cast<int*>(c->cache + L.posi_off), reinterpret_cast<int*>(c->cache + L.posu_off),
                               c->max_seq, reinterpret_cast<int*>(c->cache + L.ni_off),
                               reinterpret_cast<int*>(c->cache + L.nu_off), s));
      ZDC_CUDA_TRY(launch_pack(ks, L.rk_p, reinterpret_cast<uint16_t*>(c->cache + L.k_off),
                               reinterpret_cast<uint16_t*>(c->cache + L.ku_off), L.rku_p, L.rku, B, Nkv, S, c->max_seq,
                               didx, c->max_seq, s));
      ZDC_CUDA_TRY(launch_pack(vs, L.rv_p, reinterpret_cast<uint16_t*>(c->cache + L.v_off),
                               reinterpret_cast<uint16_t*>(c->cache + L.vu_off), L.rvu_p, L.rvu, B, Nkv, S, c->max_seq,
                               didx, c->max_seq, s));
    }
    // a5: y = O' W_O^R
    Epilogue e5;
    e5.mode = 0;
    e5.d = y;
    e5.ldd = d;
    e5.pdl = 1;
    g_prof_class = kProfGemmO;
    ZDC_CUDA_TRY(launch_gemm(a.o, L.ko_p, reinterpret_cast<const uint16_t*>(c->w + L.w_o), L.ko_p, M, d, L.ko_p, e5,
                             s));
    g_prof_class = kProfOther;
    ZDC_CUDA_TRY(launch_set_int(c->len_dev() + l, S, s));
    c->len[l] = S;
    c->last_layer = l;
    c->last_T = S;
  }
  c->batch = B;
  return ZDC_OK;
}

static void set_splitk_ws(zdc_ctx* c, Epilogue& e, int M, int N) {
  e.ws = reinterpret_cast<float*>(c->scratch + c->s_gsk);
  e.ws_cnt = reinterpret_cast<int*>(e.ws + static_cast<int64_t>(std::min(c->max_batch, 128)) *
                                             std::max(c->max_nqkv, c->dims.d_model));
  (void)M;
  (void)N;
}

static zdc_status enqueue_decode(zdc_ctx* c, int l0, int l1, const uint16_t* x, uint16_t* y, int B,
                                 cudaStream_t s) {
  const int d = c->dims.d_model, Nh = c->dims.n_heads, Nkv = c->dims.n_kv_heads;
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& L = c->layers[l];
    const uint16_t* xin = l == l0 ? x : y;
    int* len_dev = c->len_dev() + l;  // tokens in the cache before this step
    // a1 + a2: the new token's Q' to staging, K'/V' into the cache at position *len_dev
    Epilogue e1;
    e1.mode = 1;
    e1.qkv = qkv_dest(c, L, 1, 0, nullptr);
    e1.qkv.pos_ptr = len_dev;
    e1.qkv.pos_cap = c->max_seq;
    uint16_t* knew = reinterpret_cast<uint16_t*>(c->scratch + c->s_new);
    uint16_t* vnew = knew + static_cast<int64_t>(B) * Nkv * L.rk_p;
    if (L.split || c->kv_fp8) {  // stage the new row; the class-aware / quantizing append places it below
      e1.qkv.k = knew;
      e1.qkv.v = vnew;
      e1.qkv.pos_ptr = nullptr;
      e1.qkv.pos0 = 0;
      e1.qkv.kg = L.rk_p;
      e1.qkv.kb = static_cast<int64_t>(Nkv) * L.rk_p;
      e1.qkv.vg = L.rv_p;
      e1.qkv.vb = static_cast<int64_t>(Nkv) * L.rv_p;
    }
    const uint16_t* wqkv = reinterpret_cast<const uint16_t*>(c->w + L.w_qkv);
    const uint16_t* wo = reinterpret_cast<const uint16_t*>(c->w + L.w_o);
    const int mode = g_decode_mode;
    const bool fused_on = mode != 3 && knob("ZDC_DEC_FUSED", 1) != 0 && !c->kv_fp8;
    if (fused_on && mode != 1 && !L.split && L.w_od >= 0 && L.w_qd >= 0) {
      // the cluster layer-step: one cluster per KV group, no grid barrier (decode_cluster.cuh)
      const int C = decode_cluster_size(B, L.rk_p, c->G, Nkv, d);
      // opt-in (mode 2): at the c2 shape it measured 23.4 us per layer-step against 22.7 us for
      // the persistent kernel (profiles/r01/NOTES.md), so automatic mode keeps the latter
      if (C > 0 && mode == 2) {
        DecClusterArgs f;
        f.wqd = reinterpret_cast<const uint16_t*>(c->w + L.w_qd);
        f.wod = reinterpret_cast<const uint16_t*>(c->w + L.w_od);
        f.kc = reinterpret_cast<uint16_t*>(c->cache + L.k_off);
        f.vc = reinterpret_cast<uint16_t*>(c->cache + L.v_off);
        f.len_ptr = len_dev;
        f.err = c->len_dev() + c->dims.n_layers;
        f.x = xin;
        f.ldx = d;
        f.y = y;
        f.ldy = d;
        f.ybuf = reinterpret_cast<float*>(c->scratch + c->s_ybuf);
        f.ycnt = reinterpret_cast<int*>(f.ybuf + static_cast<int64_t>(8) * d);
        f.lse = reinterpret_cast<float*>(c->scratch + c->s_lse);
        f.B = B;
        f.d = d;
        f.nq = L.nq;
        f.nk = L.nk;
        f.Nh = Nh;
        f.Nkv = Nkv;
        f.S_cap = c->max_seq;
        f.C = C;
        static const int l2pf = knob("ZDC_CL_PF", 6);
        f.l2_prefetch = l2pf;
        f.trace = fused_trace_buffer();
        f.scale = 1.0f / std::sqrt(static_cast<float>(c->dims.d_head));
        g_prof_class = kProfDecodeLayer;
        cudaError_t e = launch_decode_cluster(f, L.rk_p, s);
        g_prof_class = kProfOther;
        if (e == cudaSuccess) continue;
        if (e != cudaErrorNotSupported) return fail(ZDC_ERR_CUDA, "cluster decode layer %d: %s", l, cudaGetErrorString(e));
        cudaGetLastError();
      }
    }
    auto fusable = [&](const LayerInfo& X) {
      return fused_on && !X.split && decode_fused_supported(B, X.rk_p, c->G) && X.rk_p == L.rk_p &&
             X.n_qkv == L.n_qkv && X.ko_p == L.ko_p;
    };
    if (fusable(L)) {
      // the run of consecutive fusable layers [l, le): ONE persistent kernel (decode_fused.cuh)
      int le = l + 1;
      while (le < l1 && fusable(c->layers[le])) ++le;
      DecFusedArgs f;
      f.layers = reinterpret_cast<const DecLayer*>(c->scratch + c->s_ltab) + l;
      f.nl = le - l;
      f.x = xin;
      f.ldx = d;
      f.y = y;
      f.ldy = d;
      f.q = reinterpret_cast<uint16_t*>(c->scratch + c->s_q);
      f.ldq = L.nq;
      f.part = reinterpret_cast<float*>(c->scratch + c->s_part);
      f.lse = reinterpret_cast<float*>(c->scratch + c->s_lse);
      f.gbar = reinterpret_cast<unsigned long long*>(c->scratch + c->s_gbar);
      f.o = reinterpret_cast<uint16_t*>(c->scratch + c->s_o);
      f.counters = reinterpret_cast<int*>(c->scratch + c->s_cnt);
      f.trace = fused_trace_buffer();
      f.B = B;
      f.d = d;
      f.n_qkv = L.n_qkv;
      f.nq = L.nq;
      f.nk = L.nk;
      f.Nh = Nh;
      f.Nkv = Nkv;
      f.S_cap = c->max_seq;
      f.splits = decode_fused_splits(B, Nkv);
      f.ko_p = L.ko_p;
      f.scale = 1.0f / std::sqrt(static_cast<float>(c->dims.d_head));
      f.err = c->len_dev() + c->dims.n_layers;
      g_prof_class = kProfDecodeLayer;
      cudaError_t e = launch_decode_fused(f, L.rk_p, s);
      g_prof_class = kProfOther;
      if (e == cudaSuccess) {
        l = le - 1;
        continue;
      }
      if (e != cudaErrorNotSupported) return fail(ZDC_ERR_CUDA, "fused decode layers [%d, %d): %s", l, le, cudaGetErrorString(e));
      cudaGetLastError();
    }
    g_prof_class = kProfGemvQkv;
    if (gemv_supported(B, d))
      ZDC_CUDA_TRY(launch_gemv(wqkv, xin, d, B, L.n_qkv, d, e1, s));
    else
    {
      if (c->s_gsk >= 0 && B <= 128) set_splitk_ws(c, e1, B, L.n_qkv);
      e1.pdl = 1;
      ZDC_CUDA_TRY(launch_gemm(xin, d, wqkv, d, B, L.n_qkv, d, e1, s));
    }
    const LayerInfo& R = c->layers[L.rep];
    const bool is_rep = L.rep == l;
    if (c->kv_fp8) {  // NEXT-4: quantize the new row into the FP8 cache at position *len_dev
      g_prof_class = kProfOther;
      ZDC_CUDA_TRY(launch_quantize_kv(knew, 1, c->cache + L.k_off, c->max_seq, B * Nkv, 0, 1, L.rk_p, len_dev, s));
      ZDC_CUDA_TRY(launch_quantize_kv(vnew, 1, c->cache + L.v_off, c->max_seq, B * Nkv, 0, 1, L.rv_p, len_dev, s));
    }
    if (L.split) {
      g_prof_class = kProfOther;
      ZDC_CUDA_TRY(launch_append(knew, vnew, L.rk_p, Nkv, reinterpret_cast<uint16_t*>(c->cache + L.k_off),
                                 reinterpret_cast<uint16_t*>(c->cache + L.v_off),
                                 reinterpret_cast<uint16_t*>(c->cache + L.ku_off),
                                 reinterpret_cast<uint16_t*>(c->cache + L.vu_off), L.rku_p, L.rku, c->max_seq,
                                 reinterpret_cast<int*>(c->cache + L.ni_off), reinterpret_cast<int*>(c->cache + L.nu_off),
                                 reinterpret_cast<int*>(c->cache + L.posi_off),
                                 reinterpret_cast<int*>(c->cache + L.posu_off), c->max_seq, len_dev,
                                 reinterpret_cast<const uint8_t*>(c->cache + R.cls_off), c->max_seq,
                                 is_rep || L.evict ? 1 : 0, B, s));  // eviction: attend first, evict after
    }
    // a3: split-K attention over the *len_dev + 1 cached keys (two pools with a token split)
    DecodeAttnArgs a;
    a.q = reinterpret_cast<const uint16_t*>(c->scratch + c->s_q);
    a.ldq = L.nq;
    a.k = reinterpret_cast<const uint16_t*>(c->cache + L.k_off);
    a.v = reinterpret_cast<const uint16_t*>(c->cache + L.v_off);
    a.S_cap = c->max_seq;
    a.len = c->max_seq;  // upper bound (fixes the split count, so the graph is length-independent)
    a.len_ptr = len_dev;
    a.o = reinterpret_cast<uint16_t*>(c->scratch + c->s_o);
    a.ldo = L.ko_p;
    a.lse = reinterpret_cast<float*>(c->scratch + c->s_lse);
    a.part = reinterpret_cast<float*>(c->scratch + c->s_part);
    a.counters = reinterpret_cast<int*>(c->scratch + c->s_cnt);
    // cached K'/V' rows before the PDL wait: 2 = into shared memory, 1 = into L2, 0 = none
    a.prefetch_before_wait = knob("ZDC_ATTN_PREWAIT", 2);
    a.B = B;
    a.Nh = Nh;
    a.Nkv = Nkv;
    a.rk = L.rk_p;
    a.rv = L.rv_p;
    a.scale = 1.0f / std::sqrt(static_cast<float>(c->dims.d_head));
    a.splits = decode_splits(B, Nkv, c->max_seq);
    {
      // L2 prefetch of the weights read next (bit 0: this layer's W_O^R, bit 1: the next layer's
      // W_QKV^R, wrapping to layer 0 for the next step); off by default (ZDC_DEC_L2PF=3 enables it):
      // measured slower in round 1, the prefetches delay the attention's own bulk copies
      static const int pf_mode = knob("ZDC_DEC_L2PF", 0);
      const LayerInfo& N = c->layers[(l + 1) % c->dims.n_layers];
      if (pf_mode & 1) {
        a.pf_ptr[0] = wo;
        a.pf_bytes[0] = static_cast<int64_t>(d) * L.ko_p * 2;
      }
      if (pf_mode & 2) {
        a.pf_ptr[1] = c->w + N.w_qkv;
        a.pf_bytes[1] = static_cast<int64_t>(N.n_qkv) * d * 2;
      }
      // only while the working set stays well inside the 126 MB L2 (the KV rows stream through too)
      if (a.pf_bytes[0] > (64ll << 20)) a.pf_bytes[0] = 0;
      if (a.pf_bytes[0] + a.pf_bytes[1] > (64ll << 20)) a.pf_bytes[1] = 0;
    }
    if (L.split) {
      a.len_ptr = nullptr;
      a.n0_ptr = reinterpret_cast<const int*>(c->cache + L.ni_off);
      a.n1_ptr = reinterpret_cast<const int*>(c->cache + L.nu_off);
      if (!L.evict) {  // evicted rows are never attended (no pool_U)
        a.k1 = reinterpret_cast<const uint16_t*>(c->cache + L.ku_off);
        a.v1 = reinterpret_cast<const uint16_t*>(c->cache + L.vu_off);
        a.rk1 = L.rku_p;
        a.rv1 = L.rvu_p;
      }
    }
    static const bool attn_tc_on = knob("ZDC_DEC_ATTN_TC", 1) != 0;
    cudaError_t ea = cudaErrorNotSupported;
    if (c->kv_fp8) {
      a.kv_fp8 = 1;
      a.splits = decode2_splits(B, Nkv, c->max_seq, L.rk_p, c->G);
      ea = launch_decode2_f8(a, s);
      if (ea != cudaSuccess) return fail(ZDC_ERR_CUDA, "decode attention (FP8 cache) layer %d: %s", l, cudaGetErrorString(ea));
    }
    if (attn_tc_on && !L.split && !c->kv_fp8 && decode_attention_tc_supported(L.rk_p, L.rv_p, c->G)) {
      // grouped-query heads: the tensor-core kernel (decode_attn_tc.cu)
      DecodeAttnArgs at = a;
      at.splits = decode_tc_splits(B, Nkv, c->max_seq);
      ea = launch_decode_attention_tc(at, s);
      if (ea != cudaSuccess && ea != cudaErrorNotSupported)
        return fail(ZDC_ERR_CUDA, "decode attention (tensor cores) layer %d: %s", l, cudaGetErrorString(ea));
      if (ea == cudaErrorNotSupported) cudaGetLastError();
    }
    if (ea != cudaSuccess) ZDC_CUDA_TRY(launch_decode_attention(a, s));
    if (L.evict && !is_rep) {  // the token attended itself; evict it now if its group classed it unimportant
      g_prof_class = kProfOther;
      ZDC_CUDA_TRY(launch_evict_last(reinterpret_cast<const uint8_t*>(c->cache + R.cls_off), c->max_seq,
                                     reinterpret_cast<int*>(c->cache + L.ni_off), reinterpret_cast<int*>(c->cache + L.nu_off),
                                     reinterpret_cast<int*>(c->cache + L.posu_off), c->max_seq, len_dev, c->max_seq, B, s));
    }
    if (L.split && is_rep) {
      g_prof_class = kProfOther;
      ZDC_CUDA_TRY(launch_classify(a.lse, Nh, c->importance_mode, reinterpret_cast<const float*>(c->cache + L.tau_off),
                                   reinterpret_cast<float*>(c->cache + L.score_off),
                                   reinterpret_cast<uint8_t*>(c->cache + L.cls_off), c->max_seq, nullptr, 0, L.rk_p,
                                   Nkv, reinterpret_cast<uint16_t*>(c->cache + L.k_off),
                                   reinterpret_cast<uint16_t*>(c->cache + L.v_off),
                                   reinterpret_cast<uint16_t*>(c->cache + L.ku_off),
                                   reinterpret_cast<uint16_t*>(c->cache + L.vu_off), L.rku_p, L.rku, c->max_seq,
                                   reinterpret_cast<int*>(c->cache + L.ni_off), reinterpret_cast<int*>(c->cache + L.nu_off),
                                   reinterpret_cast<int*>(c->cache + L.posi_off),
                                   reinterpret_cast<int*>(c->cache + L.posu_off), len_dev, B, s));
    }
    // a5: y = O' W_O^R; this kernel also advances *len_dev (all readers of it have run)
    Epilogue e5;
    e5.mode = 0;
    e5.d = y;
    e5.ldd = d;
    e5.len_inc = len_dev;
    e5.len_cap = c->max_seq;
    e5.err = c->len_dev() + c->dims.n_layers;
    g_prof_class = kProfGemvO;
    if (gemv_supported(B, L.ko_p))
      ZDC_CUDA_TRY(launch_gemv(wo, a.o, L.ko_p, B, d, L.ko_p, e5, s));
    else
    {
      if (c->s_gsk >= 0 && B <= 128) set_splitk_ws(c, e5, B, d);
      e5.pdl = 1;
      ZDC_CUDA_TRY(launch_gemm(a.o, L.ko_p, wo, L.ko_p, B, d, L.ko_p, e5, s));
    }
    g_prof_class = kProfOther;
  }
  return ZDC_OK;
}

zdc_status zdc_decode(zdc_ctx* c, int32_t l0, int32_t l1, const uint16_t* x, uint16_t* y, int32_t B, void* stream) {
  zdc_status st = check_run(c, l0, l1, x, y, "zdc_decode");
  if (st == ZDC_OK && B > 0 && ranges_overlap(x, 2LL * B * c->dims.d_model, y, 2LL * B * c->dims.d_model))
    return fail(ZDC_ERR_INVALID_ARG, "zdc_decode: x and y overlap");
  if (st != ZDC_OK) return st;
  if (B <= 0 || B > c->max_batch) return fail(ZDC_ERR_CAPACITY, "zdc_decode: B=%d (max_batch %d)", B, c->max_batch);
  if (c->batch != 0 && B != c->batch) return fail(ZDC_ERR_SHAPE, "zdc_decode: B=%d but cache batch is %d", B, c->batch);
  for (int l = l0; l < l1; ++l) {
    if (c->len[l] + 1 > c->max_seq)
      return fail(ZDC_ERR_CAPACITY, "zdc_decode: layer %d len %d + 1 > max_seq %d", l, c->len[l], c->max_seq);
    if (c->sp_layer[l])
      return fail(ZDC_ERR_UNSUPPORTED, "zdc_decode: layer %d holds an SP-sharded cache (SP decode is NEXT-2)", l);
    const LayerInfo& L = c->layers[l];
    if (L.split && L.rep != l) {
      // the representative must have classified this position (in this call or an earlier one)
      const int rep_len = c->len[L.rep] + ((L.rep >= l0 && L.rep < l) ? 1 : 0);
      if (rep_len <= c->len[l])
        return fail(ZDC_ERR_STATE, "zdc_decode: layer %d: representative %d has not classified position %d", l, L.rep,
                    c->len[l]);
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  g_launches = 0;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (s) ZDC_CUDA_TRY(cudaStreamIsCapturing(s, &cap));
  const bool graph = c->use_graphs && !prof_enabled() && s != nullptr && s != cudaStreamPerThread &&
                     cap == cudaStreamCaptureStatusNone;
  if (graph) {
    // The whole [l0, l1) decode step is one CUDA graph, replayed every step: lengths live on the
    // device, so the same graph serves every position.
    auto key = std::make_tuple(static_cast<int>(l0), static_cast<int>(l1), static_cast<int>(B),
                               static_cast<const void*>(x), static_cast<void*>(y), s);
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
      cudaGraph_t gr = nullptr;
      ZDC_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      zdc_status est = enqueue_decode(c, l0, l1, x, y, B, s);
      cudaError_t ce = cudaStreamEndCapture(s, &gr);
      if (est != ZDC_OK) {
        if (gr) cudaGraphDestroy(gr);
        return est;
      }
      if (ce != cudaSuccess) return fail(ZDC_ERR_CUDA, "zdc_decode: capture failed: %s", cudaGetErrorString(ce));
      zdc_ctx::GraphEntry ent;
      ce = cudaGraphInstantiate(&ent.exec, gr, 0);
      cudaGraphDestroy(gr);
      if (ce != cudaSuccess) return fail(ZDC_ERR_CUDA, "zdc_decode: instantiate: %s", cudaGetErrorString(ce));
      ent.kernels = g_launches;
      it = c->graphs.emplace(key, ent).first;
    }
    ZDC_CUDA_TRY(cudaGraphLaunch(it->second.exec, s));
    g_launches = it->second.kernels;
  } else {
    st = enqueue_decode(c, l0, l1, x, y, B, s);
    if (st != ZDC_OK) return st;
  }
  for (int l = l0; l < l1; ++l) c->len[l] += 1;
  c->last_layer = l1 - 1;
  c->last_T = 1;
  c->batch = B;
  return ZDC_OK;
}

// ------------------------------------------------------------------ inspection
zdc_status zdc_cache_length(const zdc_ctx* c, int32_t layer, int32_t* len) {
  if (!c || !len) return fail(ZDC_ERR_INVALID_ARG, "zdc_cache_length: null argument");
  if (layer < 0 || layer >= c->dims.n_layers) return fail(ZDC_ERR_SHAPE, "zdc_cache_length: layer %d", layer);
  *len = c->len[layer];
  return ZDC_OK;
}

zdc_status zdc_cache_sync(zdc_ctx* c, void* stream) {
  if (!c) return fail(ZDC_ERR_INVALID_ARG, "zdc_cache_sync: null ctx");
  if (!c->cache) return fail(ZDC_ERR_STATE, "zdc_cache_sync: ctx not bound");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int> h(c->dims.n_layers + 2);
  ZDC_CUDA_TRY(cudaMemcpyAsync(h.data(), c->len_dev(), h.size() * 4, cudaMemcpyDeviceToHost, s));
  ZDC_CUDA_TRY(cudaStreamSynchronize(s));
  for (int l = 0; l < c->dims.n_layers; ++l) c->len[l] = h[l];
  if (h[c->dims.n_layers + 1])
    return fail(ZDC_ERR_INVALID_ARG, "zdc_cache_sync: a representative layer produced a NaN importance score "
                "(non-finite activations); its classes are invalid (zdc_cache_reset clears)");
  if (h[c->dims.n_layers])
    return fail(ZDC_ERR_CAPACITY, "zdc_cache_sync: decode steps replayed past max_seq = %d (each step uses one "
                "row; the overflowing steps rewrote the last row and their outputs are invalid; zdc_cache_reset clears)",
                c->max_seq);
  return ZDC_OK;
}

zdc_status zdc_cache_reset(zdc_ctx* c, void* stream) {
  if (!c) return fail(ZDC_ERR_INVALID_ARG, "zdc_cache_reset: null ctx");
  if (!c->cache) return fail(ZDC_ERR_STATE, "zdc_cache_reset: ctx not bound");
  // Only the lengths are reset: no kernel ever reads a cache row at or beyond its layer's length.
  ZDC_CUDA_TRY(cudaMemsetAsync(c->len_dev(), 0, static_cast<size_t>(c->dims.n_layers + 2) * 4,
                               static_cast<cudaStream_t>(stream)));
  c->len.assign(c->dims.n_layers, 0);
  c->sp_layer.assign(c->dims.n_layers, 0);
  c->sp_prompt.assign(c->dims.n_layers, 0);
  c->batch = 0;
  return ZDC_OK;
}

static float bf16_to_f32(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

zdc_status zdc_cache_export(const zdc_ctx* c, int32_t layer, float* k, float* v, uint8_t* is_imp, float* tau,
                            void* stream) {
  if (!c) return fail(ZDC_ERR_INVALID_ARG, "zdc_cache_export: null ctx");
  if (!c->cache) return fail(ZDC_ERR_STATE, "zdc_cache_export: ctx not bound");
  if (layer < 0 || layer >= c->dims.n_layers) return fail(ZDC_ERR_SHAPE, "zdc_cache_export: layer %d", layer);
  const LayerInfo& L = c->layers[layer];
  if (c->sp_layer[layer]) {
    // an SP layer keeps a gather buffer (all-gather) or only its head groups (Ulysses): the rows
    // are not exported; the classes and tau of a split group are (global positions)
    if (k || v) return fail(ZDC_ERR_UNSUPPORTED, "zdc_cache_export: layer %d holds an SP-sharded cache (k, v)", layer);
    ZDC_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    const int B = c->batch, len = c->len[layer];
    if (is_imp) {
      if (!L.split) {
        std::memset(is_imp, 1, static_cast<size_t>(B) * len);
      } else {
        for (int b = 0; b < B; ++b)
          ZDC_CUDA_TRY(cudaMemcpy(is_imp + static_cast<int64_t>(b) * len,
                                  c->cache + c->layers[L.rep].cls_off + static_cast<int64_t>(b) * c->max_seq, len,
                                  cudaMemcpyDeviceToHost));
      }
    }
    if (tau) {
      if (L.split)
        ZDC_CUDA_TRY(cudaMemcpy(tau, c->cache + c->layers[L.rep].tau_off, static_cast<size_t>(B) * 4,
                                cudaMemcpyDeviceToHost));
      else
        for (int b = 0; b < B; ++b) tau[b] = INFINITY;
    }
    return ZDC_OK;
  }
  const int B = c->batch, len = c->len[layer], Nkv = c->dims.n_kv_heads, S_cap = c->max_seq;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ZDC_CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t rows = static_cast<int64_t>(c->max_batch) * Nkv * S_cap;
  auto fetch16 = [&](int64_t off, int64_t n, std::vector<uint16_t>& h) {
    h.resize(n);
    return cudaMemcpy(h.data(), c->cache + off, n * 2, cudaMemcpyDeviceToHost);
  };
  auto fetch32 = [&](int64_t off, int64_t n, std::vector<int>& h) {
    h.resize(n);
    return cudaMemcpy(h.data(), c->cache + off, n * 4, cudaMemcpyDeviceToHost);
  };
  if (c->kv_fp8) {  // NEXT-4: rows of r E4M3 codes + f32 scale + 12 pad bytes -> code * scale
    const int64_t rb = L.rk_p + 16;
    std::vector<uint8_t> k8(rows * rb), v8(rows * rb);
    ZDC_CUDA_TRY(cudaMemcpy(k8.data(), c->cache + L.k_off, k8.size(), cudaMemcpyDeviceToHost));
    ZDC_CUDA_TRY(cudaMemcpy(v8.data(), c->cache + L.v_off, v8.size(), cudaMemcpyDeviceToHost));
    auto e4m3 = [](uint8_t code) {
      const int e = (code >> 3) & 15, m = code & 7;
      const float mag = e == 0 ? std::ldexp(m / 8.0f, -6) : std::ldexp(1.0f + m / 8.0f, e - 7);
      return (code & 0x80) ? -mag : mag;
    };
    for (int b = 0; b < B; ++b)
      for (int t = 0; t < len; ++t)
        for (int g = 0; g < Nkv; ++g) {
          const int64_t row = (static_cast<int64_t>(b) * Nkv + g) * S_cap + t;
          const int64_t o = (static_cast<int64_t>(b) * len + t) * Nkv + g;
          float ks, vs;
          std::memcpy(&ks, &k8[row * rb + L.rk_p], 4);
          std::memcpy(&vs, &v8[row * rb + L.rk_p], 4);
          for (int e2 = 0; e2 < L.rk; ++e2) {
            if (k) k[o * L.rk + e2] = e4m3(k8[row * rb + e2]) * ks;
            if (v) v[o * L.rv + e2] = e4m3(v8[row * rb + e2]) * vs;
          }
        }
    if (is_imp) std::memset(is_imp, 1, static_cast<size_t>(B) * len);
    if (tau)
      for (int b = 0; b < B; ++b) tau[b] = INFINITY;
    return ZDC_OK;
  }
  std::vector<uint16_t> ki, vi, ku, vu;
  std::vector<int> posi, posu, ni, nu;
  ZDC_CUDA_TRY(fetch16(L.k_off, rows * L.rk_p, ki));
  ZDC_CUDA_TRY(fetch16(L.v_off, rows * L.rv_p, vi));
  if (L.split) {
    ZDC_CUDA_TRY(fetch16(L.ku_off, rows * L.rku_p, ku));
    ZDC_CUDA_TRY(fetch16(L.vu_off, rows * L.rvu_p, vu));
    ZDC_CUDA_TRY(fetch32(L.posi_off, static_cast<int64_t>(c->max_batch) * S_cap, posi));
    ZDC_CUDA_TRY(fetch32(L.posu_off, static_cast<int64_t>(c->max_batch) * S_cap, posu));
    ZDC_CUDA_TRY(fetch32(L.ni_off, c->max_batch, ni));
    ZDC_CUDA_TRY(fetch32(L.nu_off, c->max_batch, nu));
  }
  const int64_t nk_out = static_cast<int64_t>(B) * len * Nkv;
  if (k) std::fill(k, k + nk_out * L.rk, 0.f);
  if (v) std::fill(v, v + nk_out * L.rv, 0.f);
  if (is_imp) std::memset(is_imp, L.split ? 0 : 1, static_cast<size_t>(B) * len);
  // place pool row i of (b, g) at position t, zero-filled to the important widths
  auto place = [&](int b, int t, int i, const std::vector<uint16_t>& K, const std::vector<uint16_t>& V, int wk, int wv,
                   int rk_valid, int rv_valid) {
    if (t < 0 || t >= len) return;
    for (int g = 0; g < Nkv; ++g) {
      const int64_t row = (static_cast<int64_t>(b) * Nkv + g) * S_cap + i;
      const int64_t o = (static_cast<int64_t>(b) * len + t) * Nkv + g;
      if (k)
        for (int e = 0; e < rk_valid; ++e) k[o * L.rk + e] = bf16_to_f32(K[row * wk + e]);
      if (v)
        for (int e = 0; e < rv_valid; ++e) v[o * L.rv + e] = bf16_to_f32(V[row * wv + e]);
    }
  };
  for (int b = 0; b < B; ++b) {
    if (!L.split) {
      for (int t = 0; t < len; ++t) place(b, t, t, ki, vi, L.rk_p, L.rv_p, L.rk, L.rv);
      continue;
    }
    for (int i = 0; i < ni[b]; ++i) {
      const int t = posi[static_cast<int64_t>(b) * S_cap + i];
      place(b, t, i, ki, vi, L.rk_p, L.rv_p, L.rk, L.rv);
      if (is_imp && t >= 0 && t < len) is_imp[static_cast<int64_t>(b) * len + t] = 1;
    }
    for (int i = 0; i < nu[b]; ++i) {
      const int t = posu[static_cast<int64_t>(b) * S_cap + i];
      place(b, t, i, ku, vu, L.rku_p, L.rvu_p, L.rku, L.rvu);
    }
  }
  if (tau) {
    if (L.split) {
      ZDC_CUDA_TRY(cudaMemcpy(tau, c->cache + c->layers[L.rep].tau_off, static_cast<size_t>(B) * 4,
                              cudaMemcpyDeviceToHost));
    } else {
      for (int b = 0; b < B; ++b) tau[b] = INFINITY;
    }
  }
  return ZDC_OK;
}

zdc_status zdc_scores_export(const zdc_ctx* c, int32_t layer, float* scores, void* stream) {
  if (!c || !scores) return fail(ZDC_ERR_INVALID_ARG, "zdc_scores_export: null argument");
  if (layer < 0 || layer >= c->dims.n_layers) return fail(ZDC_ERR_SHAPE, "zdc_scores_export: layer %d", layer);
  const LayerInfo& L = c->layers[layer];
  if (!L.split || L.rep != layer)
    return fail(ZDC_ERR_STATE, "zdc_scores_export: layer %d is not the representative of a split group", layer);
  ZDC_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  const int B = c->batch, len = c->len[layer];
  std::vector<float> h(static_cast<size_t>(c->max_batch) * c->max_seq);
  ZDC_CUDA_TRY(cudaMemcpy(h.data(), c->cache + L.score_off, h.size() * 4, cudaMemcpyDeviceToHost));
  for (int b = 0; b < B; ++b)
    for (int t = 0; t < len; ++t) scores[static_cast<int64_t>(b) * len + t] = h[static_cast<size_t>(b) * c->max_seq + t];
  return ZDC_OK;
}

zdc_status zdc_last_lse(const zdc_ctx* c, int32_t layer, float* lse_host, void* stream) {
  if (!c || !lse_host) return fail(ZDC_ERR_INVALID_ARG, "zdc_last_lse: null argument");
  if (layer != c->last_layer) return fail(ZDC_ERR_STATE, "zdc_last_lse: layer %d is not the last processed (%d)",
                                          layer, c->last_layer);
  const int B = c->batch, Nh = c->dims.n_heads, T = c->last_T;
  ZDC_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  ZDC_CUDA_TRY(cudaMemcpy(lse_host, c->scratch + c->s_lse, static_cast<size_t>(B) * Nh * T * 4, cudaMemcpyDeviceToHost));
  return ZDC_OK;
}

// ------------------------------------------------------------------ kernel-level entry
zdc_status zdc_gemm_bf16(const uint16_t* a, const uint16_t* b, uint16_t* d, int32_t M, int32_t N, int32_t K,
                         void* stream) {
  if (!a || !b || !d) return fail(ZDC_ERR_INVALID_ARG, "zdc_gemm_bf16: null pointer");
  if (M <= 0 || N <= 0 || K <= 0 || K % 64 != 0 || N % 8 != 0)
    return fail(ZDC_ERR_SHAPE, "zdc_gemm_bf16: M=%d N=%d K=%d (need K %% 64 == 0, N %% 8 == 0)", M, N, K);
  zdc_status st = check_sticky();
  if (st != ZDC_OK) return st;
  g_launches = 0;
  Epilogue e;
  e.mode = 0;
  e.d = d;
  e.ldd = N;
  ZDC_CUDA_TRY(launch_gemm(a, K, b, K, M, N, K, e, static_cast<cudaStream_t>(stream)));
  return ZDC_OK;
}

zdc_status zdc_prefill_attention_bf16(const uint16_t* q, const uint16_t* k, const uint16_t* v, uint16_t* o,
                                      float* lse, int32_t B, int32_t S, int32_t Nh, int32_t Nkv, int32_t r,
                                      float scale, void* stream) {
  if (!q || !k || !v || !o) return fail(ZDC_ERR_INVALID_ARG, "zdc_prefill_attention_bf16: null pointer");
  if (B <= 0 || S <= 0 || Nh <= 0 || Nkv <= 0 || Nh % Nkv != 0 || r <= 0 || r > 128 || r % 16 != 0)
    return fail(ZDC_ERR_SHAPE, "zdc_prefill_attention_bf16: B=%d S=%d Nh=%d Nkv=%d r=%d", B, S, Nh, Nkv, r);
  const int G = Nh / Nkv;
  if (G != 1 && G != 2 && G != 4 && G != 8) return fail(ZDC_ERR_UNSUPPORTED, "group size %d", G);
  zdc_status st = check_sticky();
  if (st != ZDC_OK) return st;
  g_launches = 0;
  PrefillAttnArgs a;
  a.q = q;
  a.ldq = static_cast<int64_t>(Nh) * r;
  a.k = k;
  a.v = v;
  a.S_cap = S;
  a.o = o;
  a.ldo = static_cast<int64_t>(Nh) * r;
  a.lse = lse;
  a.B = B;
  a.S = S;
  a.Nh = Nh;
  a.Nkv = Nkv;
  a.rk = r;
  a.rv = r;
  a.scale = scale;
  a.q_pos0 = 0;
  a.q_row0 = 0;
  a.n_q = S;
  ZDC_CUDA_TRY(launch_prefill_attention(a, static_cast<cudaStream_t>(stream)));
  return ZDC_OK;
}

int64_t zdc_decode_attention_workspace(int32_t B, int32_t Nh, int32_t Nkv, int32_t r) {
  return static_cast<int64_t>(B) * Nh * 128 * (r + 2) * 4 + static_cast<int64_t>(B) * Nkv * 4 + 256;
}

zdc_status zdc_decode_attention_bf16(const uint16_t* q, const uint16_t* k, const uint16_t* v, uint16_t* o,
                                     float* lse, int32_t B, int32_t Nh, int32_t Nkv, int32_t r, int32_t len,
                                     int32_t S_cap, float scale, void* workspace, void* stream) {
  if (!q || !k || !v || !o || !workspace) return fail(ZDC_ERR_INVALID_ARG, "zdc_decode_attention_bf16: null pointer");
  if (B <= 0 || Nh <= 0 || Nkv <= 0 || Nh % Nkv != 0 || r <= 0 || r > 128 || r % 16 != 0 || len <= 0 ||
      len > S_cap)
    return fail(ZDC_ERR_SHAPE, "zdc_decode_attention_bf16: B=%d Nh=%d Nkv=%d r=%d len=%d S_cap=%d", B, Nh, Nkv, r,
                len, S_cap);
  zdc_status st = check_sticky();
  if (st != ZDC_OK) return st;
  g_launches = 0;
  DecodeAttnArgs a;
  a.q = q;
  a.ldq = static_cast<int64_t>(Nh) * r;
  a.k = k;
  a.v = v;
  a.rk = r;
  a.rv = r;
  a.S_cap = S_cap;
  a.len = len;
  a.o = o;
  a.ldo = static_cast<int64_t>(Nh) * r;
  a.lse = lse;
  a.part = static_cast<float*>(workspace);
  a.counters = reinterpret_cast<int*>(static_cast<uint8_t*>(workspace) +
                                      static_cast<int64_t>(B) * Nh * 128 * (r + 2) * 4);
  a.B = B;
  a.Nh = Nh;
  a.Nkv = Nkv;
  a.scale = scale;
  a.splits = decode_splits(B, Nkv, len);
  a.prefetch_before_wait = 0;
  ZDC_CUDA_TRY(launch_decode_attention(a, static_cast<cudaStream_t>(stream)));
  return ZDC_OK;
}

zdc_status zdc_gemv_bf16(const uint16_t* w, const uint16_t* x, uint16_t* y, int32_t B, int32_t N, int32_t K,
                         void* stream) {
  if (!w || !x || !y) return fail(ZDC_ERR_INVALID_ARG, "zdc_gemv_bf16: null pointer");
  if (B <= 0 || B > 8 || N <= 0 || K <= 0 || K % 8 != 0)
    return fail(ZDC_ERR_SHAPE, "zdc_gemv_bf16: B=%d N=%d K=%d (need 1 <= B <= 8, K %% 8 == 0)", B, N, K);
  zdc_status st = check_sticky();
  if (st != ZDC_OK) return st;
  g_launches = 0;
  Epilogue e;
  e.mode = 0;
  e.d = y;
  e.ldd = N;
  ZDC_CUDA_TRY(launch_gemv(w, x, K, B, N, K, e, static_cast<cudaStream_t>(stream)));
  return ZDC_OK;
}

}  // extern "C"
