// ctx.h — host-side state behind the opaque zdc_ctx (internal).
#pragma once
#include <stdint.h>

#include <cstdlib>
#include <map>
#include <tuple>
#include <vector>

#include <cuda_runtime.h>

#include "zdc.h"
#include "knobs.h"

namespace zdc {

// Per-layer packing / cache layout.  Ranks are the plan's; *_p are padded to 16.
struct LayerInfo {
  int rk = 0, rku = 0, rv = 0, rvu = 0;
  int rk_p = 0, rv_p = 0, rku_p = 0, rvu_p = 0;
  int g_bp = 10000, rep = 0;
  bool split = false;
  bool evict = false;  // split group with r^u = 0: unimportant tokens are evicted (H2O-ZDC, NEXT-4)
  int nq = 0, nk = 0, nv = 0, n_qkv = 0, ko_p = 0;
  int64_t w_qkv = 0, w_o = 0;                      // byte offsets in the weight region
  int64_t w_od = -1;  // W_O decode copy [Nkv][d][G*r] for the cluster decode kernel (-1: none)
  int64_t w_qd = -1;  // W_QKV decode copy (pre-swizzled tiles) for the cluster decode kernel
  int64_t k_off = 0, v_off = 0;                    // byte offsets in the cache region
  int64_t cls_off = 0, tau_off = 0, score_off = 0;  // representative layers of split groups
  // token split: pool_U (unimportant rows, truncated width), positions and per-sequence counts
  int64_t ku_off = 0, vu_off = 0, posi_off = 0, posu_off = 0, ni_off = 0, nu_off = 0;
};

struct CommState;

}  // namespace zdc

struct zdc_ctx {
  zdc_dims dims{};
  int G = 1;
  int max_batch = 0, max_seq = 0;
  int importance_mode = 0;
  int kv_fp8 = 0;  // FP8 E4M3 compressed cache (NEXT-4): rows of r codes + f32 scale + 12 pad bytes
  std::vector<zdc::LayerInfo> layers;
  int64_t weight_bytes = 0, cache_bytes = 0, scratch_bytes = 0;
  int64_t s_q = 0, s_o = 0, s_lse = 0, s_part = 0;  // scratch offsets
  int64_t s_ks = 0, s_vs = 0, s_didx = 0, s_new = 0;  // token-split staging
  int64_t s_cnt = 0;                                  // decode merge counters
  int64_t s_gbar = 0;                                 // fused decode grid barrier (monotonic counter)
  int64_t s_ltab = 0;                                 // fused decode layer table
  int64_t s_ybuf = 0;
  int64_t s_gsk = -1;                                 // split-K decode GEMM workspace (max_batch > 8)
  int64_t s_sp = 0;                                   // Ulysses SP all-to-all send | recv slabs
  int max_nqkv = 0;                                 // cluster decode: f32 y accumulator [8][d] + counters [16]
  int ldq = 0, ldo = 0;
  uint8_t* w = nullptr;
  uint8_t* cache = nullptr;
  uint8_t* scratch = nullptr;
  std::vector<int> len;  // per-layer cache length
  std::vector<int> sp_layer;  // 1 = the layer's cache holds an SP gather buffer (not position-ordered)
  std::vector<int> sp_prompt;  // SP prefill length of each such layer (zdc_sp_decode counts tokens after it)
  int batch = 0;
  int last_layer = -1, last_T = 0;
  zdc::CommState* comm = nullptr;
  int64_t len_dev_off = 0;  // int32 [n_layers] device-side cache lengths (in the cache region)
  // zdc_decode CUDA graphs, keyed by (l0, l1, B, x, y, stream)
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
  };
  std::map<std::tuple<int, int, int, const void*, void*, cudaStream_t>, GraphEntry> graphs;
  bool use_graphs = zdc::knob("ZDC_NO_GRAPH", 0) == 0;  // zdc_decode replays one CUDA graph per call shape
  int* len_dev() { return reinterpret_cast<int*>(cache + len_dev_off); }
};

namespace zdc {
void comm_destroy(zdc_ctx* c);
void graphs_destroy(zdc_ctx* c);
}
