// comm.cpp — a6: sequence-parallel prefill that exchanges ONLY the compressed K'/V'
// (§5.3: "transmitting compressed Q, K, and V tensors ... significantly reduces
// communication time overhead"; this build all-gathers K'/V', reading c17).
//
// Per layer, on rank p of P (one process per GPU):
//   a1  local tokens -> Q' (staging) and K'/V' written by the GEMM epilogue straight into this
//       rank's slot of the gather buffer [P][K|V][B][N_kv][n_local][r] (no pack pass)
//   a6  in-place ncclAllGather of the slots over NVLink (bytes = (P-1)/P B S N_kv (r_k+r_v) 2)
//   a3  local queries (global positions: contiguous or zigzag) attend to every key at or before
//       them; the tcgen05 attention kernel maps key tiles to (owner rank, local row) itself
//   a5  local rows -> y_local
// zdc_sp_prefill_ulysses is the paper's own dataflow instead (Fig. bkg:fig:all2all): a1 writes
// per-destination slabs of the compressed Q'/K'/V' (GEMM epilogue mode 2), all-to-all #1 gives every
// rank ALL tokens of its N_h/P heads, a3 runs the ordinary causal kernel over the full sequence for
// those heads (the rank keeps their K'/V' cache), all-to-all #2 returns O' to the token owners, a5.
// NCCL is resolved at run time (dlopen of libnccl.so.2, i.e. the copy torch already loaded), so
// the library has no link-time NCCL dependency.  zdc_sp_set_exchange_hook / _alltoall_hook replace
// the NCCL collectives by caller callbacks for single-GPU multi-process tests.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "api_util.h"
#include "ctx.h"
#include "kernels.h"

typedef void (*zdc_exchange_fn)(void* user, void* gather_buf, int64_t chunk_bytes, int32_t rank, int32_t world,
                                void* stream);
typedef void (*zdc_alltoall_fn)(void* user, const void* send, void* recv, int64_t chunk_bytes, int32_t rank,
                                int32_t world, void* stream);

namespace zdc {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

static NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.h, "ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.h, "ncclAllGather"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.h, "ncclGetErrorString"));
    api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(api.h, "ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(api.h, "ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(api.h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(api.h, "ncclGroupEnd"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.GetErrorString &&
             api.Send && api.Recv && api.GroupStart && api.GroupEnd;
  });
  return &api;
}

struct CommState {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  zdc_exchange_fn hook = nullptr;
  void* hook_user = nullptr;
  zdc_alltoall_fn a2a_hook = nullptr;
  void* a2a_user = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // overlapped exchange (layout 2): a dedicated comm stream and its handoff events
  cudaStream_t cs = nullptr;
  cudaEvent_t e_a1[2] = {nullptr, nullptr}, e_ag[2] = {nullptr, nullptr};
};

static cudaError_t comm_stream(CommState* cm) {
  if (cm->cs) return cudaSuccess;
  cudaError_t e = cudaStreamCreateWithFlags(&cm->cs, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&cm->e_a1[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cm->e_ag[i], cudaEventDisableTiming);
  }
  return e;
}

void comm_destroy(zdc_ctx* c) {
  if (!c->comm) return;
  if (c->comm->cs) cudaStreamDestroy(c->comm->cs);
  for (int i = 0; i < 2; ++i) {
    if (c->comm->e_a1[i]) cudaEventDestroy(c->comm->e_a1[i]);
    if (c->comm->e_ag[i]) cudaEventDestroy(c->comm->e_ag[i]);
  }
  if (c->comm->comm && nccl_api()->ok) nccl_api()->CommDestroy(c->comm->comm);
  if (c->comm->e0) cudaEventDestroy(c->comm->e0);
  if (c->comm->e1) cudaEventDestroy(c->comm->e1);
  delete c->comm;
  c->comm = nullptr;
}

// global position of local token t on rank p (layout 0 contiguous, 1 zigzag, 2 zigzag overlapped)
static inline int sp_position(int S, int P, int p, int layout, int t) {
  const int n = S / P;
  if (layout == 0) return p * n + t;
  const int c = S / (2 * P);
  return t < c ? p * c + t : (2 * P - 1 - p) * c + (t - c);
}

}  // namespace zdc

using namespace zdc;

extern "C" {

zdc_status zdc_comm_unique_id(void* out) {
  if (!out) return fail(ZDC_ERR_INVALID_ARG, "zdc_comm_unique_id: null output");
  NcclApi* api = nccl_api();
  if (!api->ok) return fail(ZDC_ERR_NCCL, "zdc_comm_unique_id: libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t r = api->GetUniqueId(&id);
  if (r != ncclSuccess) return fail(ZDC_ERR_NCCL, "ncclGetUniqueId: %s", api->GetErrorString(r));
  std::memcpy(out, &id, sizeof(id));
  return ZDC_OK;
}

zdc_status zdc_comm_init(zdc_ctx* c, const void* uid, int32_t rank, int32_t world) {
  if (!c || !uid) return fail(ZDC_ERR_INVALID_ARG, "zdc_comm_init: null argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(ZDC_ERR_INVALID_ARG, "zdc_comm_init: rank %d world %d", rank, world);
  NcclApi* api = nccl_api();
  if (!api->ok) return fail(ZDC_ERR_NCCL, "zdc_comm_init: libnccl.so.2 not loadable");
  comm_destroy(c);
  c->comm = new CommState();
  c->comm->rank = rank;
  c->comm->world = world;
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclResult_t r = api->CommInitRank(&c->comm->comm, world, id, rank);
  if (r != ncclSuccess) {
    comm_destroy(c);
    return fail(ZDC_ERR_NCCL, "ncclCommInitRank: %s", api->GetErrorString(r));
  }
  ZDC_CUDA_TRY(cudaEventCreate(&c->comm->e0));
  ZDC_CUDA_TRY(cudaEventCreate(&c->comm->e1));
  return ZDC_OK;
}

zdc_status zdc_sp_set_exchange_hook(zdc_ctx* c, zdc_exchange_fn fn, void* user, int32_t rank, int32_t world) {
  if (!c || !fn) return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_set_exchange_hook: null argument");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_set_exchange_hook: rank %d world %d", rank, world);
  comm_destroy(c);
  c->comm = new CommState();
  c->comm->rank = rank;
  c->comm->world = world;
  c->comm->hook = fn;
  c->comm->hook_user = user;
  ZDC_CUDA_TRY(cudaEventCreate(&c->comm->e0));
  ZDC_CUDA_TRY(cudaEventCreate(&c->comm->e1));
  return ZDC_OK;
}

zdc_status zdc_sp_set_alltoall_hook(zdc_ctx* c, zdc_alltoall_fn fn, void* user, int32_t rank, int32_t world) {
  if (!c || !fn) return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_set_alltoall_hook: null argument");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_set_alltoall_hook: rank %d world %d", rank, world);
  if (c->comm && (c->comm->rank != rank || c->comm->world != world)) comm_destroy(c);
  if (!c->comm) {
    c->comm = new CommState();
    c->comm->rank = rank;
    c->comm->world = world;
    ZDC_CUDA_TRY(cudaEventCreate(&c->comm->e0));
    ZDC_CUDA_TRY(cudaEventCreate(&c->comm->e1));
  }
  c->comm->a2a_hook = fn;
  c->comm->a2a_user = user;
  return ZDC_OK;
}

zdc_status zdc_sp_positions(int32_t S_total, int32_t world, int32_t rank, int32_t layout, int32_t* positions) {
  if (!positions) return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_positions: null output");
  if (world < 1 || rank < 0 || rank >= world || layout < 0 || layout > 2)
    return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_positions: rank %d world %d layout %d", rank, world, layout);
  if (S_total <= 0 || S_total % (layout >= 1 ? 2 * world : world) != 0)
    return fail(ZDC_ERR_SHAPE, "zdc_sp_positions: S_total %d not divisible by %d", S_total,
                layout >= 1 ? 2 * world : world);
  const int n = S_total / world;
  for (int t = 0; t < n; ++t) positions[t] = sp_position(S_total, world, rank, layout, t);
  return ZDC_OK;
}

// in-place all-gather of P equal slots of buf (slot q = rank q's chunk)
static zdc_status sp_allgather(zdc_ctx* c, uint8_t* buf, int64_t chunk_bytes, cudaStream_t s) {
  const int p = c->comm->rank;
  if (c->comm->hook) {
    c->comm->hook(c->comm->hook_user, buf, chunk_bytes, p, c->comm->world, s);
    return ZDC_OK;
  }
  if (!c->comm->comm) return fail(ZDC_ERR_STATE, "zdc_sp_prefill: no NCCL communicator and no exchange hook");
  ncclResult_t r = nccl_api()->AllGather(buf + p * chunk_bytes, buf, static_cast<size_t>(chunk_bytes), ncclUint8,
                                         c->comm->comm, s);
  if (r != ncclSuccess) return fail(ZDC_ERR_NCCL, "ncclAllGather: %s", nccl_api()->GetErrorString(r));
  return ZDC_OK;
}

zdc_status zdc_sp_prefill(zdc_ctx* c, int32_t l0, int32_t l1, const uint16_t* x, uint16_t* y, int32_t B,
                          int32_t S_total, int32_t layout, zdc_sp_stats* stats, void* stream) {
  if (!c || !x || !y) return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_prefill: null argument");
  if (x == y || (B > 0 && S_total > 0 && ranges_overlap(x, 2LL * B * (S_total / std::max(1, c->comm ? c->comm->world : 1)) * c->dims.d_model,
                                                      y, 2LL * B * (S_total / std::max(1, c->comm ? c->comm->world : 1)) * c->dims.d_model)))
    return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_prefill: x and y overlap");
  if (!c->w) return fail(ZDC_ERR_STATE, "zdc_sp_prefill: ctx not bound");
  if (c->kv_fp8) return fail(ZDC_ERR_UNSUPPORTED, "zdc_sp_prefill: the FP8 cache (kv_fp8) is single-GPU");
  if (!c->comm) return fail(ZDC_ERR_STATE, "zdc_sp_prefill: zdc_comm_init not called");
  if (l0 < 0 || l1 > c->dims.n_layers || l0 >= l1)
    return fail(ZDC_ERR_SHAPE, "zdc_sp_prefill: layer range [%d, %d)", l0, l1);
  const int P = c->comm->world, p = c->comm->rank;
  if (layout < 0 || layout > 2) return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_prefill: layout %d", layout);
  const int parts = layout >= 1 ? 2 * P : P;
  if (B <= 0 || S_total <= 0 || S_total % parts != 0)
    return fail(ZDC_ERR_SHAPE, "zdc_sp_prefill: S_total %d not divisible by %d (%s layout)", S_total, parts,
                layout >= 1 ? "zigzag" : "contiguous");
  const int n_local = S_total / P;
  const int chunk = S_total / parts;
  if (P > 1 && chunk % 128 != 0)
    return fail(ZDC_ERR_UNSUPPORTED, "zdc_sp_prefill: sequence chunk %d is not a multiple of the 128-key tile", chunk);
  if (B > c->max_batch || S_total > c->max_seq)
    return fail(ZDC_ERR_CAPACITY, "zdc_sp_prefill: B=%d S_total=%d exceeds max_batch=%d max_seq=%d", B, S_total,
                c->max_batch, c->max_seq);
  const bool overlap = layout == 2 && P > 1;  // half-major gather buffer, exchange on the comm stream
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& L = c->layers[l];
    if (layout == 2 && L.split)
      return fail(ZDC_ERR_UNSUPPORTED, "zdc_sp_prefill: layout 2 (overlapped exchange) with a token split (layer %d)", l);
    if (L.evict) return fail(ZDC_ERR_UNSUPPORTED, "zdc_sp_prefill: eviction (r_unimp = 0) under SP (layer %d)", l);
    // a layer reusing classes needs its representative classified by an SP prefill of this prompt
    if (L.split && L.rep != l && L.rep < l0 && c->sp_layer[L.rep] != 1)
      return fail(ZDC_ERR_STATE, "zdc_sp_prefill: layer %d: representative %d has not classified this prompt", l, L.rep);
    if (c->len[l] != 0) return fail(ZDC_ERR_STATE, "zdc_sp_prefill: layer %d cache is not empty", l);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int d = c->dims.d_model, Nh = c->dims.n_heads, Nkv = c->dims.n_kv_heads;
  const int M = B * n_local;
  g_launches = 0;
  float exch_ms = 0.f;
  int64_t bytes_recv = 0, bytes_recv_unc = 0;
  cudaEvent_t t_begin = nullptr, t_end = nullptr;
  std::vector<cudaEvent_t> ev;  // exchange brackets, read after the loop (no per-layer host sync)
  auto mark = [&]() -> cudaError_t {
    cudaEvent_t e;
    cudaError_t r = cudaEventCreate(&e);
    if (r == cudaSuccess) r = cudaEventRecord(e, s);
    ev.push_back(e);
    return r;
  };
  if (stats) {
    ZDC_CUDA_TRY(cudaEventCreate(&t_begin));
    ZDC_CUDA_TRY(cudaEventCreate(&t_end));
    ZDC_CUDA_TRY(cudaEventRecord(t_begin, s));
  }
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& L = c->layers[l];
    const LayerInfo& R = c->layers[L.rep];
    const bool split_rep = L.split && L.rep == l, split_other = L.split && L.rep != l;
    const uint8_t* rep_cls = c->cache + R.cls_off;  // [B][max_seq] classes of the group (global positions)
    const uint16_t* xin = l == l0 ? x : y;
    uint16_t* gbuf = reinterpret_cast<uint16_t*>(c->cache + L.k_off);  // [P][K|V][B][Nkv][n_local][r]
    const int64_t slot_rows = static_cast<int64_t>(B) * Nkv * n_local;
    const int64_t chunk_elems = 2 * slot_rows * L.rk_p;
    // a1 + a2: epilogue writes this rank's K'/V' slot of the gather buffer
    Epilogue e1;
    e1.mode = 1;
    QkvDest& q = e1.qkv;
    q.q = reinterpret_cast<uint16_t*>(c->scratch + c->s_q);
    q.ldq = L.nq;
    q.nq = L.nq;
    q.nk = L.nk;
    q.k = gbuf + p * chunk_elems;
    q.v = q.k + slot_rows * L.rk_p;
    q.rk = L.rk_p;
    q.rv = L.rv_p;
    q.S = n_local;
    q.kg = static_cast<int64_t>(n_local) * L.rk_p;
    q.kb = q.kg * Nkv;
    q.vg = static_cast<int64_t>(n_local) * L.rv_p;
    q.vb = q.vg * Nkv;
    q.pos0 = 0;
    g_prof_class = kProfGemmQkv;
    if (overlap) {
      // layout 2: the gather buffer is half-major [2][P][K|V][B][Nkv][chunk][r]; the a1 rows of each
      // local chunk (half h) go to block (h, p), and each half is all-gathered on the comm stream as
      // soon as its rows exist: half 0 (the first P chunks, every key of the local early chunk's
      // queries) overlaps the second half's a1; half 1 overlaps the early chunk's attention
      ZDC_CUDA_TRY(comm_stream(c->comm));
      const int64_t bnc = static_cast<int64_t>(B) * Nkv * chunk;
      const int64_t half_elems = static_cast<int64_t>(P) * 2 * bnc * L.rk_p;
      const int64_t hchunk_bytes = 2 * bnc * L.rk_p * 2;
      for (int h = 0; h < 2; ++h) {
        for (int b = 0; b < B; ++b) {
          Epilogue eh = e1;
          QkvDest& qh = eh.qkv;
          qh.q = q.q + (static_cast<int64_t>(b) * n_local + h * chunk) * L.nq;
          qh.k = gbuf + h * half_elems + p * 2 * bnc * L.rk_p + static_cast<int64_t>(b) * Nkv * chunk * L.rk_p;
          qh.v = qh.k + bnc * L.rk_p;
          qh.S = chunk;
          qh.kg = static_cast<int64_t>(chunk) * L.rk_p;
          qh.kb = qh.kg * Nkv;
          qh.vg = static_cast<int64_t>(chunk) * L.rv_p;
          qh.vb = qh.vg * Nkv;
          ZDC_CUDA_TRY(launch_gemm(xin + (static_cast<int64_t>(b) * n_local + h * chunk) * d, d,
                                   reinterpret_cast<const uint16_t*>(c->w + L.w_qkv), d, chunk, L.n_qkv, d, eh, s));
        }
        ZDC_CUDA_TRY(cudaEventRecord(c->comm->e_a1[h], s));
        ZDC_CUDA_TRY(cudaStreamWaitEvent(c->comm->cs, c->comm->e_a1[h], 0));
        if (stats) {
          cudaEvent_t e;
          ZDC_CUDA_TRY(cudaEventCreate(&e));
          ZDC_CUDA_TRY(cudaEventRecord(e, c->comm->cs));
          ev.push_back(e);
        }
        if (zdc_status st = sp_allgather(c, reinterpret_cast<uint8_t*>(gbuf + h * half_elems), hchunk_bytes, c->comm->cs))
          return st;
        if (stats) {
          cudaEvent_t e;
          ZDC_CUDA_TRY(cudaEventCreate(&e));
          ZDC_CUDA_TRY(cudaEventRecord(e, c->comm->cs));
          ev.push_back(e);
        }
        ZDC_CUDA_TRY(cudaEventRecord(c->comm->e_ag[h], c->comm->cs));
      }
      g_prof_class = kProfOther;
      bytes_recv += (P - 1) * 2 * hchunk_bytes;
      bytes_recv_unc += (P - 1) * 2 * slot_rows * c->dims.d_head * 2;
      for (int sg = 0; sg < 2; ++sg) {  // the early chunk needs half 0 only; the late chunk both
        ZDC_CUDA_TRY(cudaStreamWaitEvent(s, c->comm->e_ag[sg], 0));
        PrefillAttnArgs a;
        a.q = reinterpret_cast<const uint16_t*>(c->scratch + c->s_q);
        a.ldq = L.nq;
        a.k = gbuf;
        a.v = gbuf;
        a.kv_mode = 2;
        a.sp_P = P;
        a.sp_n_local = n_local;
        a.sp_chunk = chunk;
        a.sp_zigzag = 1;
        a.v_row_off = bnc;
        a.kv_rows_total = static_cast<int64_t>(P) * 2 * slot_rows;
        a.S_cap = n_local;
        a.o = reinterpret_cast<uint16_t*>(c->scratch + c->s_o);
        a.ldo = L.ko_p;
        a.lse = reinterpret_cast<float*>(c->scratch + c->s_lse);
        a.B = B;
        a.S = n_local;
        a.Nh = Nh;
        a.Nkv = Nkv;
        a.rk = L.rk_p;
        a.rv = L.rv_p;
        a.scale = 1.0f / std::sqrt(static_cast<float>(c->dims.d_head));
        a.q_row0 = sg * chunk;
        a.n_q = chunk;
        a.q_pos0 = sp_position(S_total, P, p, 1, a.q_row0);
        ZDC_CUDA_TRY(launch_prefill_attention(a, s));
      }
      Epilogue e5o;
      e5o.mode = 0;
      e5o.d = y;
      e5o.ldd = d;
      g_prof_class = kProfGemmO;
      ZDC_CUDA_TRY(launch_gemm(reinterpret_cast<const uint16_t*>(c->scratch + c->s_o), L.ko_p,
                               reinterpret_cast<const uint16_t*>(c->w + L.w_o), L.ko_p, M, d, L.ko_p, e5o, s));
      g_prof_class = kProfOther;
      c->len[l] = S_total;
      c->sp_layer[l] = 3;
      c->sp_prompt[l] = S_total;
      c->last_layer = l;
      c->last_T = n_local;
      continue;
    }
    ZDC_CUDA_TRY(launch_gemm(xin, d, reinterpret_cast<const uint16_t*>(c->w + L.w_qkv), d, M, L.n_qkv, d, e1, s));
    // a layer that reuses its representative's classes: unimportant rows of this rank's slot lose
    // dims >= r^u BEFORE the exchange and the attention (P:774-776 DEL; reading c13)
    if (split_other)
      ZDC_CUDA_TRY(launch_sp_truncate(gbuf, p, p + 1, P, layout, S_total, B, Nkv, n_local, L.rk_p, L.rku, rep_cls,
                                      c->max_seq, s));
    // a6: in-place all-gather of the compressed K'/V' slots
    const int64_t chunk_bytes = chunk_elems * 2;
    if (P > 1) {
      if (stats) ZDC_CUDA_TRY(mark());
      if (zdc_status st = sp_allgather(c, reinterpret_cast<uint8_t*>(gbuf), chunk_bytes, s)) return st;
      if (stats) ZDC_CUDA_TRY(mark());
      bytes_recv += (P - 1) * chunk_bytes;
      bytes_recv_unc += (P - 1) * 2 * slot_rows * c->dims.d_head * 2;
    }
    // a3: local query segments against every earlier key in the gathered buffer
    const int segs = layout == 1 ? 2 : 1;
    for (int sg = 0; sg < segs; ++sg) {
      PrefillAttnArgs a;
      a.q = reinterpret_cast<const uint16_t*>(c->scratch + c->s_q);
      a.ldq = L.nq;
      a.k = gbuf;
      a.v = gbuf;
      a.kv_mode = 1;
      a.sp_P = P;
      a.sp_n_local = n_local;
      a.sp_chunk = chunk;
      a.sp_zigzag = layout;
      a.v_row_off = slot_rows;
      a.kv_rows_total = static_cast<int64_t>(P) * 2 * slot_rows;
      a.S_cap = n_local;
      a.o = reinterpret_cast<uint16_t*>(c->scratch + c->s_o);
      a.ldo = L.ko_p;
      a.lse = reinterpret_cast<float*>(c->scratch + c->s_lse);
      a.B = B;
      a.S = n_local;
      a.Nh = Nh;
      a.Nkv = Nkv;
      a.rk = L.rk_p;
      a.rv = L.rv_p;
      a.scale = 1.0f / std::sqrt(static_cast<float>(c->dims.d_head));
      a.q_row0 = sg * chunk;
      a.n_q = layout == 1 ? chunk : n_local;
      a.q_pos0 = sp_position(S_total, P, p, layout, a.q_row0);
      ZDC_CUDA_TRY(launch_prefill_attention(a, s));
    }
    if (split_rep) {
      // a4 under SP (NEXT-2): scores of the local rows -> all-gather -> the same global top-g
      // selection on every rank (identical inputs, deterministic select) -> truncate the stored rows
      float* slots = reinterpret_cast<float*>(c->scratch + c->s_sp);  // [P][B][n_local]
      const int64_t sc_chunk = static_cast<int64_t>(B) * n_local * 4;
      ZDC_CUDA_TRY(launch_sp_importance(reinterpret_cast<const float*>(c->scratch + c->s_lse), n_local, Nh, B,
                                        c->importance_mode, S_total, P, p, layout,
                                        slots + static_cast<int64_t>(p) * B * n_local, s));
      if (P > 1) {
        if (stats) ZDC_CUDA_TRY(mark());
        if (zdc_status st = sp_allgather(c, reinterpret_cast<uint8_t*>(slots), sc_chunk, s)) return st;
        if (stats) ZDC_CUDA_TRY(mark());
        bytes_recv += (P - 1) * sc_chunk;
        bytes_recv_unc += (P - 1) * sc_chunk;
      }
      float* scores = reinterpret_cast<float*>(c->cache + L.score_off);
      ZDC_CUDA_TRY(launch_sp_scores_global(slots, P, B, n_local, S_total, layout, scores, c->max_seq, s));
      ZDC_CUDA_TRY(launch_select(scores, c->max_seq, S_total, L.g_bp, B, c->cache + L.cls_off,
                                 reinterpret_cast<float*>(c->cache + L.tau_off), s, c->len_dev() + c->dims.n_layers + 1));
      ZDC_CUDA_TRY(launch_sp_truncate(gbuf, 0, P, P, layout, S_total, B, Nkv, n_local, L.rk_p, L.rku,
                                      c->cache + L.cls_off, c->max_seq, s));
    }
    // a5
    Epilogue e5;
    e5.mode = 0;
    e5.d = y;
    e5.ldd = d;
    g_prof_class = kProfGemmO;
    ZDC_CUDA_TRY(launch_gemm(reinterpret_cast<const uint16_t*>(c->scratch + c->s_o), L.ko_p,
                             reinterpret_cast<const uint16_t*>(c->w + L.w_o), L.ko_p, M, d, L.ko_p, e5, s));
    g_prof_class = kProfOther;
    c->len[l] = S_total;
    c->sp_layer[l] = 1;
    c->sp_prompt[l] = S_total;
    c->last_layer = l;
    c->last_T = n_local;
  }
  c->batch = B;
  if (stats) {
    ZDC_CUDA_TRY(cudaEventRecord(t_end, s));
    ZDC_CUDA_TRY(cudaEventSynchronize(t_end));
    float tot = 0.f;
    ZDC_CUDA_TRY(cudaEventElapsedTime(&tot, t_begin, t_end));
    cudaEventDestroy(t_begin);
    cudaEventDestroy(t_end);
    for (size_t i = 0; i + 1 < ev.size(); i += 2) {
      float ms = 0.f;
      ZDC_CUDA_TRY(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      exch_ms += ms;
    }
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    stats->bytes_recv = bytes_recv;
    stats->bytes_sent = bytes_recv;  // all-gather: each slot goes to the P-1 peers
    stats->bytes_recv_uncompressed = bytes_recv_unc;
    stats->exchange_ms = exch_ms;
    stats->total_ms = tot;
  }
  return ZDC_OK;
}

// all-to-all of P equal chunks: recv[q] = send_q[p] (chunk q of send goes to rank q)
static zdc_status sp_alltoall(zdc_ctx* c, const uint8_t* send, uint8_t* recv, int64_t chunk, cudaStream_t s) {
  const int P = c->comm->world, p = c->comm->rank;
  if (c->comm->a2a_hook) {
    c->comm->a2a_hook(c->comm->a2a_user, send, recv, chunk, p, P, s);
    return ZDC_OK;
  }
  if (!c->comm->comm) return fail(ZDC_ERR_STATE, "zdc_sp_prefill_ulysses: no NCCL communicator and no all-to-all hook");
  NcclApi* api = nccl_api();
  ZDC_CUDA_TRY(cudaMemcpyAsync(recv + p * chunk, send + p * chunk, static_cast<size_t>(chunk), cudaMemcpyDeviceToDevice, s));
  ncclResult_t r = api->GroupStart();
  for (int q = 0; q < P && r == ncclSuccess; ++q) {
    if (q == p) continue;
    r = api->Send(send + q * chunk, static_cast<size_t>(chunk), ncclUint8, q, c->comm->comm, s);
    if (r == ncclSuccess) r = api->Recv(recv + q * chunk, static_cast<size_t>(chunk), ncclUint8, q, c->comm->comm, s);
  }
  const ncclResult_t r2 = api->GroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return fail(ZDC_ERR_NCCL, "ncclSend/Recv all-to-all: %s", api->GetErrorString(r != ncclSuccess ? r : r2));
  return ZDC_OK;
}

zdc_status zdc_sp_prefill_ulysses(zdc_ctx* c, int32_t l0, int32_t l1, const uint16_t* x, uint16_t* y, int32_t B,
                                  int32_t S_total, int32_t layout, zdc_sp_stats* stats, void* stream) {
  if (!c || !x || !y) return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_prefill_ulysses: null argument");
  if (x == y || (B > 0 && S_total > 0 && ranges_overlap(x, 2LL * B * (S_total / std::max(1, c->comm ? c->comm->world : 1)) * c->dims.d_model,
                                                      y, 2LL * B * (S_total / std::max(1, c->comm ? c->comm->world : 1)) * c->dims.d_model)))
    return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_prefill_ulysses: x and y overlap");
  if (!c->w) return fail(ZDC_ERR_STATE, "zdc_sp_prefill_ulysses: ctx not bound");
  if (c->kv_fp8) return fail(ZDC_ERR_UNSUPPORTED, "zdc_sp_prefill_ulysses: the FP8 cache (kv_fp8) is single-GPU");
  if (!c->comm) return fail(ZDC_ERR_STATE, "zdc_sp_prefill_ulysses: zdc_comm_init / an all-to-all hook not set");
  if (l0 < 0 || l1 > c->dims.n_layers || l0 >= l1)
    return fail(ZDC_ERR_SHAPE, "zdc_sp_prefill_ulysses: layer range [%d, %d)", l0, l1);
  const int P = c->comm->world, p = c->comm->rank;
  const int d = c->dims.d_model, Nh = c->dims.n_heads, Nkv = c->dims.n_kv_heads;
  if (layout != 0 && layout != 1) return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_prefill_ulysses: layout %d", layout);
  if (Nkv % P != 0)
    return fail(ZDC_ERR_SHAPE, "zdc_sp_prefill_ulysses: N_kv = %d KV heads do not split over P = %d ranks", Nkv, P);
  const int parts = layout == 1 ? 2 * P : P;
  if (B <= 0 || S_total <= 0 || S_total % parts != 0)
    return fail(ZDC_ERR_SHAPE, "zdc_sp_prefill_ulysses: S_total %d not divisible by %d (%s layout)", S_total, parts,
                layout == 1 ? "zigzag" : "contiguous");
  if (B > c->max_batch || S_total > c->max_seq)
    return fail(ZDC_ERR_CAPACITY, "zdc_sp_prefill_ulysses: B=%d S_total=%d exceeds max_batch=%d max_seq=%d", B,
                S_total, c->max_batch, c->max_seq);
  for (int l = l0; l < l1; ++l) {
    if (c->layers[l].split)
      return fail(ZDC_ERR_UNSUPPORTED, "zdc_sp_prefill_ulysses: token split under SP is NEXT-2 (layer %d)", l);
    if (c->len[l] != 0) return fail(ZDC_ERR_STATE, "zdc_sp_prefill_ulysses: layer %d cache is not empty", l);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n_local = S_total / P;
  const int M = B * n_local;
  const int hpr = Nh / P, gpr = Nkv / P;  // heads / KV groups per rank
  g_launches = 0;
  float exch_ms = 0.f;
  int64_t bytes_recv = 0, bytes_recv_unc = 0;
  cudaEvent_t t_begin = nullptr, t_end = nullptr;
  std::vector<cudaEvent_t> ev;  // exchange brackets, read after the loop (no per-layer host sync)
  auto mark = [&](std::vector<cudaEvent_t>& v) -> cudaError_t {
    cudaEvent_t e;
    cudaError_t r = cudaEventCreate(&e);
    if (r == cudaSuccess) r = cudaEventRecord(e, s);
    v.push_back(e);
    return r;
  };
  if (stats) {
    ZDC_CUDA_TRY(cudaEventCreate(&t_begin));
    ZDC_CUDA_TRY(cudaEventCreate(&t_end));
    ZDC_CUDA_TRY(cudaEventRecord(t_begin, s));
  }
  uint8_t* sp = c->scratch + c->s_sp;
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& L = c->layers[l];
    const uint16_t* xin = l == l0 ? x : y;
    const int hq = hpr * L.rk_p, kq = gpr * L.rk_p, vq = gpr * L.rv_p, cols = hq + kq + vq;
    const int ho = hpr * L.rv_p;
    const int64_t chunk1 = static_cast<int64_t>(M) * cols * 2, chunk2 = static_cast<int64_t>(M) * ho * 2;
    uint8_t* send = sp;
    uint8_t* recv = P > 1 ? sp + P * chunk1 : sp;  // one rank: nothing moves
    // a1: compressed Q'/K'/V' of the local tokens, written as per-destination slabs (epilogue mode 2)
    Epilogue e1;
    e1.mode = 2;
    e1.uly.send = reinterpret_cast<uint16_t*>(send);
    e1.uly.nq = L.nq;
    e1.uly.nk = L.nk;
    e1.uly.hq = hq;
    e1.uly.kq = kq;
    e1.uly.vq = vq;
    e1.uly.cols = cols;
    e1.uly.rows = M;
    g_prof_class = kProfGemmQkv;
    ZDC_CUDA_TRY(launch_gemm(xin, d, reinterpret_cast<const uint16_t*>(c->w + L.w_qkv), d, M, L.n_qkv, d, e1, s));
    g_prof_class = kProfOther;
    // all-to-all #1: tokens gathered along the sequence, heads distributed (compressed bytes)
    if (P > 1) {
      if (stats) ZDC_CUDA_TRY(mark(ev));
      if (zdc_status st = sp_alltoall(c, send, recv, chunk1, s)) return st;
      if (stats) ZDC_CUDA_TRY(mark(ev));
    }
    // this rank's heads for all S tokens: Q' in position order, K'/V' into its groups' cache
    uint16_t* qpos = reinterpret_cast<uint16_t*>(c->scratch + c->s_q);
    uint16_t* kc = reinterpret_cast<uint16_t*>(c->cache + L.k_off);
    uint16_t* vc = reinterpret_cast<uint16_t*>(c->cache + L.v_off);
    ZDC_CUDA_TRY(launch_ulysses_unpack_qkv(reinterpret_cast<const uint16_t*>(recv), P, B, n_local, S_total, layout, hq,
                                           kq, vq, L.rk_p, L.rv_p, qpos, kc, vc, c->max_seq, s));
    // a3: ordinary causal attention over the full sequence for the rank's N_h/P heads
    uint16_t* opos = reinterpret_cast<uint16_t*>(c->scratch + c->s_o);
    PrefillAttnArgs a;
    a.q = qpos;
    a.ldq = hq;
    a.k = kc;
    a.v = vc;
    a.S_cap = c->max_seq;
    a.o = opos;
    a.ldo = ho;
    a.lse = reinterpret_cast<float*>(c->scratch + c->s_lse);
    a.B = B;
    a.S = S_total;
    a.Nh = hpr;
    a.Nkv = gpr;
    a.rk = L.rk_p;
    a.rv = L.rv_p;
    a.scale = 1.0f / std::sqrt(static_cast<float>(c->dims.d_head));
    a.q_pos0 = 0;
    a.q_row0 = 0;
    a.n_q = S_total;
    g_prof_class = kProfAttnPrefill;
    ZDC_CUDA_TRY(launch_prefill_attention(a, s));
    g_prof_class = kProfOther;
    // all-to-all #2: O' back to the token owners (heads gathered, sequence split)
    ZDC_CUDA_TRY(launch_ulysses_pack_o(opos, P, B, n_local, S_total, layout, ho, reinterpret_cast<uint16_t*>(send), s));
    if (P > 1) {
      if (stats) ZDC_CUDA_TRY(mark(ev));
      if (zdc_status st = sp_alltoall(c, send, recv, chunk2, s)) return st;
      if (stats) ZDC_CUDA_TRY(mark(ev));
    }
    // O'_local [M][ko_p] reuses the position-ordered O' region (dead once packed into the send slabs)
    uint16_t* oloc = opos;
    ZDC_CUDA_TRY(launch_ulysses_unpack_o(reinterpret_cast<const uint16_t*>(recv), P, B, n_local, ho, oloc, L.ko_p, s));
    // a5: y_local = O'_local W_O^R
    Epilogue e5;
    e5.mode = 0;
    e5.d = y;
    e5.ldd = d;
    g_prof_class = kProfGemmO;
    ZDC_CUDA_TRY(launch_gemm(oloc, L.ko_p, reinterpret_cast<const uint16_t*>(c->w + L.w_o), L.ko_p, M, d, L.ko_p, e5, s));
    g_prof_class = kProfOther;
    if (P > 1) {
      bytes_recv += (P - 1) * (chunk1 + chunk2);
      const int64_t cols_u = static_cast<int64_t>(hpr + 2 * gpr) * c->dims.d_head;  // uncompressed Q/K/V columns
      bytes_recv_unc += (P - 1) * (static_cast<int64_t>(M) * cols_u * 2 + static_cast<int64_t>(M) * hpr * c->dims.d_head * 2);
    }
    c->len[l] = S_total;
    c->sp_layer[l] = 2;
    c->last_layer = l;
    c->last_T = S_total;
  }
  c->batch = B;
  if (stats) {
    ZDC_CUDA_TRY(cudaEventRecord(t_end, s));
    ZDC_CUDA_TRY(cudaEventSynchronize(t_end));
    float tot = 0.f;
    ZDC_CUDA_TRY(cudaEventElapsedTime(&tot, t_begin, t_end));
    for (size_t i = 0; i + 1 < ev.size(); i += 2) {
      float ms = 0.f;
      ZDC_CUDA_TRY(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      exch_ms += ms;
    }
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    cudaEventDestroy(t_begin);
    cudaEventDestroy(t_end);
    stats->bytes_recv = bytes_recv;
    stats->bytes_sent = bytes_recv;  // all-to-all: every rank sends what its peers receive from it
    stats->bytes_recv_uncompressed = bytes_recv_unc;
    stats->exchange_ms = exch_ms;
    stats->total_ms = tot;
  }
  return ZDC_OK;
}

zdc_status zdc_sp_decode(zdc_ctx* c, int32_t l0, int32_t l1, const uint16_t* x, uint16_t* y, int32_t B, void* stream) {
  if (!c || !x || !y) return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_decode: null argument");
  if (x == y || (B > 0 && ranges_overlap(x, 2LL * B * c->dims.d_model, y, 2LL * B * c->dims.d_model)))
    return fail(ZDC_ERR_INVALID_ARG, "zdc_sp_decode: x and y overlap");
  if (!c->w || !c->comm) return fail(ZDC_ERR_STATE, "zdc_sp_decode: ctx not bound / no communicator");
  if (l0 < 0 || l1 > c->dims.n_layers || l0 >= l1) return fail(ZDC_ERR_SHAPE, "zdc_sp_decode: layer range [%d, %d)", l0, l1);
  if (B != c->batch) return fail(ZDC_ERR_SHAPE, "zdc_sp_decode: B=%d but the SP prefill had B=%d", B, c->batch);
  const int P = c->comm->world, p = c->comm->rank;
  const int d = c->dims.d_model, Nh = c->dims.n_heads, Nkv = c->dims.n_kv_heads;
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& L = c->layers[l];
    if (c->sp_layer[l] != 1)
      return fail(ZDC_ERR_STATE, "zdc_sp_decode: layer %d was not prefilled by zdc_sp_prefill (all-gather)", l);
    if (L.split) return fail(ZDC_ERR_UNSUPPORTED, "zdc_sp_decode: layer %d has a token split", l);
    const int S = c->sp_prompt[l], n_local = S / P, j = c->len[l] - S;
    // this rank's decode tail has n_local rows per (sequence, KV head), after the gather buffer
    if (j / P + 1 > n_local || S + n_local > c->max_seq)
      return fail(ZDC_ERR_CAPACITY, "zdc_sp_decode: layer %d: decode token %d exceeds the sharded tail (%d rows per rank, "
                  "max_seq >= S + S/P needed)", l, j, n_local);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  g_launches = 0;
  uint8_t* sp = c->scratch + c->s_sp;
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& L = c->layers[l];
    const uint16_t* xin = l == l0 ? x : y;
    const int S = c->sp_prompt[l], n_local = S / P, j = c->len[l] - S;
    const int owner = j % P, own_before = (j + P - 1 - p) / P;  // decode tokens this rank held before
    const int64_t slot_rows = static_cast<int64_t>(B) * Nkv * n_local;
    uint16_t* gbuf = reinterpret_cast<uint16_t*>(c->cache + L.k_off);
    uint16_t* tail_k = gbuf + 2 * static_cast<int64_t>(P) * slot_rows * L.rk_p;  // [B][Nkv][n_local][r]
    uint16_t* tail_v = tail_k + slot_rows * L.rk_p;
    // scratch: per-sequence pool counts, the new K'/V' rows, the exchanged partials
    int* n0 = reinterpret_cast<int*>(sp);
    int* n1 = n0 + B;
    uint16_t* knew = reinterpret_cast<uint16_t*>(sp + 4096);
    uint16_t* vnew = knew + static_cast<int64_t>(B) * Nkv * L.rk_p;
    float* parts = reinterpret_cast<float*>(sp + 4096 + 4 * static_cast<int64_t>(B) * Nkv * L.rk_p + 4096);
    // a1 (replicated: every rank has the weights): Q' to staging, the new K'/V' rows to knew/vnew
    Epilogue e1;
    e1.mode = 1;
    QkvDest& q = e1.qkv;
    q.q = reinterpret_cast<uint16_t*>(c->scratch + c->s_q);
    q.ldq = L.nq;
    q.nq = L.nq;
    q.nk = L.nk;
    q.k = knew;
    q.v = vnew;
    q.rk = L.rk_p;
    q.rv = L.rv_p;
    q.S = 1;
    q.kg = L.rk_p;
    q.kb = static_cast<int64_t>(Nkv) * L.rk_p;
    q.vg = L.rv_p;
    q.vb = static_cast<int64_t>(Nkv) * L.rv_p;
    q.pos0 = 0;
    const uint16_t* wqkv = reinterpret_cast<const uint16_t*>(c->w + L.w_qkv);
    if (gemv_supported(B, d))
      ZDC_CUDA_TRY(launch_gemv(wqkv, xin, d, B, L.n_qkv, d, e1, s));
    else
      ZDC_CUDA_TRY(launch_gemm(xin, d, wqkv, d, B, L.n_qkv, d, e1, s));
    // a2: the owner appends the new token to its tail (decode token j -> rank j mod P)
    const int own_now = own_before + (owner == p ? 1 : 0);
    if (owner == p) {
      ZDC_CUDA_TRY(cudaMemcpy2DAsync(tail_k + static_cast<int64_t>(own_before) * L.rk_p, n_local * L.rk_p * 2, knew,
                                     L.rk_p * 2, L.rk_p * 2, static_cast<size_t>(B) * Nkv, cudaMemcpyDeviceToDevice, s));
      ZDC_CUDA_TRY(cudaMemcpy2DAsync(tail_v + static_cast<int64_t>(own_before) * L.rv_p, n_local * L.rv_p * 2, vnew,
                                     L.rv_p * 2, L.rv_p * 2, static_cast<size_t>(B) * Nkv, cudaMemcpyDeviceToDevice, s));
    }
    std::vector<int> hcnt(2 * B);
    for (int b = 0; b < B; ++b) {
      hcnt[b] = n_local;
      hcnt[B + b] = own_now;
    }
    ZDC_CUDA_TRY(cudaMemcpyAsync(n0, hcnt.data(), 2 * B * sizeof(int), cudaMemcpyHostToDevice, s));
    // a3 over this rank's keys: pool 0 = its prompt slot, pool 1 = the decode rows it owns
    DecodeAttnArgs a;
    a.q = reinterpret_cast<const uint16_t*>(c->scratch + c->s_q);
    a.ldq = L.nq;
    a.k = gbuf + static_cast<int64_t>(p) * 2 * slot_rows * L.rk_p;
    a.v = a.k + slot_rows * L.rk_p;
    a.rk = L.rk_p;
    a.rv = L.rv_p;
    a.k1 = tail_k;
    a.v1 = tail_v;
    a.rk1 = L.rk_p;
    a.rv1 = L.rv_p;
    a.S_cap = n_local;
    a.len = n_local;
    a.n0_ptr = n0;
    a.n1_ptr = n1;
    a.o = reinterpret_cast<uint16_t*>(c->scratch + c->s_o);
    a.ldo = L.ko_p;
    a.lse = reinterpret_cast<float*>(c->scratch + c->s_lse);
    a.part = reinterpret_cast<float*>(c->scratch + c->s_part);
    a.counters = reinterpret_cast<int*>(c->scratch + c->s_cnt);
    a.B = B;
    a.Nh = Nh;
    a.Nkv = Nkv;
    a.scale = 1.0f / std::sqrt(static_cast<float>(c->dims.d_head));
    a.splits = decode_splits(B, Nkv, n_local);
    ZDC_CUDA_TRY(launch_decode_attention(a, s));
    // exchange {O'_p, LSE_p} and merge over the ranks (the LSE merge of P:254-260's softmax)
    const int64_t chunk = static_cast<int64_t>(B) * Nh * (L.rv_p + 1) * 4;
    ZDC_CUDA_TRY(launch_sp_decode_pack(a.o, L.ko_p, a.lse, B, Nh, L.rv_p,
                                       parts + static_cast<int64_t>(p) * B * Nh * (L.rv_p + 1), s));
    if (P > 1)
      if (zdc_status st = sp_allgather(c, reinterpret_cast<uint8_t*>(parts), chunk, s)) return st;
    ZDC_CUDA_TRY(launch_sp_decode_merge(parts, P, B, Nh, L.rv_p, a.o, L.ko_p, a.lse, s));
    // a5 (replicated)
    Epilogue e5;
    e5.mode = 0;
    e5.d = y;
    e5.ldd = d;
    const uint16_t* wo = reinterpret_cast<const uint16_t*>(c->w + L.w_o);
    if (gemv_supported(B, L.ko_p))
      ZDC_CUDA_TRY(launch_gemv(wo, a.o, L.ko_p, B, d, L.ko_p, e5, s));
    else
      ZDC_CUDA_TRY(launch_gemm(a.o, L.ko_p, wo, L.ko_p, B, d, L.ko_p, e5, s));
    c->len[l] += 1;
    c->last_layer = l;
    c->last_T = 1;
  }
  return ZDC_OK;
}

}  // extern "C"
