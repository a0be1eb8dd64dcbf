"""Python binding of libzdc.so (include/zdc.h) — argument marshalling only.

Every step of the ZDC hot path runs in the library's sm_100a kernels; this module only
converts arguments (torch device tensors / numpy host arrays -> pointers) and raises
ZdcError on a non-zero status.  There is no CPU fallback: importing works without a GPU,
but any call that needs the device fails loudly if libzdc.so or the GPU is missing.
PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

__all__ = ["ZdcError", "lib", "lib_path", "Dims", "Plan", "Context", "fold_weights", "gemm_bf16",
           "sp_positions", "EXPORTED_SYMBOLS", "last_launch_count", "decode_mode"]

_HERE = os.path.dirname(os.path.abspath(__file__))
# ZDC_LIB_PATH: an alternative in-tree build of the same library (same-box A/B of kernel variants)
_LIB_PATH = os.environ.get("ZDC_LIB_PATH") or os.path.join(_HERE, "libzdc.so")
_lib = None

ZDC_STATUS = {0: "ZDC_OK", -1: "ZDC_ERR_INVALID_ARG", -2: "ZDC_ERR_SHAPE", -3: "ZDC_ERR_NOT_ORTHONORMAL",
              -4: "ZDC_ERR_NO_CONVERGENCE", -5: "ZDC_ERR_CAPACITY", -6: "ZDC_ERR_CUDA", -7: "ZDC_ERR_NCCL",
              -8: "ZDC_ERR_UNSUPPORTED", -9: "ZDC_ERR_STATE"}

EXPORTED_SYMBOLS = ["zdc_last_error", "zdc_version", "zdc_fold_weights", "zdc_ctx_create", "zdc_ctx_sizes",
                    "zdc_ctx_bind", "zdc_ctx_destroy", "zdc_load_folded", "zdc_load_folded_device",
                    "zdc_prefill", "zdc_decode", "zdc_comm_unique_id", "zdc_comm_init",
                    "zdc_sp_set_exchange_hook", "zdc_sp_prefill", "zdc_sp_positions",
                    "zdc_sp_prefill_ulysses", "zdc_sp_set_alltoall_hook",
                    "zdc_fold_gpu_workspace", "zdc_fold_weights_gpu", "zdc_layer_groups", "zdc_sp_decode",
                    "zdc_cache_export", "zdc_cache_length", "zdc_cache_sync", "zdc_scores_export", "zdc_cache_reset", "zdc_last_lse",
                    "zdc_gemm_bf16", "zdc_gemv_bf16", "zdc_prefill_attention_bf16",
                    "zdc_decode_attention_workspace", "zdc_decode_attention_bf16",
                    "zdc_kernel_launch_count", "zdc_profile", "zdc_profile_read", "zdc_trace_read",
                    "zdc_decode_mode"]


class ZdcError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        self.status = status
        super().__init__("%s -> %s: %s" % (fn, ZDC_STATUS.get(status, status), msg))


class Dims(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("d_model", ctypes.c_int32), ("n_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("d_head", ctypes.c_int32)]


class Plan(ctypes.Structure):
    _fields_ = [("r_qk_imp", ctypes.POINTER(ctypes.c_int32)), ("r_qk_unimp", ctypes.POINTER(ctypes.c_int32)),
                ("r_vl_imp", ctypes.POINTER(ctypes.c_int32)), ("r_vl_unimp", ctypes.POINTER(ctypes.c_int32)),
                ("g_bp", ctypes.POINTER(ctypes.c_int32)), ("group_rep", ctypes.POINTER(ctypes.c_int32)),
                ("importance_mode", ctypes.c_int32), ("kv_fp8", ctypes.c_int32)]


class SpStats(ctypes.Structure):
    _fields_ = [("bytes_sent", ctypes.c_int64), ("bytes_recv", ctypes.c_int64),
                ("bytes_recv_uncompressed", ctypes.c_int64), ("exchange_ms", ctypes.c_float),
                ("total_ms", ctypes.c_float)]


# test transport of zdc_sp_set_exchange_hook: fn(user, gather_buf, chunk_bytes, rank, world, stream)
EXCHANGE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                               ctypes.c_int32, ctypes.c_void_p)
# test transport of zdc_sp_set_alltoall_hook: fn(user, send, recv, chunk_bytes, rank, world, stream)
ALLTOALL_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                               ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p)


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """Load libzdc.so (built in-tree by paper_2408_04107_b200.build).  Raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError("libzdc.so not built: run `python -m paper_2408_04107_b200.build` "
                              "(no CPU fallback exists)")
        L = ctypes.CDLL(_LIB_PATH)
        P, I32, I64, F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        dp = ctypes.POINTER(ctypes.c_double)
        sig = {
            "zdc_last_error": ([], ctypes.c_char_p), "zdc_version": ([], ctypes.c_char_p),
            "zdc_fold_weights": ([ctypes.POINTER(Dims), dp, dp, dp, dp, dp, I64, dp, dp, dp, dp, dp, dp, dp, dp], I32),
            "zdc_ctx_create": ([ctypes.POINTER(Dims), ctypes.POINTER(Plan), I32, I32, ctypes.POINTER(P)], I32),
            "zdc_fold_gpu_workspace": ([ctypes.POINTER(Dims), I64, I32], I64),
            "zdc_layer_groups": ([P, I32, I64, I32, ctypes.POINTER(I32)], I32),
            "zdc_fold_weights_gpu": ([ctypes.POINTER(Dims)] + [P] * 5 + [I64, I32, I32] + [P] * 8 + [P, I64, P], I32),
            "zdc_ctx_sizes": ([P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)], I32),
            "zdc_ctx_bind": ([P, P, P, P], I32), "zdc_ctx_destroy": ([P], None),
            "zdc_load_folded": ([P, I32, dp, dp, dp, dp, P], I32),
            "zdc_load_folded_device": ([P, I32, P, P, P, P, P], I32),
            "zdc_prefill": ([P, I32, I32, P, P, I32, I32, P, P], I32),
            "zdc_decode": ([P, I32, I32, P, P, I32, P], I32),
            "zdc_comm_unique_id": ([P], I32),
            "zdc_comm_init": ([P, P, I32, I32], I32),
            "zdc_sp_set_exchange_hook": ([P, EXCHANGE_FN, P, I32, I32], I32),
            "zdc_sp_prefill": ([P, I32, I32, P, P, I32, I32, I32, ctypes.POINTER(SpStats), P], I32),
            "zdc_sp_prefill_ulysses": ([P, I32, I32, P, P, I32, I32, I32, ctypes.POINTER(SpStats), P], I32),
            "zdc_sp_set_alltoall_hook": ([P, ALLTOALL_FN, P, I32, I32], I32),
            "zdc_sp_decode": ([P, I32, I32, P, P, I32, P], I32),
            "zdc_sp_positions": ([I32, I32, I32, I32, ctypes.POINTER(I32)], I32),
            "zdc_cache_export": ([P, I32, P, P, P, P, P], I32),
            "zdc_cache_length": ([P, I32, ctypes.POINTER(I32)], I32),
            "zdc_cache_sync": ([P, P], I32),
            "zdc_scores_export": ([P, I32, P, P], I32),
            "zdc_cache_reset": ([P, P], I32),
            "zdc_last_lse": ([P, I32, P, P], I32),
            "zdc_gemm_bf16": ([P, P, P, I32, I32, I32, P], I32),
            "zdc_gemv_bf16": ([P, P, P, I32, I32, I32, P], I32),
            "zdc_prefill_attention_bf16": ([P, P, P, P, P, I32, I32, I32, I32, I32, F, P], I32),
            "zdc_decode_attention_workspace": ([I32, I32, I32, I32], I64),
            "zdc_decode_attention_bf16": ([P, P, P, P, P, I32, I32, I32, I32, I32, I32, F, P, P], I32),
            "zdc_kernel_launch_count": ([], I64),
            "zdc_profile": ([ctypes.c_int], None),
            "zdc_profile_read": ([ctypes.POINTER(F), ctypes.POINTER(I64), ctypes.c_int], ctypes.c_int),
            "zdc_trace_read": ([ctypes.POINTER(ctypes.c_uint64), ctypes.c_int], ctypes.c_int),
            "zdc_decode_mode": ([ctypes.c_int], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _ = F
        _lib = L
    return _lib


def _check(status: int, fn: str):
    if status != 0:
        raise ZdcError(status, fn, lib().zdc_last_error().decode())


def last_launch_count() -> int:
    return int(lib().zdc_kernel_launch_count())


PROFILE_CLASSES = ["a1_prefill_gemm", "a3_prefill_attention", "a5_prefill_gemm", "a1_decode_gemv",
                   "a3_decode_attention", "a3_decode_combine", "a5_decode_gemv", "other"]


DECODE_MODES = {"auto": 0, "fused": 1, "cluster": 2, "separate": 3}


def decode_mode(mode: str) -> str:
    """Select the decode kernels for B <= 8 uniform-rank layers (zdc_decode_mode); returns the
    previous mode.  Takes effect for decode graphs captured afterwards."""
    old = lib().zdc_decode_mode(DECODE_MODES[mode])
    if old < 0:
        raise ValueError(mode)
    return {v: k for k, v in DECODE_MODES.items()}[old]


def profile(enable: bool):
    """Per-kernel-class CUDA-event timing inside the library (zdc_profile)."""
    lib().zdc_profile(1 if enable else 0)


def trace_read(n_cta: int = 148, launches: int = 16):
    """Fused decode kernel timelines (ZDC_FUSED_TRACE, diagnostic build): uint64 ns stamps
    [launches][n_cta][32] of the last `launches` launches, oldest first (unused slots are 0)."""
    import numpy as np
    per = 1024 * 32
    buf = (ctypes.c_uint64 * (16 * per))()
    got = lib().zdc_trace_read(buf, 16 * per)
    if got <= 0:
        return None
    a = np.frombuffer(buf, dtype=np.uint64).reshape(16, 1024, 32)[:, :n_cta].copy()
    return a[16 - launches:]


def profile_read():
    """{class: (ms_total, launches)} since the previous read (synchronises)."""
    n = len(PROFILE_CLASSES)
    ms = (ctypes.c_float * n)()
    cnt = (ctypes.c_int64 * n)()
    lib().zdc_profile_read(ms, cnt, n)
    return {PROFILE_CLASSES[i]: (float(ms[i]), int(cnt[i])) for i in range(n)}


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i32arr(v: Sequence[int]):
    arr = (ctypes.c_int32 * len(v))(*[int(x) for x in v])
    return arr


def _stream(stream=None) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _tptr(t, dtype_name: str):
    """Device pointer of a contiguous torch tensor of the expected dtype."""
    import torch
    want = {"bf16": torch.bfloat16, "f32": torch.float32, "u16": torch.int16}[dtype_name]
    if t.dtype != want and not (dtype_name == "bf16" and t.dtype == torch.int16):
        raise TypeError("expected %s tensor, got %s" % (dtype_name, t.dtype))
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def make_dims(d) -> Dims:
    return Dims(d.n_layers, d.d_model, d.n_heads, d.n_kv_heads, d.d_head)


def fold_weights(dims, wq, wk, wv, wo, xc):
    """zdc_fold_weights (host fp64, one layer).  Returns dict like the oracle's fold."""
    nkv, dh = dims.n_kv_heads, dims.d_head
    c = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    wq, wk, wv, wo, xc = c(wq), c(wk), c(wv), c(wo), c(xc)
    out = dict(r_qk=np.zeros((nkv, dh, dh)), r_vl=np.zeros((nkv, dh, dh)), sigma_qk=np.zeros((nkv, dh)),
               sigma_vl=np.zeros((nkv, dh)), wq_f=np.zeros_like(wq), wk_f=np.zeros_like(wk),
               wv_f=np.zeros_like(wv), wo_f=np.zeros_like(wo))
    D = make_dims(dims)
    st = lib().zdc_fold_weights(ctypes.byref(D), _dptr(wq), _dptr(wk), _dptr(wv), _dptr(wo), _dptr(xc),
                                xc.shape[0], _dptr(out["r_qk"]), _dptr(out["r_vl"]), _dptr(out["sigma_qk"]),
                                _dptr(out["sigma_vl"]), _dptr(out["wq_f"]), _dptr(out["wk_f"]),
                                _dptr(out["wv_f"]), _dptr(out["wo_f"]))
    _check(st, "zdc_fold_weights")
    return out


def fold_weights_gpu(dims, wq, wk, wv, wo, xc, k_clusters: int = 0, kmeans_iters: int = 0, stream=None,
                     return_device: bool = False):
    """zdc_fold_weights_gpu (NEXT-3): the fold on the GPU in fp64, with optional K-means
    consolidation of the calibration Q / K / V vectors.  Host numpy (or device fp64 torch) inputs;
    returns a dict like fold_weights (numpy, or device tensors with return_device=True)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    t = lambda a: (a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))  # noqa: E731
                   ).to(device=dev, dtype=torch.float64).contiguous()
    wq, wk, wv, wo, xc = t(wq), t(wk), t(wv), t(wo), t(xc)
    nkv, dh = dims.n_kv_heads, dims.d_head
    out = dict(r_qk=torch.empty(nkv, dh, dh, dtype=torch.float64, device=dev),
               r_vl=torch.empty(nkv, dh, dh, dtype=torch.float64, device=dev),
               sigma_qk=torch.empty(nkv, dh, dtype=torch.float64, device=dev),
               sigma_vl=torch.empty(nkv, dh, dtype=torch.float64, device=dev),
               wq_f=torch.empty_like(wq), wk_f=torch.empty_like(wk), wv_f=torch.empty_like(wv), wo_f=torch.empty_like(wo))
    D = make_dims(dims)
    nbytes = int(lib().zdc_fold_gpu_workspace(ctypes.byref(D), xc.shape[0], int(k_clusters)))
    ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
    p = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731
    _check(lib().zdc_fold_weights_gpu(ctypes.byref(D), p(wq), p(wk), p(wv), p(wo), p(xc), xc.shape[0], int(k_clusters),
                                      int(kmeans_iters), p(out["r_qk"]), p(out["r_vl"]), p(out["sigma_qk"]),
                                      p(out["sigma_vl"]), p(out["wq_f"]), p(out["wk_f"]), p(out["wv_f"]), p(out["wo_f"]),
                                      p(ws), nbytes, ctypes.c_void_p(_stream(stream))), "zdc_fold_weights_gpu")
    if return_device:
        return out
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def layer_groups(classes, threshold_bp: int = 9500):
    """zdc_layer_groups: classes bool/uint8 [L][B][S] -> group_rep list."""
    c = np.ascontiguousarray(np.asarray(classes).astype(np.uint8))
    L = c.shape[0]
    out = (ctypes.c_int32 * L)()
    _check(lib().zdc_layer_groups(ctypes.c_void_p(c.ctypes.data), L, int(c.size // L), int(threshold_bp), out),
           "zdc_layer_groups")
    return list(out)


def sp_positions(S_total: int, world: int, rank: int, layout: int) -> np.ndarray:
    n = S_total // world
    buf = (ctypes.c_int32 * max(n, 1))()
    _check(lib().zdc_sp_positions(S_total, world, rank, layout, buf), "zdc_sp_positions")
    return np.array(buf[:n], dtype=np.int64)


def comm_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it; the caller broadcasts it)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().zdc_comm_unique_id(buf), "zdc_comm_unique_id")
    return buf.raw


def gemm_bf16(a, b, d, stream=None):
    """D[M][N] = A[M][K] B[N][K]^T through zdc_gemm_bf16 (tcgen05)."""
    M, K = a.shape
    N = b.shape[0]
    _check(lib().zdc_gemm_bf16(_tptr(a, "bf16"), _tptr(b, "bf16"), _tptr(d, "bf16"), M, N, K, _stream(stream)),
           "zdc_gemm_bf16")


def gemv_bf16(w, x, y, stream=None):
    """y[B][N] = x[B][K] w[N][K]^T through zdc_gemv_bf16 (decode projection kernel, B <= 8)."""
    N, K = w.shape
    _check(lib().zdc_gemv_bf16(_tptr(w, "bf16"), _tptr(x, "bf16"), _tptr(y, "bf16"), x.shape[0], N, K,
                               _stream(stream)), "zdc_gemv_bf16")


def prefill_attention_bf16(q, k, v, o, lse=None, scale=None, stream=None):
    """Causal attention kernel alone: q, o [B][S][Nh*r]; k, v [B][Nkv][S][r]; lse [B][Nh][S] f32."""
    B, S, nhr = q.shape
    Nkv, r = k.shape[1], k.shape[3]
    Nh = nhr // r
    scale = 1.0 / r ** 0.5 if scale is None else scale
    _check(lib().zdc_prefill_attention_bf16(_tptr(q, "bf16"), _tptr(k, "bf16"), _tptr(v, "bf16"), _tptr(o, "bf16"),
                                            _tptr(lse, "f32") if lse is not None else None, B, S, Nh, Nkv, r,
                                            float(scale), _stream(stream)), "zdc_prefill_attention_bf16")


def decode_attention_bf16(q, k, v, o, length, lse=None, scale=None, workspace=None, stream=None):
    """Decode attention kernel alone: q, o [B][Nh*r]; k, v [B][Nkv][S_cap][r]; keys [0, length)."""
    import torch
    B, nhr = q.shape
    Nkv, S_cap, r = k.shape[1], k.shape[2], k.shape[3]
    Nh = nhr // r
    scale = 1.0 / r ** 0.5 if scale is None else scale
    if workspace is None:
        workspace = torch.zeros(int(lib().zdc_decode_attention_workspace(B, Nh, Nkv, r)), dtype=torch.uint8,
                                device=q.device)
    _check(lib().zdc_decode_attention_bf16(_tptr(q, "bf16"), _tptr(k, "bf16"), _tptr(v, "bf16"), _tptr(o, "bf16"),
                                           _tptr(lse, "f32") if lse is not None else None, B, Nh, Nkv, r,
                                           int(length), S_cap, float(scale), ctypes.c_void_p(workspace.data_ptr()),
                                           _stream(stream)), "zdc_decode_attention_bf16")
    return workspace


class Context:
    """zdc_ctx plus its three caller-owned device regions (allocated with torch)."""

    def __init__(self, dims, plan, max_batch: int, max_seq: int, device="cuda"):
        import torch
        self.dims, self.plan = dims, plan
        self._keep = [_i32arr(plan.r_qk_imp), _i32arr(plan.r_qk_unimp), _i32arr(plan.r_vl_imp),
                      _i32arr(plan.r_vl_unimp), _i32arr(plan.g_bp), _i32arr(plan.group_rep)]
        P = Plan(*[ctypes.cast(a, ctypes.POINTER(ctypes.c_int32)) for a in self._keep], int(plan.importance_mode),
                 int(getattr(plan, "kv_fp8", 0)))
        D = make_dims(dims)
        h = ctypes.c_void_p()
        _check(lib().zdc_ctx_create(ctypes.byref(D), ctypes.byref(P), max_batch, max_seq, ctypes.byref(h)),
               "zdc_ctx_create")
        self.h = h
        wb, cb, sb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().zdc_ctx_sizes(h, ctypes.byref(wb), ctypes.byref(cb), ctypes.byref(sb)), "zdc_ctx_sizes")
        self.sizes = (wb.value, cb.value, sb.value)
        self.weights = torch.empty(max(wb.value, 256), dtype=torch.uint8, device=device)
        self.cache = torch.empty(max(cb.value, 256), dtype=torch.uint8, device=device)
        self.scratch = torch.empty(max(sb.value, 256), dtype=torch.uint8, device=device)
        _check(lib().zdc_ctx_bind(h, ctypes.c_void_p(self.weights.data_ptr()), ctypes.c_void_p(self.cache.data_ptr()),
                                  ctypes.c_void_p(self.scratch.data_ptr())), "zdc_ctx_bind")
        self.max_batch, self.max_seq = max_batch, max_seq

    def close(self):
        if getattr(self, "h", None):
            lib().zdc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_folded(self, layer: int, wq_f, wk_f, wv_f, wo_f, stream=None):
        c = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
        arrs = [c(wq_f), c(wk_f), c(wv_f), c(wo_f)]
        _check(lib().zdc_load_folded(self.h, layer, *[_dptr(a) for a in arrs], ctypes.c_void_p(_stream(stream))),
               "zdc_load_folded")

    def load_folded_device(self, layer: int, wq_f, wk_f, wv_f, wo_f, stream=None):
        _check(lib().zdc_load_folded_device(self.h, layer, *[_tptr(t, "bf16") for t in (wq_f, wk_f, wv_f, wo_f)],
                                            ctypes.c_void_p(_stream(stream))), "zdc_load_folded_device")

    def prefill(self, x, y, l0: int = 0, l1: Optional[int] = None, importance=None, stream=None):
        l1 = self.dims.n_layers if l1 is None else l1
        B, S, _ = x.shape
        imp = _tptr(importance, "f32") if importance is not None else None
        _check(lib().zdc_prefill(self.h, l0, l1, _tptr(x, "bf16"), _tptr(y, "bf16"), B, S, imp,
                                 ctypes.c_void_p(_stream(stream))), "zdc_prefill")

    def decode(self, x, y, l0: int = 0, l1: Optional[int] = None, stream=None):
        l1 = self.dims.n_layers if l1 is None else l1
        _check(lib().zdc_decode(self.h, l0, l1, _tptr(x, "bf16"), _tptr(y, "bf16"), x.shape[0],
                                ctypes.c_void_p(_stream(stream))), "zdc_decode")

    def cache_length(self, layer: int) -> int:
        n = ctypes.c_int32()
        _check(lib().zdc_cache_length(self.h, layer, ctypes.byref(n)), "zdc_cache_length")
        return n.value

    def cache_sync(self, stream=None):
        """Refresh the host copy of the cache lengths from the device (after replaying zdc_decode
        calls inside a caller-captured CUDA graph)."""
        _check(lib().zdc_cache_sync(self.h, ctypes.c_void_p(_stream(stream))), "zdc_cache_sync")

    def cache_export(self, layer: int, B: int, stream=None):
        length = self.cache_length(layer)
        nkv = self.dims.n_kv_heads
        rk, rv = self.plan.r_qk_imp[layer], self.plan.r_vl_imp[layer]
        k = np.zeros((B, length, nkv, rk), dtype=np.float32)
        v = np.zeros((B, length, nkv, rv), dtype=np.float32)
        imp = np.zeros((B, length), dtype=np.uint8)
        tau = np.zeros(B, dtype=np.float32)
        ptr = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
        _check(lib().zdc_cache_export(self.h, layer, ptr(k), ptr(v), ptr(imp), ptr(tau),
                                      ctypes.c_void_p(_stream(stream))), "zdc_cache_export")
        return k, v, imp.astype(bool), tau

    def classes_export(self, layer: int, B: int, stream=None):
        """(is_important bool [B][len], tau [B]) of a layer's group, also for SP layers."""
        length = self.cache_length(layer)
        imp = np.zeros((B, length), dtype=np.uint8)
        tau = np.zeros(B, dtype=np.float32)
        ptr = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
        _check(lib().zdc_cache_export(self.h, layer, None, None, ptr(imp), ptr(tau), ctypes.c_void_p(_stream(stream))),
               "zdc_cache_export")
        return imp.astype(bool), tau

    def scores_export(self, layer: int, B: int, stream=None) -> np.ndarray:
        """GPU importance scores (f32) of every cached token of a representative layer."""
        length = self.cache_length(layer)
        out = np.zeros((B, length), dtype=np.float32)
        _check(lib().zdc_scores_export(self.h, layer, ctypes.c_void_p(out.ctypes.data),
                                       ctypes.c_void_p(_stream(stream))), "zdc_scores_export")
        return out

    def last_lse(self, layer: int, B: int, T: int, stream=None) -> np.ndarray:
        out = np.zeros((B, self.dims.n_heads, T), dtype=np.float32)
        _check(lib().zdc_last_lse(self.h, layer, ctypes.c_void_p(out.ctypes.data), ctypes.c_void_p(_stream(stream))),
               "zdc_last_lse")
        return out

    def comm_init(self, unique_id: bytes, rank: int, world: int):
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(lib().zdc_comm_init(self.h, buf, rank, world), "zdc_comm_init")

    def set_exchange_hook(self, fn, rank: int, world: int):
        """Test transport for zdc_sp_prefill (fn is an EXCHANGE_FN); keeps a reference to fn."""
        self._hook = fn
        _check(lib().zdc_sp_set_exchange_hook(self.h, fn, None, rank, world), "zdc_sp_set_exchange_hook")

    def set_alltoall_hook(self, fn, rank: int, world: int):
        """Test transport of zdc_sp_prefill_ulysses (fn is an ALLTOALL_FN); keeps a reference to fn."""
        self._a2a_hook = fn
        _check(lib().zdc_sp_set_alltoall_hook(self.h, fn, None, rank, world), "zdc_sp_set_alltoall_hook")

    def sp_prefill(self, x_local, y_local, S_total: int, layout: int = 1, l0: int = 0, l1: Optional[int] = None,
                   stats: bool = False, stream=None, dataflow: str = "allgather"):
        """dataflow "allgather" (zdc_sp_prefill) or "ulysses" (zdc_sp_prefill_ulysses)."""
        l1 = self.dims.n_layers if l1 is None else l1
        st = SpStats()
        name = {"allgather": "zdc_sp_prefill", "ulysses": "zdc_sp_prefill_ulysses"}[dataflow]
        _check(getattr(lib(), name)(self.h, l0, l1, _tptr(x_local, "bf16"), _tptr(y_local, "bf16"),
                                    x_local.shape[0], S_total, layout, ctypes.byref(st) if stats else None,
                                    ctypes.c_void_p(_stream(stream))), name)
        if stats:
            return {"bytes_sent": st.bytes_sent, "bytes_recv": st.bytes_recv,
                    "bytes_recv_uncompressed": st.bytes_recv_uncompressed, "exchange_ms": st.exchange_ms,
                    "total_ms": st.total_ms}
        return None

    def sp_decode(self, x, y, l0: int = 0, l1: Optional[int] = None, stream=None):
        """zdc_sp_decode: one token per sequence over the sequence-sharded cache of an SP prefill."""
        l1 = self.dims.n_layers if l1 is None else l1
        _check(lib().zdc_sp_decode(self.h, l0, l1, _tptr(x, "bf16"), _tptr(y, "bf16"), x.shape[0],
                                   ctypes.c_void_p(_stream(stream))), "zdc_sp_decode")

    def reset(self, stream=None):
        _check(lib().zdc_cache_reset(self.h, ctypes.c_void_p(_stream(stream))), "zdc_cache_reset")
