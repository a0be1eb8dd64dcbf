"""CPU checks of the C-ABI boundary: the library loads, exports every symbol include/zdc.h
declares, and rejects bad arguments synchronously (no GPU needed for any of these)."""
import ctypes
import os
import re

import pytest

import paper_2408_04107_b200 as zdc
from zdc_synth import Dims, plan_uniform

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "zdc.h")).read()
    return sorted(set(re.findall(r"\b(zdc_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    L = zdc.lib()
    syms = _header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(zdc.EXPORTED_SYMBOLS)


def test_version_and_error_strings():
    assert b"sm_100a" in zdc.lib().zdc_version()


def _create(dims, plan, B=1, S=16):
    return zdc.Context.__new__(zdc.Context), dims, plan


def test_ctx_create_rejects_bad_shapes():
    L = zdc.lib()
    bad = [
        (Dims(1, 64, 3, 2, 32), plan_uniform(1, 16), "n_heads"),        # Nh % Nkv
        (Dims(1, 60, 2, 2, 30), plan_uniform(1, 16), "d_model"),        # d % 64
        (Dims(1, 64, 2, 2, 32), plan_uniform(1, 40), "ranks"),          # r > d_head
        (Dims(1, 64, 2, 2, 32), plan_uniform(1, 24), "padded ranks"),   # 24 -> 32 ok; make unequal below
    ]
    for dims, plan, why in bad[:3]:
        keep = [zdc._i32arr(a) for a in (plan.r_qk_imp, plan.r_qk_unimp, plan.r_vl_imp, plan.r_vl_unimp,
                                          plan.g_bp, plan.group_rep)]
        P = zdc.Plan(*[ctypes.cast(a, ctypes.POINTER(ctypes.c_int32)) for a in keep], 0)
        D = zdc.make_dims(dims)
        h = ctypes.c_void_p()
        st = L.zdc_ctx_create(ctypes.byref(D), ctypes.byref(P), 1, 16, ctypes.byref(h))
        assert st < 0, why
        assert len(L.zdc_last_error()) > 0


def test_ctx_sizes_closed_form():
    """Cache bytes = L * B * S * N_kv * (r_k + r_v) * 2 (P12, uniform plan, padded ranks)."""
    L = zdc.lib()
    dims = Dims(2, 256, 4, 2, 64)
    plan = plan_uniform(2, 32)
    keep = [zdc._i32arr(a) for a in (plan.r_qk_imp, plan.r_qk_unimp, plan.r_vl_imp, plan.r_vl_unimp,
                                      plan.g_bp, plan.group_rep)]
    P = zdc.Plan(*[ctypes.cast(a, ctypes.POINTER(ctypes.c_int32)) for a in keep], 0)
    D = zdc.make_dims(dims)
    h = ctypes.c_void_p()
    assert L.zdc_ctx_create(ctypes.byref(D), ctypes.byref(P), 3, 100, ctypes.byref(h)) == 0
    wb, cb, sb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    assert L.zdc_ctx_sizes(h, ctypes.byref(wb), ctypes.byref(cb), ctypes.byref(sb)) == 0
    assert cb.value == 2 * 3 * 100 * 2 * (32 + 32) * 2 + 256  # + int32 lengths, 256-B aligned
    # weights: [N_h r + N_kv (r + r)] x d  +  d x roundup(N_h r, 64), bf16
    wqkv = (4 * 32 + 2 * 64) * 256 * 2
    assert wb.value == 2 * (wqkv + 256 * 128 * 2)
    L.zdc_ctx_destroy(h)
    # decode mode 2 (cluster kernel) adds its decode copies: W_O group-major (N_h r x d) and W_QKV
    # pre-tiled ([N_h r + N_kv (r + r)] x d)
    old = L.zdc_decode_mode(2)
    try:
        assert L.zdc_ctx_create(ctypes.byref(D), ctypes.byref(P), 3, 100, ctypes.byref(h)) == 0
        assert L.zdc_ctx_sizes(h, ctypes.byref(wb), ctypes.byref(cb), ctypes.byref(sb)) == 0
        assert wb.value == 2 * (wqkv + 256 * 128 * 2 + 4 * 32 * 256 * 2 + wqkv)
        L.zdc_ctx_destroy(h)
    finally:
        L.zdc_decode_mode(old)


def test_unbound_ctx_calls_fail():
    L = zdc.lib()
    dims = Dims(1, 64, 2, 2, 32)
    plan = plan_uniform(1, 16)
    keep = [zdc._i32arr(a) for a in (plan.r_qk_imp, plan.r_qk_unimp, plan.r_vl_imp, plan.r_vl_unimp,
                                      plan.g_bp, plan.group_rep)]
    P = zdc.Plan(*[ctypes.cast(a, ctypes.POINTER(ctypes.c_int32)) for a in keep], 0)
    D = zdc.make_dims(dims)
    h = ctypes.c_void_p()
    assert L.zdc_ctx_create(ctypes.byref(D), ctypes.byref(P), 1, 16, ctypes.byref(h)) == 0
    st = L.zdc_prefill(h, 0, 1, ctypes.c_void_p(16), ctypes.c_void_p(32), 1, 4, None, None)
    assert st == -9  # ZDC_ERR_STATE: not bound
    L.zdc_ctx_destroy(h)
