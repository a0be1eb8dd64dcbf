"""NEXT-4: the FP8 (E4M3) compressed KV cache, GEAR-ZDC (P:1642 DEL; reading c23), against the fp64
oracle's kv_fp8 mode: the prompt attends at full precision, the cache keeps per-row-scaled E4M3
codes, decode attends the quantized cache (its own new row included)."""
import numpy as np
import pytest

import oracle as O
import zdc_synth as Z
from zdc_synth import Dims, plan_split, plan_uniform
from zdc_testlib import fold_stack, from_dev, make_context, normwise, to_dev_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _plan8(L, r):
    p = plan_uniform(L, r)
    p.kv_fp8 = 1
    return p


@pytest.mark.parametrize("dims,r,B,S,T", [
    (Z.dims_of(1), 32, 1, 128, 8),            # c1 shape
    (Dims(1, 512, 8, 8, 64), 64, 2, 300, 6),  # MHA, r = d_h / 2
    (Dims(1, 512, 16, 4, 64), 64, 3, 200, 5),  # GQA G = 4
    (Dims(2, 384, 4, 4, 96), 96, 2, 130, 4),   # r = 96, 2-layer chain
    (Dims(1, 256, 2, 2, 128), 64, 1, 3000, 3),  # long context: every warp's ring wraps many times
])
def test_fp8_cache_prefill_decode(dims, r, B, S, T):
    plan = _plan8(dims.n_layers, r)
    _, folded = fold_stack(dims, 1, n_calib=512)
    x = Z.prompt(dims, 1, B, S + T, seed=61)
    ctx = make_context(dims, plan, folded, B, S + T + 2)
    xd = to_dev_bf16(x[:, :S])
    yp = torch.empty_like(xd)
    ctx.prefill(xd, yp)
    ys = []
    for t in range(T):
        xt = to_dev_bf16(x[:, S + t])
        yt = torch.empty_like(xt)
        ctx.decode(xt, yt)
        ys.append(from_dev(yt))
    torch.cuda.synchronize()
    m = O.OracleModel(dims, plan, folded, faithful=True)
    want_p = m.prefill(x[:, :S])
    want_d = np.stack([m.decode(x[:, S + t]) for t in range(T)], axis=1)
    assert normwise(from_dev(yp), want_p) <= 2e-2
    assert normwise(np.stack(ys, axis=1), want_d) <= 2e-2
    # the cache holds quantize_rows of the K'/V' rows: within one E4M3 step of the oracle's codes
    # (layer 0: its input is the exact x; a chained layer's input carries layer 0's bf16 error)
    l = 0
    k, v, _, _ = ctx.cache_export(l, B)
    kk, vv = k.transpose(0, 2, 1, 3), v.transpose(0, 2, 1, 3)
    assert normwise(kk, m.K[l]) <= 2e-2 and normwise(vv, m.V[l]) <= 2e-2
    exact = np.mean(np.abs(kk - m.K[l]) <= 1e-6 * np.abs(m.K[l]) + 1e-30)
    assert exact >= 0.95, exact
    # FP8 rows are really quantized: every cached row is code x scale with |code| <= 448
    amax = np.max(np.abs(kk), axis=-1, keepdims=True)
    scale = np.where(amax > 0, amax / 448.0, 1.0)
    assert np.allclose(O.e4m3(kk / scale) * scale, kk, rtol=1e-5, atol=0)
    ctx.close()


def test_fp8_cache_graph_replay_and_rejects():
    import paper_2408_04107_b200 as zdc
    dims = Dims(1, 256, 4, 4, 64)
    plan = _plan8(1, 32)
    _, folded = fold_stack(dims, 1, n_calib=256)
    T = 10
    x = Z.prompt(dims, 1, 2, T, seed=62)
    ctx = make_context(dims, plan, folded, 2, T + 2)
    s = torch.cuda.Stream()
    xb = torch.empty(2, 256, device="cuda", dtype=torch.bfloat16)
    yb = torch.empty_like(xb)
    ys = []
    with torch.cuda.stream(s):
        xb.copy_(to_dev_bf16(x[:, 0]))
        ctx.decode(xb, yb)
        ys.append(yb.clone())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ctx.decode(xb, yb)
        for t in range(1, T):
            xb.copy_(to_dev_bf16(x[:, t]))
            g.replay()
            ys.append(yb.clone())
    s.synchronize()
    m = O.OracleModel(dims, plan, folded, faithful=True)
    m.prefill(x[:, :1])   # decode from empty: token 0 by prefill (P7) ...
    want = [None] + [m.decode(x[:, t]) for t in range(1, T)]
    got = np.stack([from_dev(v) for v in ys[1:]], axis=1)
    assert normwise(got, np.stack(want[1:], axis=1)) <= 2e-2
    ctx.close()
    bad = plan_split(1, 32, 16, [[0]], [5000])
    bad.kv_fp8 = 1
    with pytest.raises(zdc.ZdcError):
        zdc.Context(dims, bad, 1, 16)
    with pytest.raises(zdc.ZdcError):
        zdc.Context(dims, _plan8(1, 16), 1, 16)
