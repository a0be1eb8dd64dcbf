"""zdc_prefill parity vs the fp64 oracle: tcgen05 QKV projection (a1) with the fused cache
append (a2), tcgen05 causal attention at head dim r (a3) with its LSE, tcgen05 output
projection (a5).  Tolerance: north star normwise 2e-2 (BF16 storage, FP32 accumulation)."""
import math

import numpy as np
import pytest

import oracle as O
import zdc_synth as Z
from zdc_synth import Dims, plan_uniform
from zdc_testlib import fold_stack, from_dev, make_context, normwise, to_dev_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2


def _prefill(ctx, x, l0=0, l1=None):
    xd = to_dev_bf16(x)
    y = torch.empty_like(xd)
    ctx.prefill(xd, y, l0, l1)
    torch.cuda.synchronize()
    return from_dev(y)


@pytest.mark.parametrize("B,S", [(1, 128), (2, 128), (1, 200), (3, 77), (1, 1)])
def test_prefill_c1(B, S):
    dims = Z.dims_of(1)
    plan = plan_uniform(1, 16)
    _, folded = fold_stack(dims, 1)
    x = Z.prompt(dims, 1, B, S, seed=11)
    ctx = make_context(dims, plan, folded, B, S + 8)
    y = _prefill(ctx, x)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    want = m.prefill(x)
    assert normwise(y, want) <= TOL
    # LSE of every row (natural log of the Eq. 3 denominator), absolute tolerance
    lse = ctx.last_lse(0, B, S)
    assert np.max(np.abs(lse - m.lse[0])) <= 0.05
    # the cache holds K'/V' of every prompt token (a2)
    k, v, _, _ = ctx.cache_export(0, B)
    assert normwise(k.transpose(0, 2, 1, 3), m.K[0]) <= 1e-2
    assert normwise(v.transpose(0, 2, 1, 3), m.V[0]) <= 1e-2


@pytest.mark.parametrize("dims,r,S", [
    (Dims(1, 128, 4, 2, 64), 32, 300),     # GQA G=2, r=32 (64B swizzle), 3 ragged tiles
    (Dims(1, 256, 8, 1, 128), 64, 260),    # G=8 (MQA-like)
    (Dims(1, 256, 2, 2, 128), 128, 140),   # r = d_h = 128: two 64-wide chunks
    (Dims(2, 256, 4, 4, 64), 64, 129),     # 2-layer chain
])
def test_prefill_shapes(dims, r, S):
    plan = plan_uniform(dims.n_layers, r)
    _, folded = fold_stack(dims, 1, n_calib=256)
    x = Z.prompt(dims, 1, 2, S, seed=12)
    ctx = make_context(dims, plan, folded, 2, S)
    y = _prefill(ctx, x)
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    assert normwise(y, want) <= TOL


def test_prefill_then_decode_equals_prefill_rows():
    """P7 on the GPU: prefill S tokens then decode T tokens == rows S..S+T-1 of the oracle prefill."""
    dims = Dims(2, 256, 4, 4, 64)
    plan = plan_uniform(2, 64)
    _, folded = fold_stack(dims, 1, n_calib=256)
    S, T = 150, 10
    x = Z.prompt(dims, 1, 2, S + T, seed=13)
    ctx = make_context(dims, plan, folded, 2, S + T)
    _prefill(ctx, x[:, :S])
    ys = []
    for t in range(T):
        xd = to_dev_bf16(x[:, S + t])
        y = torch.empty_like(xd)
        ctx.decode(xd, y)
        ys.append(from_dev(y))
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    assert normwise(np.stack(ys, 1), want[:, S:]) <= TOL


@pytest.mark.slow
def test_prefill_c2_layer_full_size_sampled():
    """c2 at full size (S=2048, d=4096, 32 heads, r=64), one layer, in bench.py's launch
    configuration; the oracle computes sampled rows one by one (it projects all K'/V')."""
    dims = Z.dims_of(2, n_layers=1)
    plan = plan_uniform(1, 64)
    _, folded = fold_stack(dims, 2, n_calib=1024)
    x = Z.prompt(dims, 2, 1, 2048, seed=14)
    ctx = make_context(dims, plan, folded, 1, 2048 + 256)
    y = _prefill(ctx, x)
    rows = np.array([0, 1, 2, 127, 128, 129, 1000, 1023, 1024, 2046, 2047])
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill_rows(0, x, rows)
    assert normwise(y[:, rows], want) <= TOL
    # property at any size: no NaN/Inf anywhere and row norms in the expected band
    assert np.all(np.isfinite(y))
