"""Parity at the full layer shapes of B:configs c3 and c4 (one layer each, short sequences so the
fp64 oracle finishes in seconds): prefill, then decode steps, against the oracle's prefill rows
over the whole sequence (P7).  c4 exercises GQA G = 8 at d = 8192 through both
decode paths: the fused layer-step kernel (B = 8) and the separate GEMM + split-K kernels (B = 64,
the c4 batch).  c3 exercises d = 5120, 40 heads at rank 96 (a 3 x 32 swizzle width) with B = 32."""
import numpy as np
import pytest

import oracle as O
import zdc_synth as Z
from zdc_synth import plan_uniform
from zdc_testlib import fold_stack, from_dev, make_context, normwise, to_dev_bf16

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL = 2e-2


def _prefill_then_decode(dims, plan, folded, x, S, T):
    B = x.shape[0]
    ctx = make_context(dims, plan, folded, B, S + T + 4)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        xp = to_dev_bf16(x[:, :S])
        yp = torch.empty_like(xp)
        ctx.prefill(xp, yp)
        ys = []
        for t in range(T):
            xt = to_dev_bf16(x[:, S + t])
            yt = torch.empty_like(xt)
            ctx.decode(xt, yt)
            ys.append(yt)
    s.synchronize()
    return from_dev(yp), np.stack([from_dev(v) for v in ys], axis=1)


@pytest.fixture(scope="module")
def c4_layer():
    dims = Z.dims_of(4, n_layers=1)
    _, folded = fold_stack(dims, 4, n_calib=1024)
    return dims, folded


@pytest.mark.parametrize("B,S,T", [(8, 48, 3), (64, 32, 2)])
def test_c4_layer_prefill_decode(c4_layer, B, S, T):
    dims, folded = c4_layer
    plan = plan_uniform(1, 64)
    x = Z.prompt(dims, 4, B, S + T, seed=21)
    yp, yd = _prefill_then_decode(dims, plan, folded, x, S, T)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    want = m.prefill(x)
    assert normwise(yp, want[:, :S]) <= TOL
    assert normwise(yd, want[:, S:]) <= TOL


def test_c3_layer_prefill_decode_rank96():
    dims = Z.dims_of(3, n_layers=1)
    plan = plan_uniform(1, 96)
    _, folded = fold_stack(dims, 3, n_calib=1024)
    B, S, T = 32, 40, 2
    x = Z.prompt(dims, 3, B, S + T, seed=22)
    yp, yd = _prefill_then_decode(dims, plan, folded, x, S, T)
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    assert normwise(yp, want[:, :S]) <= TOL
    assert normwise(yd, want[:, S:]) <= TOL
