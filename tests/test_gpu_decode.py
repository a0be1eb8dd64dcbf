"""zdc_decode parity vs the fp64 oracle (north star: normwise max error <= 2e-2, BF16 storage,
FP32 accumulation).  Decode from an empty cache: by pin P7 the rows of
T decode steps equal the rows of a prefill over the same T tokens, which is what the oracle
computes.  Both sides get the same BF16-rounded inputs and the same folded weights (the
library rounds them to BF16 at load)."""
import numpy as np
import pytest

import oracle as O
import zdc_synth as Z
from zdc_synth import Dims, plan_uniform
from zdc_testlib import fold_stack, from_dev, make_context, normwise, to_dev_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2


def _run_decode(dims, plan, folded, x_steps, B):
    ctx = make_context(dims, plan, folded, B, x_steps.shape[1] + 4)
    ys = []
    for t in range(x_steps.shape[1]):
        x = to_dev_bf16(x_steps[:, t])
        y = torch.empty_like(x)
        ctx.decode(x, y)
        ys.append(from_dev(y))
    torch.cuda.synchronize()
    return ctx, np.stack(ys, axis=1)


@pytest.mark.parametrize("B", [1, 3])
def test_decode_c1_layer(B):
    dims = Z.dims_of(1)
    plan = plan_uniform(1, 16)
    _, folded = fold_stack(dims, 1)
    T = 40
    x = Z.prompt(dims, 1, B, T, seed=3)
    ctx, y = _run_decode(dims, plan, folded, x, B)
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    assert normwise(y, want) <= TOL
    want64 = O.OracleModel(dims, plan, folded).prefill(x)
    assert normwise(y, want64) <= TOL
    # the cache holds K'/V' of every token (a2), bf16 of the oracle's projections
    k, v, imp, tau = ctx.cache_export(0, B)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    m.prefill(x)
    assert k.shape == (B, T, 2, 16) and imp.all() and np.isinf(tau).all()
    assert normwise(k.transpose(0, 2, 1, 3), m.K[0]) <= 1e-2
    assert normwise(v.transpose(0, 2, 1, 3), m.V[0]) <= 1e-2


@pytest.mark.parametrize("dims,r", [(Dims(2, 128, 4, 2, 64), 32), (Dims(1, 256, 8, 1, 128), 64),
                                    (Dims(1, 512, 8, 8, 64), 64)])
def test_decode_gqa_chain(dims, r):
    """GQA groups (G = 2, 8), a 2-layer chain, ranks 32/64."""
    plan = plan_uniform(dims.n_layers, r)
    _, folded = fold_stack(dims, 1, n_calib=256)
    x = Z.prompt(dims, 1, 2, 24, seed=4)
    _, y = _run_decode(dims, plan, folded, x, 2)
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    assert normwise(y, want) <= TOL


def test_decode_c2_layer_long_context():
    """c2 shape (d=4096, 32 heads, d_h=128, r=64), one layer: 300 decode steps so the split-K
    attention spans several chunks with a ragged tail."""
    dims = Z.dims_of(2, n_layers=1)
    plan = plan_uniform(1, 64)
    _, folded = fold_stack(dims, 2, n_calib=1024)
    T = 300
    x = Z.prompt(dims, 2, 1, T, seed=5)
    _, y = _run_decode(dims, plan, folded, x, 1)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    rows = np.array([0, 1, 63, 64, 127, 128, 255, 299])
    want = m.prefill_rows(0, x, rows)
    assert normwise(y[:, rows], want) <= TOL


def test_decode_side_stream_graphs_pdl():
    """The production decode path: a non-default stream makes zdc_decode capture each call shape
    into a CUDA graph (device-side lengths) whose kernels use programmatic dependent launch.
    Per-layer calls (as bench.py issues them), 8 layers x 24 steps, parity with the oracle."""
    dims = Dims(8, 256, 4, 4, 64)
    plan = plan_uniform(8, 32)
    _, folded = fold_stack(dims, 1, n_calib=256)
    T = 24
    x = Z.prompt(dims, 1, 1, T, seed=9)
    ctx = make_context(dims, plan, folded, 1, T + 4)
    s = torch.cuda.Stream()
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    # (a) per-layer calls, buffer l feeds layer l: one graph per (layer, x, y, stream) shape
    with torch.cuda.stream(s):
        bufs = [torch.empty(1, 256, device="cuda", dtype=torch.bfloat16) for _ in range(9)]
        ys = []
        for t in range(T):
            bufs[0].copy_(to_dev_bf16(x[:, t]))
            for l in range(8):
                ctx.decode(bufs[l], bufs[l + 1], l, l + 1)
            ys.append(bufs[8].clone())
    s.synchronize()
    got = np.stack([from_dev(v) for v in ys], 1)
    assert normwise(got, want) <= TOL
    # (b) one chained call per step over the 8 layers (a single graph)
    ctx.reset()
    with torch.cuda.stream(s):
        xb = torch.empty(1, 256, device="cuda", dtype=torch.bfloat16)
        yb = torch.empty_like(xb)
        ys = []
        for t in range(T):
            xb.copy_(to_dev_bf16(x[:, t]))
            ctx.decode(xb, yb, 0, 8)
            ys.append(yb.clone())
    s.synchronize()
    got = np.stack([from_dev(v) for v in ys], 1)
    assert normwise(got, want) <= TOL


@pytest.mark.parametrize("B", [9, 16])
def test_decode_batch_above_gemv_limit(B):
    """B > 8 decode rows take the tcgen05 GEMM path for a1 / a5 (with the fused append and the
    device-side length advance in its epilogue / prologue)."""
    dims = Dims(2, 256, 4, 2, 64)
    plan = plan_uniform(2, 32)
    _, folded = fold_stack(dims, 1, n_calib=256)
    T = 12
    x = Z.prompt(dims, 1, B, T, seed=10)
    _, y = _run_decode(dims, plan, folded, x, B)
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    assert normwise(y, want) <= TOL
