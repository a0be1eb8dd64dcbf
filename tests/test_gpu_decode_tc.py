"""Decode through the tensor-core GQA attention kernel (decode_attn_tc.cu) vs the fp64 oracle:
grouped-query layers (G = N_h / N_kv in {2, 4, 8}) at uniform rank r in {64, 128} with B > 8
(the separate-kernel decode path), one- and multi-tile contexts with ragged last tiles, and a
prefill + decode continuation long enough for several key splits per (sequence, KV head) whose
partials the last CTA LSE-merges.  By P7 decode rows equal prefill rows."""
import numpy as np
import pytest

import oracle as O
import zdc_synth as Z
from zdc_synth import Dims, plan_uniform
from zdc_testlib import fold_stack, from_dev, make_context, normwise, to_dev_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2


def _decode(ctx, x_steps):
    ys = []
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for t in range(x_steps.shape[1]):
            x = to_dev_bf16(x_steps[:, t])
            y = torch.empty_like(x)
            ctx.decode(x, y)
            ys.append(y)
    s.synchronize()
    return np.stack([from_dev(v) for v in ys], axis=1)


@pytest.mark.parametrize("dims,r,B,T", [
    (Dims(1, 512, 16, 2, 64), 64, 12, 40),     # G = 8, one ragged tile
    (Dims(1, 512, 8, 2, 128), 128, 10, 150),   # G = 4 at full rank r = d_h, two tiles
    (Dims(2, 256, 4, 2, 64), 64, 9, 33),       # G = 2, 2-layer chain
])
def test_decode_tc_from_empty(dims, r, B, T):
    plan = plan_uniform(dims.n_layers, r)
    _, folded = fold_stack(dims, 1, n_calib=max(256, 2 * dims.d_head))
    x = Z.prompt(dims, 1, B, T, seed=31)
    ctx = make_context(dims, plan, folded, B, T + 2)
    y = _decode(ctx, x)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    want = m.prefill(x)
    assert normwise(y, want) <= TOL
    # LSE of the last step's query heads (natural log of the Eq. 3 denominator)
    lse = ctx.last_lse(dims.n_layers - 1, B, 1)[:, :, 0]
    assert np.max(np.abs(lse - m.lse[dims.n_layers - 1][:, :, T - 1])) <= 0.05
    ctx.close()


def test_decode_tc_splits_after_prefill():
    """B = 16 sequences, G = 4: a 600-token prefill, then 8 decode steps; the context splits into
    3 key ranges per (sequence, KV head) (ragged last range) merged by the last CTA."""
    dims = Dims(1, 256, 8, 2, 64)
    plan = plan_uniform(1, 64)
    _, folded = fold_stack(dims, 1, n_calib=256)
    B, S, T = 16, 600, 8
    x = Z.prompt(dims, 1, B, S + T, seed=32)
    ctx = make_context(dims, plan, folded, B, S + T + 4)
    y0 = torch.empty(B, S, dims.d_model, dtype=torch.bfloat16, device="cuda")
    ctx.prefill(to_dev_bf16(x[:, :S]), y0)
    y = _decode(ctx, x[:, S:])
    m = O.OracleModel(dims, plan, folded, faithful=True)
    rows = np.array([S, S + 3, S + T - 1])
    want = m.prefill_rows(0, x, rows)
    assert normwise(y[:, rows - S], want) <= TOL
    ctx.close()
