"""Decode attention v3 (decode_attn3.cu: byte-balanced flat split of every (sequence, KV head)
pair's pool-0 / pool-1 rows over one resident warp set, warp-MMA scores and PV) through the full
decode path, against the fp64 oracle (faithful rounding mode).

Cases span the kernel's instantiations (pool widths 96/32, 64/16, 32/16, uniform 64), grouped-query
layers (G = 2, 4, 8 query heads per KV group share one MMA row block), batches above the fused
kernel's limit, and per-sequence pool counts that differ (the token split classifies each sequence
separately), so pairs straddle warps and are merged from several pieces.  The decode class rule
(strict > tau, reading c12) is checked on the GPU's own scores.  PAPER.md:249-260 (Eqs. 2-3),
:1409-1442 (§5.2)."""
import numpy as np
import pytest

import oracle as O
import zdc_synth as Z
from zdc_synth import Dims, plan_split, plan_uniform
from zdc_testlib import fold_stack, from_dev, make_context, normwise, to_dev_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2


def _prefill(ctx, x):
    xd = to_dev_bf16(x)
    y = torch.empty_like(xd)
    ctx.prefill(xd, y)
    torch.cuda.synchronize()
    return from_dev(y)


def _decode(ctx, x):
    xd = to_dev_bf16(x)
    y = torch.empty_like(xd)
    ctx.decode(xd, y)
    torch.cuda.synchronize()
    return from_dev(y)


SPLIT_CASES = [
    # dims (L, d, Nh, Nkv, d_h), r^i, r^u, B, S, T, g_bp, importance mode
    (Dims(2, 384, 4, 4, 128), 96, 32, 9, 120, 5, 5000, 1),    # c3 widths, B > 8
    (Dims(2, 256, 8, 2, 64), 64, 16, 5, 100, 5, 3000, 0),     # GQA G = 4, raw importance
    (Dims(2, 256, 8, 1, 64), 32, 16, 3, 90, 6, 6000, 1),      # GQA G = 8 (one KV head)
    (Dims(2, 256, 4, 2, 64), 64, 32, 12, 70, 4, 2500, 1),     # G = 2, B = 12
]


@pytest.mark.parametrize("dims,ri,ru,B,S,T,g,mode", SPLIT_CASES)
def test_v3_split_decode_parity(dims, ri, ru, B, S, T, g, mode):
    plan = plan_split(dims.n_layers, ri, ru, [list(range(dims.n_layers))], [g], importance_mode=mode)
    _, folded = fold_stack(dims, 1, n_calib=max(256, 2 * dims.d_head))
    x = Z.prompt(dims, 1, B, S + T, seed=71)
    ctx = make_context(dims, plan, folded, B, S + T)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    _prefill(ctx, x[:, :S])
    m.prefill(x[:, :S])
    ys, wants = [], []
    for t in range(T):
        ys.append(_decode(ctx, x[:, S + t]))
        wants.append(m.decode(x[:, S + t]))
    scores = ctx.scores_export(0, B)
    _, _, imp, tau = ctx.cache_export(0, B)
    for b in range(B):
        for t in range(S, S + T):
            assert bool(imp[b, t]) == bool(np.float32(scores[b, t]) > np.float32(tau[b]))
    err = normwise(np.stack(ys, 1), np.stack(wants, 1))
    assert err <= TOL, "v3 split decode normwise error %.3g" % err


@pytest.mark.parametrize("dims,r,B,S,T", [
    (Dims(1, 256, 16, 16, 64), 64, 10, 150, 4),   # uniform, G = 1, 160 pairs >= the SMs (v3 64 / 0)
    (Dims(1, 256, 16, 16, 64), 32, 12, 40, 3),    # uniform r = 32, short context (few rows per warp)
])
def test_v3_uniform_decode_parity(dims, r, B, S, T):
    plan = plan_uniform(dims.n_layers, r)
    _, folded = fold_stack(dims, 1, n_calib=256)
    x = Z.prompt(dims, 1, B, S + T, seed=72)
    ctx = make_context(dims, plan, folded, B, S + T)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    _prefill(ctx, x[:, :S])
    m.prefill(x[:, :S])
    ys, wants = [], []
    for t in range(T):
        ys.append(_decode(ctx, x[:, S + t]))
        wants.append(m.decode(x[:, S + t]))
    err = normwise(np.stack(ys, 1), np.stack(wants, 1))
    assert err <= TOL, "v3 uniform decode normwise error %.3g" % err
