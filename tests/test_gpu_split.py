"""Token-level split (a4 + class-aware a2, §5.2) on the GPU.

* Selection is bit-exact given the GPU's own f32 scores: the oracle's selector (integer k,
  (score desc, index asc) order) runs on the exported score array.
* Packing is bit-exact given the same K'/V' rows: important rows equal the uniform-rank cache
  rows of the same projection, unimportant rows equal them truncated to r^u (zero-fill).
* End to end: y vs the fp64 oracle (which classifies with its own fp64 scores) within 2e-2,
  with the class agreement reported.
"""
import numpy as np
import pytest

import oracle as O
import zdc_synth as Z
from zdc_synth import Dims, plan_split, plan_uniform
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


def _decode(ctx, x):
    xd = to_dev_bf16(x)
    y = torch.empty_like(xd)
    ctx.decode(xd, y)
    torch.cuda.synchronize()
    return from_dev(y)


CASES = [
    # dims, r_imp, r_unimp, groups, g_bp per group, B, S, mode
    (Dims(4, 256, 4, 4, 64), 48, 16, [[0, 1], [2, 3]], [4000, 7000], 2, 200, 0),
    (Dims(2, 256, 8, 2, 64), 64, 32, [[0, 1]], [2500], 3, 130, 1),     # GQA G=4, mean mode
    (Dims(2, 128, 2, 2, 64), 64, 16, [[0, 1]], [10], 1, 64, 0),        # k = 1 of 64
]


@pytest.mark.parametrize("dims,ri,ru,groups,g,B,S,mode", CASES)
def test_split_prefill_selection_packing_parity(dims, ri, ru, groups, g, B, S, mode):
    plan = plan_split(dims.n_layers, ri, ru, groups, g, importance_mode=mode)
    _, folded = fold_stack(dims, 1, n_calib=256)
    x = Z.prompt(dims, 1, B, S, seed=31)
    ctx = make_context(dims, plan, folded, B, S + 8)
    y = _prefill(ctx, x)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    want = m.prefill(x)
    agree = []
    for grp, gbp in zip(groups, g):
        rep = grp[0]
        scores = ctx.scores_export(rep, B)                          # GPU f32 scores
        # scores vs the oracle's fp64 importance (log domain): absolute tolerance like the LSE
        assert np.max(np.abs(scores - m.scores[rep])) <= 0.05
        k_, v_, imp, tau = ctx.cache_export(rep, B)
        for b in range(B):
            # bit-exact selection given the GPU's own f32 scores
            sel, t_o, k = O.select_important(scores[b], gbp)
            assert np.array_equal(sel, imp[b]), (b, np.nonzero(sel != imp[b]))
            assert imp[b].sum() == O.important_count(gbp, S) == k
            if 0 < k < S:
                assert np.float32(t_o) == tau[b]
            agree.append(np.mean(imp[b] == m.classes[rep][b]))
        for l in grp:  # every layer of the group reuses the representative's classes
            _, _, imp_l, _ = ctx.cache_export(l, B)
            assert np.array_equal(imp_l, imp)
    assert np.mean(agree) >= 0.95
    assert normwise(y, want) <= TOL


def test_split_packing_bit_exact():
    """Representative layer: stored rows == the uniform-rank cache rows of the same projection
    (important) or those rows with dims >= r^u zeroed (unimportant)."""
    dims = Dims(1, 256, 4, 4, 64)
    ri, ru = 48, 16
    _, folded = fold_stack(dims, 1, n_calib=256)
    x = Z.prompt(dims, 1, 2, 150, seed=32)
    split = make_context(dims, plan_split(1, ri, ru, [[0]], [3000]), folded, 2, 160)
    uni = make_context(dims, plan_uniform(1, ri), folded, 2, 160)
    _prefill(split, x)
    _prefill(uni, x)
    ks, vs, imp, _ = split.cache_export(0, 2)
    ku, vu, _, _ = uni.cache_export(0, 2)
    assert imp.sum() == 2 * O.important_count(3000, 150)
    assert np.array_equal(ks[imp], ku[imp]) and np.array_equal(vs[imp], vu[imp])
    trunc_k, trunc_v = ku.copy(), vu.copy()
    trunc_k[..., ru:] = 0
    trunc_v[..., ru:] = 0
    assert np.array_equal(ks[~imp], trunc_k[~imp]) and np.array_equal(vs[~imp], trunc_v[~imp])


def test_split_decode_classes_and_parity():
    dims = Dims(2, 256, 4, 4, 64)
    plan = plan_split(2, 48, 16, [[0, 1]], [5000], importance_mode=1)
    _, folded = fold_stack(dims, 1, n_calib=256)
    B, S, T = 2, 120, 12
    x = Z.prompt(dims, 1, B, S + T, seed=33)
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
            # decode rule (reading c12) on the GPU's own f32 score and tau: strict >
            assert bool(imp[b, t]) == bool(np.float32(scores[b, t]) > np.float32(tau[b]))
    _, _, imp1, _ = ctx.cache_export(1, B)
    assert np.array_equal(imp1, imp)
    assert normwise(np.stack(ys, 1), np.stack(wants, 1)) <= TOL


@pytest.mark.slow
def test_split_c3_shape_slice():
    """c3 shape (d=5120, 40 heads, d_h=128, r^i=96, r^u=32), a 2-layer group, B=2, S=256."""
    dims = Z.dims_of(3, n_layers=2)
    plan = plan_split(2, 96, 32, [[0, 1]], [5000])
    _, folded = fold_stack(dims, 3, n_calib=1024)
    B, S = 2, 256
    x = Z.prompt(dims, 3, B, S, seed=34)
    ctx = make_context(dims, plan, folded, B, S + 16)
    y = _prefill(ctx, x)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    want = m.prefill(x)
    scores = ctx.scores_export(0, B)
    _, _, imp, _ = ctx.cache_export(0, B)
    for b in range(B):
        sel, _, _ = O.select_important(scores[b], 5000)
        assert np.array_equal(sel, imp[b])
    assert normwise(y, want) <= TOL
    for t in range(4):
        yd = _decode(ctx, Z.decode_input(dims, 3, B, t))
        wd = m.decode(Z.decode_input(dims, 3, B, t))
        assert normwise(yd, wd) <= TOL


def test_nan_importance_is_reported_and_overlap_rejected():
    """A NaN importance score (non-finite activations) is flagged by the selector and reported by
    zdc_cache_sync (the oracle's selector raises on NaN, reading c11); x / y ranges that overlap
    without being equal are rejected (ADVICE / VERDICT r1 hygiene)."""
    import paper_2408_04107_b200 as zdc
    dims = Dims(1, 64, 2, 2, 32)
    plan = plan_split(1, 16, 8, [[0]], [5000])
    _, folded = fold_stack(dims, 1, n_calib=256)
    ctx = make_context(dims, plan, folded, 1, 64)
    x = Z.prompt(dims, 1, 1, 32, seed=71)
    x[0, 5, :] = np.nan
    xd = to_dev_bf16(x)
    y = torch.empty_like(xd)
    ctx.prefill(xd, y)
    torch.cuda.synchronize()
    with pytest.raises(zdc.ZdcError) as e:
        ctx.cache_sync()
    assert e.value.status == -1
    ctx.reset()
    ctx.cache_sync()
    buf = torch.zeros(2 * 32 * 64, dtype=torch.bfloat16, device="cuda")
    xa = buf[: 32 * 64].view(1, 32, 64)
    ya = buf[16 * 64: 48 * 64].view(1, 32, 64)   # overlaps xa by 16 rows
    with pytest.raises(zdc.ZdcError):
        ctx.prefill(xa, ya)
    ctx.close()
