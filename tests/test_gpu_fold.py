"""NEXT-3: the offline fold on the GPU (zdc_fold_weights_gpu) against the fp64 oracle fold
(P:989-990 SVD of the stacked Q/K and V/W_L blocks; P:1157-1167 K-means consolidation of the
calibration Q, K, V vectors).  R is compared after canonical signs (reading c5); the Gram-based
eigen-decomposition squares the stack's condition number, hence 1e-8 here vs 1e-10 for the host
TSQR + Jacobi fold (tests/test_fold.py)."""
import numpy as np
import pytest

import oracle as O
import zdc_synth as Z
from zdc_synth import Dims, plan_uniform
from zdc_testlib import from_dev, normwise, to_dev_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _check_fold(g, o, tol_r=1e-8):
    for key in ("r_qk", "r_vl"):
        assert np.max(np.abs(g[key] - o[key])) <= tol_r, (key, np.max(np.abs(g[key] - o[key])))
    for key in ("sigma_qk", "sigma_vl"):
        assert np.max(np.abs(g[key] - o[key]) / o[key][:, :1]) <= 1e-9, key
    for key in ("wq_f", "wk_f", "wv_f", "wo_f"):
        assert np.max(np.abs(g[key] - o[key])) <= tol_r * np.max(np.abs(o[key])), key


@pytest.mark.parametrize("dims,n", [(Z.dims_of(1), 512), (Dims(1, 256, 8, 2, 64), 1024), (Dims(1, 512, 4, 4, 128), 2048)])
def test_gpu_fold_equals_svd_fold(dims, n):
    import paper_2408_04107_b200 as zdc
    w = Z.layer_weights(dims, 1, 0)
    xc = Z.calibration(dims, 1, 0, n)
    o = O.fold_layer(dims, w.wq, w.wk, w.wv, w.wo, xc)
    g = zdc.fold_weights_gpu(dims, w.wq, w.wk, w.wv, w.wo, xc)
    _check_fold(g, o)
    # R is orthonormal
    for R in list(g["r_qk"]) + list(g["r_vl"]):
        assert np.max(np.abs(R.T @ R - np.eye(dims.d_head))) <= 1e-10


@pytest.mark.parametrize("dims,n,k,iters", [(Z.dims_of(1), 1024, 64, 4), (Dims(1, 256, 8, 2, 64), 4096, 256, 6)])
def test_gpu_kmeans_fold_equals_oracle(dims, n, k, iters):
    """The K-means fold (reading c21): same Lloyd rounds on both sides."""
    import paper_2408_04107_b200 as zdc
    w = Z.layer_weights(dims, 1, 0)
    xc = Z.calibration(dims, 1, 0, n)
    o = O.fold_layer(dims, w.wq, w.wk, w.wv, w.wo, xc, k_clusters=k, kmeans_iters=iters)
    g = zdc.fold_weights_gpu(dims, w.wq, w.wk, w.wv, w.wo, xc, k_clusters=k, kmeans_iters=iters)
    _check_fold(g, o)


def test_gpu_kmeans_fold_drives_the_hot_path():
    """A layer folded on the GPU with K-means (k = 256 of 4096 calibration rows) runs prefill and
    decode within the north-star tolerance of the oracle folded the same way."""
    import paper_2408_04107_b200 as zdc
    dims = Dims(1, 256, 4, 4, 64)
    plan = plan_uniform(1, 32)
    w = Z.layer_weights(dims, 1, 0)
    xc = Z.calibration(dims, 1, 0, 4096)
    g = zdc.fold_weights_gpu(dims, w.wq, w.wk, w.wv, w.wo, xc, k_clusters=256, kmeans_iters=5)
    o = O.fold_layer(dims, w.wq, w.wk, w.wv, w.wo, xc, k_clusters=256, kmeans_iters=5)
    ctx = zdc.Context(dims, plan, 2, 80)
    ctx.load_folded(0, g["wq_f"], g["wk_f"], g["wv_f"], g["wo_f"])
    x = Z.prompt(dims, 1, 2, 72, seed=51)
    xd = to_dev_bf16(x[:, :64])
    y = torch.empty_like(xd)
    ctx.prefill(xd, y)
    ys = [from_dev(y)]
    for t in range(64, 72):
        xt = to_dev_bf16(x[:, t])
        yt = torch.empty_like(xt)
        ctx.decode(xt, yt)
        ys.append(from_dev(yt)[:, None])
    torch.cuda.synchronize()
    want = O.OracleModel(dims, plan, [o], faithful=True).prefill(x)
    assert normwise(np.concatenate(ys, axis=1), want) <= 2e-2
    ctx.close()


def test_gpu_fold_errors():
    import paper_2408_04107_b200 as zdc
    dims = Dims(1, 64, 2, 2, 32)
    w = Z.layer_weights(dims, 1, 0)
    with pytest.raises(zdc.ZdcError):   # insufficient samples: 8 rows x (G+1) = 16 < d_head 32
        zdc.fold_weights_gpu(dims, w.wq, w.wk, w.wv, w.wo, Z.calibration(dims, 1, 0, 8))
    with pytest.raises(zdc.ZdcError):   # 8 clusters x (G+1) < d_head
        zdc.fold_weights_gpu(dims, w.wq, w.wk, w.wv, w.wo, Z.calibration(dims, 1, 0, 512), k_clusters=8,
                             kmeans_iters=2)


def test_layer_groups_from_gpu_classes():
    """NEXT-3 planner on classes the GPU computed: every layer its own representative (g = 0.5),
    layers 0 and 1 share weights (so, with the same input, identical token sets), layers 2 and 3 are
    independent.  zdc_layer_groups on the exported classes gives [0, 0, 2, 3], the same
    as the oracle's rule on the oracle's own classes."""
    import paper_2408_04107_b200 as zdc
    from zdc_synth import plan_split
    from zdc_testlib import fold_stack
    dims = Dims(4, 256, 4, 4, 64)
    _, folded = fold_stack(dims, 1, n_calib=256)
    folded[1] = folded[0]
    plan = plan_split(4, 32, 16, [[0], [1], [2], [3]], [5000] * 4)
    B, S = 2, 200
    x = Z.prompt(dims, 1, B, S, seed=52)
    ctx = zdc.Context(dims, plan, B, S)
    for l, f in enumerate(folded):
        g = f["lib"]
        ctx.load_folded(l, g["wq_f"], g["wk_f"], g["wv_f"], g["wo_f"])
    xd = to_dev_bf16(x)
    y = torch.empty_like(xd)
    for l in range(4):
        ctx.prefill(xd, y, l, l + 1)
    torch.cuda.synchronize()
    cls = np.stack([ctx.cache_export(l, B)[2] for l in range(4)])
    assert zdc.layer_groups(cls, 9500) == O.layer_groups(cls, 9500) == [0, 0, 2, 3]
    m = O.OracleModel(dims, plan, folded, faithful=True)
    for l in range(4):
        m.prefill_layer(l, x)
    ocls = np.stack([m.classes[l] for l in range(4)])
    assert O.layer_groups(ocls, 9500) == [0, 0, 2, 3]
    assert np.mean(ocls == cls) >= 0.98
    ctx.close()
