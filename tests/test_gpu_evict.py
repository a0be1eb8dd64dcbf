"""NEXT-4 eviction (H2O-ZDC, P:1642 DEL; reading c26): a split group with r^u = 0 evicts its
unimportant tokens from the compressed cache.  GPU (zdc_prefill / zdc_decode) vs the fp64 oracle's
eviction semantics: the prompt attends in full (prefill rows = the plain model's), decode tokens
attend to the kept rows and to themselves, then leave the cache if unimportant."""
import numpy as np
import pytest

import oracle as O
import zdc_synth as Z
from zdc_synth import Dims, plan_split
from zdc_testlib import fold_stack, from_dev, make_context, normwise, to_dev_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,g_bp", [(0, 4000), (1, 5000)])
def test_eviction_prefill_decode(mode, g_bp):
    dims = Dims(2, 256, 4, 4, 64)
    plan = plan_split(2, 32, 0, [[0, 1]], [g_bp], importance_mode=mode)
    _, folded = fold_stack(dims, 1, n_calib=256)
    B, S, T = 2, 200, 6
    x = Z.prompt(dims, 1, B, S + T, seed=81)
    ctx = make_context(dims, plan, folded, B, S + T + 2)
    xd = to_dev_bf16(x[:, :S])
    y = torch.empty_like(xd)
    ctx.prefill(xd, y)
    ys = []
    for t in range(T):
        xt = to_dev_bf16(x[:, S + t])
        yt = torch.empty_like(xt)
        ctx.decode(xt, yt)
        ys.append(from_dev(yt))
    torch.cuda.synchronize()
    gpu_scores = ctx.scores_export(0, B)
    _, _, imp, tau = ctx.cache_export(0, B)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    want_p = m.prefill(x[:, :S])
    want_d = np.stack([m.decode(x[:, S + t]) for t in range(T)], axis=1)
    assert normwise(from_dev(y), want_p) <= 2e-2
    assert normwise(np.stack(ys, axis=1), want_d) <= 2e-2
    # selection bit-exact on the GPU's own scores; decode classes by strict > tau
    for b in range(B):
        cls, tau_b, _ = O.select_important(gpu_scores[b, :S].astype(np.float32), g_bp)
        assert imp[b, :S].tolist() == cls.tolist()
        assert imp[b, S:].tolist() == (gpu_scores[b, S:] > tau[b]).tolist()
    # evicted rows are gone from every layer's cache (exported as zeros); kept rows are present
    for l in range(2):
        k, v, imp_l, _ = ctx.cache_export(l, B)
        assert imp_l.tolist() == imp.tolist()
        assert np.all(k[~imp] == 0.0) and np.all(v[~imp] == 0.0)
        assert np.all(np.any(k[imp] != 0.0, axis=-1))
    ctx.close()
