"""Shared helpers for the GPU parity tests (test infrastructure; imports the oracle)."""
from __future__ import annotations

import numpy as np

import oracle as O
import zdc_synth as Z


def normwise(g, o) -> float:
    """max_i |g_i - o_i| / max_i |o_i| (DESIGN.md §4.3 parity metric)."""
    g = np.asarray(g, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    return float(np.max(np.abs(g - o)) / max(float(np.max(np.abs(o))), 1e-30))


def fold_stack(dims, cfg_id, n_calib=512, seed=0, **wkw):
    """Each side folds independently (SURVEY.md §8(c) "Inputs"): the oracle with NumPy/LAPACK in
    fp64 (the dicts returned), the library with its own host fold `zdc_fold_weights` (kept under
    the "lib" key and loaded by make_context / load_lib_fold).  Both see the same BF16-rounded
    unfolded weights and calibration rows; their R agree up to the fold tolerance (test_fold.py)."""
    import paper_2408_04107_b200 as zdc
    ws, folded = [], []
    for l in range(dims.n_layers):
        w = Z.layer_weights(dims, cfg_id, l, seed, **wkw)
        xc = Z.calibration(dims, cfg_id, l, n_calib, seed)
        ws.append(w)
        f = O.fold_layer(dims, w.wq, w.wk, w.wv, w.wo, xc)
        f["lib"] = zdc.fold_weights(dims, w.wq, w.wk, w.wv, w.wo, xc)
        folded.append(f)
    return ws, folded


def load_lib_fold(ctx, layer, f):
    """Load the LIBRARY's fold of this layer (never the oracle's) into a context."""
    g = f["lib"]
    ctx.load_folded(layer, g["wq_f"], g["wk_f"], g["wv_f"], g["wo_f"])


def to_dev_bf16(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).cuda()


def from_dev(t) -> np.ndarray:
    import torch
    return t.to(torch.float32).cpu().numpy().astype(np.float64)


def make_context(dims, plan, folded, max_batch, max_seq):
    import paper_2408_04107_b200 as zdc
    ctx = zdc.Context(dims, plan, max_batch, max_seq)
    for l, f in enumerate(folded):
        load_lib_fold(ctx, l, f)
    return ctx
