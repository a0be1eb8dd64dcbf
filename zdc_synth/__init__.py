"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the ZDC method (no fold, no projection, no
attention, no selection).  It only draws the seeded random tensors both sides
receive, rounded to BF16 (round-to-nearest-even) before either side sees them,
following the recipe in DESIGN.md §"Synthetic inputs".

Generator: ``np.random.default_rng([seed, config_id, layer, tensor_id, index])``
tensor_id: 0 = X (prompt), 1 = X_c (calibration), 2 = B_g (QK basis),
3 = G_h (Q), 4 = G'_g (K), 5 = B'_g (VO basis), 6 = G''_g (V), 7 = H_h (O),
8 = decode-step inputs.

Weight recipe (makes Lemma 2's common-R premise true and mimics the paper's
"many near-zero singular values", §4.3):
  s_j = 10^(-2j/(d_h-1))                        (two decades, strictly decreasing)
  W_Q^h = a * G_h diag(s) B_g^T,  W_K^g = a * G'_g diag(s) B_g^T,  a = (4 d_h / sum s^4)^(1/4)
  W_V^g = b * G''_g diag(s) B'_g^T,            b = sqrt(d_h / sum s^2)
  W_O^h = c * B'_g diag(s) H_h^T,              c = sqrt(d_h / (N_h sum s^2))
which gives scaled logits q.k/sqrt(d_h) with standard deviation ~2.
"""
from __future__ import annotations

import dataclasses
import numpy as np

from .configs import CONFIGS, Dims, Plan, plan_uniform, plan_split, dims_of, c3_plan  # noqa: F401

T_X, T_XC, T_BQK, T_GQ, T_GK, T_BVO, T_GV, T_HO, T_DEC = range(9)


def rng(seed: int, config_id: int, layer: int, tensor_id: int, index: int = 0) -> np.random.Generator:
    return np.random.default_rng([int(seed), int(config_id), int(layer), int(tensor_id), int(index)])


def round_bf16(a) -> np.ndarray:
    """fp64 -> fp32 -> bf16 (round to nearest even) -> fp64. Input conditioning only."""
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def to_bf16_bits(a) -> np.ndarray:
    """fp64/fp32 array that is already bf16-representable -> uint16 bit pattern."""
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))
    return (f.view(np.uint32) >> 16).astype(np.uint16)


def orthonormal(g: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    """rows x cols matrix with orthonormal columns, unique (sign of R's diagonal folded in)."""
    q, r = np.linalg.qr(g.standard_normal((rows, cols)))
    return q * np.sign(np.diag(r))[None, :]


def spectrum(d_head: int) -> np.ndarray:
    j = np.arange(d_head, dtype=np.float64)
    return 10.0 ** (-2.0 * j / (d_head - 1))


@dataclasses.dataclass
class LayerWeights:
    wq: np.ndarray  # [d][Nh*dh]
    wk: np.ndarray  # [d][Nkv*dh]
    wv: np.ndarray  # [d][Nkv*dh]
    wo: np.ndarray  # [Nh*dh][d]


def layer_weights(dims: Dims, config_id: int, layer: int, seed: int = 0,
                  logit_scale: float = 1.0, qk_rank: int | None = None,
                  vo_rank: int | None = None, round_to_bf16: bool = True) -> LayerWeights:
    """Unfolded BF16-rounded weights of one attention layer (fp64 arrays).

    logit_scale multiplies a (logits scale as logit_scale^2); qk_rank/vo_rank, if
    given, zero the spectrum beyond that rank (the low-rank construction of pin P4,
    which needs round_to_bf16=False to stay exactly low-rank).
    """
    d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
    G = nh // nkv
    s = spectrum(dh)
    a = (4.0 * dh / np.sum(s ** 4)) ** 0.25 * logit_scale
    b = np.sqrt(dh / np.sum(s ** 2))
    c = np.sqrt(dh / (nh * np.sum(s ** 2)))
    s_qk = s.copy()
    s_vo = s.copy()
    if qk_rank is not None:
        s_qk[qk_rank:] = 0.0
    if vo_rank is not None:
        s_vo[vo_rank:] = 0.0
    wq = np.empty((d, nh * dh))
    wk = np.empty((d, nkv * dh))
    wv = np.empty((d, nkv * dh))
    wo = np.empty((nh * dh, d))
    for g in range(nkv):
        Bg = orthonormal(rng(seed, config_id, layer, T_BQK, g), dh, dh)
        Bp = orthonormal(rng(seed, config_id, layer, T_BVO, g), dh, dh)
        Gk = orthonormal(rng(seed, config_id, layer, T_GK, g), d, dh)
        Gv = orthonormal(rng(seed, config_id, layer, T_GV, g), d, dh)
        wk[:, g * dh:(g + 1) * dh] = a * (Gk * s_qk[None, :]) @ Bg.T
        wv[:, g * dh:(g + 1) * dh] = b * (Gv * s_vo[None, :]) @ Bp.T
        for h in range(g * G, (g + 1) * G):
            Gh = orthonormal(rng(seed, config_id, layer, T_GQ, h), d, dh)
            Hh = orthonormal(rng(seed, config_id, layer, T_HO, h), d, dh)
            wq[:, h * dh:(h + 1) * dh] = a * (Gh * s_qk[None, :]) @ Bg.T
            wo[h * dh:(h + 1) * dh, :] = c * (Bp * s_vo[None, :]) @ Hh.T
    if not round_to_bf16:
        return LayerWeights(wq, wk, wv, wo)
    return LayerWeights(round_bf16(wq), round_bf16(wk), round_bf16(wv), round_bf16(wo))


def prompt(dims: Dims, config_id: int, B: int, S: int, seed: int = 0, layer: int = 0) -> np.ndarray:
    """x [B][S][d], i.i.d. N(0,1), BF16-rounded."""
    return round_bf16(rng(seed, config_id, layer, T_X, 0).standard_normal((B, S, dims.d_model)))


def calibration(dims: Dims, config_id: int, layer: int, n_calib: int = 4096, seed: int = 0) -> np.ndarray:
    """X_c [n_calib][d] for one layer (stands in for the paper's pruned history)."""
    return round_bf16(rng(seed, config_id, layer, T_XC, 0).standard_normal((n_calib, dims.d_model)))


def decode_input(dims: Dims, config_id: int, B: int, step: int, seed: int = 0, layer: int = 0) -> np.ndarray:
    """x [B][d] for decode step `step`."""
    return round_bf16(rng(seed, config_id, layer, T_DEC, step).standard_normal((B, dims.d_model)))
