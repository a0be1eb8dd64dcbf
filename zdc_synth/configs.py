"""Workload shapes of BASELINE.json `configs` (names, dims, plans). No method arithmetic.

Ranks are integers (reading c6: the ABI takes integer ranks; where the
paper gives a drop ratio p, r = ceil((1-p) d_h)).  g is in basis
points (reading c11).
"""
from __future__ import annotations

import dataclasses
from typing import List


@dataclasses.dataclass(frozen=True)
class Dims:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_head: int

    @property
    def group(self) -> int:
        return self.n_heads // self.n_kv_heads


@dataclasses.dataclass
class Plan:
    """Per-layer compression plan (PAPER.md:1483-1498 {g^l, p_QK^i, p_QK^u, p_VL^i, p_VL^u}, as ranks)."""
    r_qk_imp: List[int]
    r_qk_unimp: List[int]
    r_vl_imp: List[int]
    r_vl_unimp: List[int]
    g_bp: List[int]          # important fraction in basis points; 10000 = no token split
    group_rep: List[int]     # representative layer of each layer's group
    importance_mode: int = 0  # 0 = raw sum_h sum_k exp(s); 1 = per-key mean
    kv_fp8: int = 0           # 1 = FP8 E4M3 compressed cache with a per-row scale (NEXT-4, GEAR-ZDC)

    @property
    def n_layers(self) -> int:
        return len(self.g_bp)


def plan_uniform(n_layers: int, r_qk: int, r_vl: int | None = None) -> Plan:
    r_vl = r_qk if r_vl is None else r_vl
    return Plan([r_qk] * n_layers, [r_qk] * n_layers, [r_vl] * n_layers, [r_vl] * n_layers,
                [10000] * n_layers, list(range(n_layers)), 0)


def plan_split(n_layers: int, r_imp: int, r_unimp: int, groups: List[List[int]],
               g_bp_per_group: List[int], importance_mode: int = 0) -> Plan:
    rep = [0] * n_layers
    g_bp = [10000] * n_layers
    for gi, layers in enumerate(groups):
        for l in layers:
            rep[l] = layers[0]
            g_bp[l] = g_bp_per_group[gi]
    return Plan([r_imp] * n_layers, [r_unimp] * n_layers, [r_imp] * n_layers, [r_unimp] * n_layers,
                g_bp, rep, importance_mode)


def c3_plan(n_layers: int = 40, importance_mode: int = 0) -> Plan:
    """Config 3: 10 groups of 4 layers, g_bp = round(2500 + 5000 k / 9) for group k."""
    n_groups = 10
    per = n_layers // n_groups
    groups = [list(range(k * per, (k + 1) * per)) for k in range(n_groups)]
    g = [int(round(2500 + 5000 * k / 9)) for k in range(n_groups)]
    return plan_split(n_layers, 96, 32, groups, g, importance_mode)


CONFIGS = {
    1: dict(name="c1_tiny", dims=Dims(1, 64, 2, 2, 32), B=1, S=128, r=16, decode_steps=8),
    2: dict(name="c2_llama2_7b", dims=Dims(32, 4096, 32, 32, 128), B=1, S=2048, r=64, decode_steps=256),
    3: dict(name="c3_llama2_13b_split", dims=Dims(40, 5120, 40, 40, 128), B=32, S=1024, r=96, r_u=32,
            decode_steps=1024),
    4: dict(name="c4_llama2_70b_gqa", dims=Dims(80, 8192, 64, 8, 128), B=64, S=8192, r=64, decode_steps=256),
    5: dict(name="c5_sp_llama2_7b", dims=Dims(32, 4096, 32, 32, 128), B=1, S=32768, r=64, decode_steps=0),
}


def dims_of(config_id: int, n_layers: int | None = None) -> Dims:
    d = CONFIGS[config_id]["dims"]
    if n_layers is None:
        return d
    return Dims(n_layers, d.d_model, d.n_heads, d.n_kv_heads, d.d_head)
