"""Small end-to-end run of every kernel family for compute-sanitizer (racecheck / synccheck /
memcheck): prefill (tcgen05 GEMM, attention v4 r<=96 and v3 r=128), decode (fused layer-step at
B=2, split-K GEMM + tcgen05 GQA attention at B=10, decode attention v3 over one / two pools), the token split
(select / rank / pack / append / classify), the FP8 cache, and the GPU fold (K-means + Jacobi)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04107_b200 as zdc  # noqa: E402
import zdc_synth as Z  # noqa: E402


def run(dims, plan, B, S, T, seed):
    ctx = zdc.Context(dims, plan, B, S + T + 2)
    g = torch.Generator(device="cuda").manual_seed(seed)
    for l in range(dims.n_layers):
        w = Z.layer_weights(dims, 1, l)
        f = zdc.fold_weights(dims, w.wq, w.wk, w.wv, w.wo, Z.calibration(dims, 1, l, 256))
        ctx.load_folded(l, f["wq_f"], f["wk_f"], f["wv_f"], f["wo_f"])
    x = torch.randn(B, S, dims.d_model, device="cuda", generator=g).to(torch.bfloat16)
    y = torch.empty_like(x)
    ctx.prefill(x, y)
    xb = torch.randn(B, dims.d_model, device="cuda", generator=g).to(torch.bfloat16)
    yb = torch.empty_like(xb)
    for _ in range(T):
        ctx.decode(xb, yb)
    torch.cuda.synchronize()
    ctx.close()


run(Z.Dims(1, 256, 4, 4, 64), Z.plan_uniform(1, 32), 2, 160, 3, 1)                 # v4, fused decode
run(Z.Dims(1, 256, 8, 2, 64), Z.plan_uniform(1, 64), 10, 140, 3, 2)                # GQA: split-K GEMM + TC attn
run(Z.Dims(1, 256, 2, 2, 128), Z.plan_uniform(1, 128), 1, 130, 2, 3)               # v3 (r = 128)
run(Z.Dims(2, 256, 4, 4, 64), Z.plan_split(2, 32, 16, [[0, 1]], [5000]), 2, 150, 3, 4)  # token split (v3 32/16)
run(Z.Dims(2, 384, 4, 4, 128), Z.plan_split(2, 96, 32, [[0, 1]], [5000]), 3, 140, 3, 6)  # token split (v3 96/32)
run(Z.Dims(1, 256, 4, 4, 64), Z.plan_uniform(1, 64), 10, 120, 3, 7)                # B > 8 uniform (v3 64/0)
p8 = Z.plan_uniform(1, 32)
p8.kv_fp8 = 1
run(Z.Dims(1, 256, 4, 4, 64), p8, 2, 150, 3, 5)                                    # FP8 cache
d = Z.Dims(1, 128, 2, 2, 64)
w = Z.layer_weights(d, 1, 0)
zdc.fold_weights_gpu(d, w.wq, w.wk, w.wv, w.wo, Z.calibration(d, 1, 0, 512), k_clusters=64, kmeans_iters=2)
print("sanitize run done")
