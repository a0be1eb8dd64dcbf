"""One config-3 group (Llama-2-13B shape, 4 layers: the representative + 3 that reuse its classes,
token split g = 0.5, r^i 96 / r^u 32), batch 32: prefill of `--prompt` tokens (per-layer calls, same
x) then `--steps` decode steps.  For ncu launch lists / captures of the split decode kernels:
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -c 200 python tools/c3_decode_once.py
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04107_b200 as zdc  # noqa: E402
import zdc_synth as Z  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--prompt", type=int, default=1024)
p.add_argument("--batch", type=int, default=32)
p.add_argument("--steps", type=int, default=2)
p.add_argument("--mode", type=int, default=1, help="importance mode: 0 raw, 1 per-key mean")
args = p.parse_args()
dev = torch.device("cuda", 0)
full = Z.dims_of(3)
L = 4
dims = Z.Dims(L, full.d_model, full.n_heads, full.n_kv_heads, full.d_head)
d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
B, S = args.batch, args.prompt
plan = Z.plan_split(L, 96, 32, [list(range(L))], [5000], args.mode)
ctx = zdc.Context(dims, plan, B, S + args.steps + 2)
g = torch.Generator(device=dev).manual_seed(5)
sc = 1.0 / math.sqrt(d)
for l in range(L):
    w = [torch.randn(d, nh * dh, device=dev, generator=g) * sc, torch.randn(d, nkv * dh, device=dev, generator=g) * sc,
         torch.randn(d, nkv * dh, device=dev, generator=g) * sc, torch.randn(nh * dh, d, device=dev, generator=g) * sc]
    ctx.load_folded_device(l, *[t.to(torch.bfloat16).contiguous() for t in w])
x = torch.randn(B, S, d, device=dev, generator=g).to(torch.bfloat16)
y = torch.empty_like(x)
for l in range(L):
    ctx.prefill(x, y, l, l + 1)
xb = torch.randn(B, d, device=dev, generator=g).to(torch.bfloat16)
yb = torch.empty_like(xb)
for _ in range(args.steps):
    for l in range(L):
        ctx.decode(xb, yb, l, l + 1)
torch.cuda.synchronize()
print("c3 group: prefill %d x %d, %d decode steps x %d layers done" % (B, S, args.steps, L))
