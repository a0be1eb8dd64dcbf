"""One c4-shaped layer (Llama-2-70B: d 8192, 64 heads, 8 KV heads, r 64), batch 64: prefill of
`--prompt` tokens then `--steps` decode steps through zdc_decode (separate kernels: split-K
tcgen05 projections + the tcgen05 GQA decode attention).  For ncu captures of the decode kernels:
    ncu --set full -k regex:decode_attn_tc -s 1 -c 1 python tools/c4_decode_once.py
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
p.add_argument("--prompt", type=int, default=8192)
p.add_argument("--batch", type=int, default=64)
p.add_argument("--steps", type=int, default=3)
args = p.parse_args()
dev = torch.device("cuda", 0)
full = Z.dims_of(4)
dims = Z.Dims(1, full.d_model, full.n_heads, full.n_kv_heads, full.d_head)
d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
B, S = args.batch, args.prompt
ctx = zdc.Context(dims, Z.plan_uniform(1, 64), B, S + args.steps + 2)
g = torch.Generator(device=dev).manual_seed(5)
sc = 1.0 / math.sqrt(d)
w = [torch.randn(d, nh * dh, device=dev, generator=g) * sc, torch.randn(d, nkv * dh, device=dev, generator=g) * sc,
     torch.randn(d, nkv * dh, device=dev, generator=g) * sc, torch.randn(nh * dh, d, device=dev, generator=g) * sc]
ctx.load_folded_device(0, *[t.to(torch.bfloat16).contiguous() for t in w])
x = torch.randn(B, S, d, device=dev, generator=g).to(torch.bfloat16)
y = torch.empty_like(x)
ctx.prefill(x, y)
xb = torch.randn(B, d, device=dev, generator=g).to(torch.bfloat16)
yb = torch.empty_like(xb)
for _ in range(args.steps):
    ctx.decode(xb, yb)
torch.cuda.synchronize()
print("c4 layer: prefill %d x %d, %d decode steps done" % (B, S, args.steps))
