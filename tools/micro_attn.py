"""Microbenchmark of the a3 kernels alone at the c2 shapes (CUDA graph of `reps` launches).

prefill: B=1, S=2048, 32 heads, r=64 (FLOPs = 4 r N_h S(S+1)/2); decode: 32 KV heads, r=64,
context `len`, rotating through 8 caches (more bytes than L2)."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04107_b200 as zdc  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
reps = 20
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
out = {}
if which in ("both", "prefill"):
    B, S, Nh, r = 1, 2048, 32, 64
    q = torch.randn(B, S, Nh * r, device="cuda").to(torch.bfloat16)
    k = torch.randn(B, Nh, S, r, device="cuda").to(torch.bfloat16)
    v = torch.randn(B, Nh, S, r, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty(B, Nh, S, device="cuda")
    zdc.prefill_attention_bf16(q, k, v, o, lse, scale=1 / math.sqrt(128))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            zdc.prefill_attention_bf16(q, k, v, o, lse, scale=1 / math.sqrt(128))
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    flops = 4.0 * r * Nh * B * S * (S + 1) / 2
    out["prefill_attention"] = {"us": round(us, 2), "TFLOPs": round(flops / us / 1e6, 1)}
if which in ("both", "decode"):
    B, Nh, Nkv, r, cap = 1, 32, 32, 64, 2304
    length = int(sys.argv[2]) if len(sys.argv) > 2 else 2176
    caches = [(torch.randn(B, Nkv, cap, r, device="cuda").to(torch.bfloat16),
               torch.randn(B, Nkv, cap, r, device="cuda").to(torch.bfloat16)) for _ in range(8)]
    q = torch.randn(B, Nh * r, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty(B, Nh, device="cuda")
    ws = zdc.decode_attention_bf16(q, caches[0][0], caches[0][1], o, length, lse)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps * 4):
            zdc.decode_attention_bf16(q, caches[i % 8][0], caches[i % 8][1], o, length, lse, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * 4)
    byts = B * Nkv * length * 2 * r * 2 + 2 * B * Nh * r * 2
    out["decode_attention"] = {"len": length, "us": round(us, 2), "GBs": round(byts / us / 1e3, 1)}
out["env"] = {k: v for k, v in os.environ.items() if k.startswith("ZDC_")}
print(json.dumps(out))
