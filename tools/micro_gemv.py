"""Microbenchmark of the decode projection kernel (zdc_gemv_bf16) in isolation.

Rotates through 8 distinct weight matrices (more bytes than L2) inside one CUDA graph of
`reps` launches and reports the average time per launch and the achieved HBM bandwidth.
Usage: python tools/micro_gemv.py [N K B reps]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04107_b200 as zdc  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 6144
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 64
nmat = 8
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(nmat)]
x = torch.randn(B, K, device="cuda").to(torch.bfloat16)
y = torch.empty(B, N, device="cuda", dtype=torch.bfloat16)
for w in ws:
    zdc.gemv_bf16(w, x, y)
torch.cuda.synchronize()
ref = (x.float() @ ws[-1].float().t())
err = float((y.float() - ref).abs().max() / ref.abs().max())
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(reps):
        zdc.gemv_bf16(ws[i % nmat], x, y)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
g.replay()
e1.record(s)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
gbs = (N * K * 2 + B * K * 2 + B * N * 2) / us / 1e3
print(json.dumps({"N": N, "K": K, "B": B, "us": round(us, 2), "GBs": round(gbs, 1), "err": err,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("ZDC_")}}))
