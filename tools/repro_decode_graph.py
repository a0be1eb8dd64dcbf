"""Debug helper: zdc_decode on a non-default stream (library CUDA-graph capture + PDL path)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2408_04107_b200 as zdc
import zdc_synth as Z

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dims = Z.Dims(L, 4096, 32, 32, 128)
ctx = zdc.Context(dims, Z.plan_uniform(L, 64), 1, 2304)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
g = torch.Generator(device="cuda").manual_seed(0)
for l in range(L):
    ws = [torch.randn(4096, 4096, device="cuda", generator=g).to(torch.bfloat16) * 0.02 for _ in range(3)]
    ctx.load_folded_device(l, ws[0], ws[1], ws[2], torch.randn(4096, 4096, device="cuda").to(torch.bfloat16) * 0.02)
x = torch.randn(1, 2048, 4096, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
for l in range(L):
    ctx.prefill(x, y, l, l + 1)
xb = torch.randn(1, 4096, device="cuda").to(torch.bfloat16)
yb = torch.empty_like(xb)
for t in range(3):
    for l in range(L):
        print("decode", t, l, flush=True)
        ctx.decode(xb, yb, l, l + 1)
torch.cuda.synchronize()
print("ok", float(yb.float().abs().sum()))
