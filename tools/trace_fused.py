"""Timeline of the fused decode kernel (ZDC_FUSED_TRACE=1): per-CTA globaltimer stamps of the
last launch, summarised as min / median / max microseconds after the earliest CTA start.
Needs the diagnostic build (knobs read from the environment, csrc/knobs.h):

    ZDC_BUILD_VARIANT=debug ZDC_BUILD_DEFS=-DZDC_DEBUG_KNOBS python -m paper_2408_04107_b200.build
    ZDC_LIB_PATH=$PWD/paper_2408_04107_b200/libzdc_debug.so ZDC_FUSED_TRACE=1 \
        python tools/trace_fused.py [--layers 4] [--ctx 2048] [--batch 1]
"""
import argparse
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04107_b200 as zdc  # noqa: E402
import zdc_synth as Z  # noqa: E402

NAMES = {0: "kernel start", 13: "layer start", 1: "x staged", 2: "phase1 done", 3: "barrier1 out", 4: "phase2 done", 5: "barrier2 out",
         6: "merge done", 7: "end", 8: "prod: ph1 issued", 9: "prod: ph2 issued", 10: "prod: all issued",
         11: "ph2 rows done / cl: ph3 done", 12: "partials staged", 13: "layer start", 14: "first KV slot ready", 15: "first W_O slot ready"}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--layers", type=int, default=4)
    p.add_argument("--ctx", type=int, default=2048)
    p.add_argument("--batch", type=int, default=1)
    p.add_argument("--steps", type=int, default=8)
    p.add_argument("--show", type=int, default=4, help="launches to print (the last ones)")
    p.add_argument("--chain", action="store_true", help="one chained zdc_decode call per step")
    p.add_argument("--mode", default="auto", help="zdc_decode_mode: auto / fused / cluster / separate")
    args = p.parse_args()
    dev = torch.device("cuda", 0)
    zdc.decode_mode(args.mode)
    base = Z.dims_of(2)
    L, B, S = args.layers, args.batch, args.ctx
    dims = Z.Dims(L, base.d_model, base.n_heads, base.n_kv_heads, base.d_head)
    d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
    ctx = zdc.Context(dims, Z.plan_uniform(L, 64), B, S + args.steps + 8)
    g = torch.Generator(device=dev).manual_seed(7)
    sc = 1.0 / math.sqrt(d)
    for l in range(L):
        w = [torch.randn(d, nh * dh, device=dev, generator=g) * sc, torch.randn(d, nkv * dh, device=dev, generator=g) * sc,
             torch.randn(d, nkv * dh, device=dev, generator=g) * sc, torch.randn(nh * dh, d, device=dev, generator=g) * sc]
        ctx.load_folded_device(l, *[t.to(torch.bfloat16).contiguous() for t in w])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x = torch.randn(B, S, d, device=dev, generator=g).to(torch.bfloat16)
        y = torch.empty_like(x)
        for l in range(L):
            ctx.prefill(x, y, l, l + 1)
        xb = torch.randn(B, d, device=dev, generator=g).to(torch.bfloat16)
        yb = torch.empty_like(xb)
        for _ in range(args.steps):
            if args.chain:
                ctx.decode(xb, yb, 0, L)
                continue
            for l in range(L):
                ctx.decode(xb, yb, l, l + 1)
    s.synchronize()
    nshow = min(args.show, args.layers * args.steps)
    tr = zdc.trace_read(148, nshow)
    if tr is None:
        print("tracing off (set ZDC_FUSED_TRACE=1)")
        return
    tr = tr.astype(np.int64)
    t0 = tr[0, :, 0][tr[0, :, 0] > 0].min()
    print("last %d launches, us after the first CTA start of the first one shown" % nshow)
    print("%-28s %9s %9s %9s" % ("stamp", "min", "median", "max"))
    for k in range(nshow):
        print("-- launch %d" % k)
        for i in NAMES:
            v = tr[k, :, i]
            v = v[v > 0]
            if len(v) == 0:
                continue
            v = (v - t0) / 1e3
            print("%-28s %9.2f %9.2f %9.2f" % (NAMES[i], v.min(), np.median(v), v.max()))


if __name__ == "__main__":
    main()
