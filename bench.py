#!/usr/bin/env python
"""bench.py — ZDC compressed-attention hot path on B200 (BASELINE.json metric, configs[1] = c2).

Workload (config "c2_llama2_7b"): Llama-2-7B-shaped attention stack, 32 layers, d=4096, 32 heads,
d_h=128, rank r = d_h/2 = 64 (uniform plan), batch 1, prompt 2048 tokens, then 256 decode steps.
One STEP = the whole hot path over one request: prefill of the 2048-token prompt through the 32
layers (a1 QKV projection + fused cache append, a3 causal attention, a5 output projection), then
256 decode steps x 32 layers.  value = tokens processed per second (2048 prompt + 256 generated
per step per GPU), whole job; prefill and decode tok/s are reported alongside.

Timing: CUDA events on the launching stream, W warm-up steps, K timed steps bracketed by a
barrier + synchronize, max over ranks.  Inputs are larger than L2 (2.1 GB of folded weights
stream through every step), so no explicit flush.  Each layer is called with the same seeded x
(no chaining: a chained stack shrinks activations towards underflow), 32
per-layer calls captured in one CUDA graph for the prefill and one per decode step.

N > 1: independent replicas (decode is "replicas only"; the c2 prefill fits one GPU), weak scaling.
--impl reference: the fp64 CPU oracle (oracle/) on a bounded sample, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compressed-attn prefill tok/s & decode tok/s per B200 (% roofline); SP K/V exchange GB/s"
_T0 = time.time()


def log(msg):
    sys.stderr.write("[bench %7.1fs] %s\n" % (time.time() - _T0, msg))
    sys.stderr.flush()
CONFIG_NAME = "c2_llama2_7b"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1,
                   help="GPUs of this node; without WORLD_SIZE in the environment bench.py launches itself "
                        "once per GPU through torch.distributed.run (127.0.0.1 rendezvous)")
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="zdc", choices=["zdc", "reference"])
    p.add_argument("--decode-steps", type=int, default=256)
    p.add_argument("--prompt", type=int, default=2048)
    p.add_argument("--rank", type=int, default=64)
    p.add_argument("--layers", type=int, default=32)
    p.add_argument("--decode-calls", default="layer", choices=["layer", "chain"],
                   help="decode step as 32 per-layer zdc_decode calls (same x per layer) or one chained call")
    p.add_argument("--decode-mode", default="auto", choices=["auto", "fused", "cluster", "separate"],
                   help="decode kernels for B <= 8 (zdc_decode_mode): auto = persistent fused layer-step where "
                        "supported")
    p.add_argument("--configs", default="c3,c4",
                   help="per-layer prefill/decode measurements of these configs at N = 1 ('' to skip)")
    p.add_argument("--sp-seq", type=int, default=32768, help="SP prefill prompt length (c5), run when N > 1")
    p.add_argument("--sp-layers", type=int, default=32)
    p.add_argument("--sp", action="store_true", help="also run the SP prefill at N = 1 (P = 1, no exchange)")
    p.add_argument("--no-sp", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-fold", action="store_true", help="skip the NEXT-3 GPU fold timing")
    p.add_argument("--no-fp8", action="store_true", help="skip the NEXT-4 FP8 cache decode timing")
    p.add_argument("--no-uncompressed", action="store_true",
                   help="skip the r = d_h (R = I) baseline and the torch SDPA / matmul comparison")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--profile-only", action="store_true", help="one eager step (for ncu), no JSON")
    p.add_argument("--launch-probe", action="store_true",
                   help="test hook: each rank joins a gloo group, all-reduces its rank and prints one JSON line")
    return p.parse_args()


# ------------------------------------------------------------------------------------ peaks
def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return dict(hbm=float(d["hbm_gbs"]), tf=float(d["bf16_tflops"]),
                    tf_sus=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), src="measured")
    return dict(hbm=6650.0, tf=1590.0, tf_sus=1400.0, src="fallback")


# ------------------------------------------------------------------------------------ algorithmic work
# SURVEY.md §8(d) "Algorithmic counts": FLOPs at the plan ranks (causal attention over the
# S(S+1)/2 pairs; no padding, masked tiles or exp), bytes = packed weights read once + K'/V' at the
# packed widths + append + x/y.  Pinned by tests/test_bench_work.py against §8(d)'s figures.
def prefill_layer_flops(d, nh, nkv, r, B, S):
    """{'a1', 'a3', 'a5'} FLOPs of one prefill layer (uniform rank r = r_k = r_v)."""
    n_qkv = nh * r + 2 * nkv * r
    return {"a1": 2.0 * B * S * n_qkv * d, "a3": 4.0 * r * nh * B * S * (S + 1) / 2.0, "a5": 2.0 * B * S * nh * r * d}


def decode_layer_bytes(d, nh, nkv, r, B, ctx, ko=None):
    """{'a1', 'a3', 'a5'} algorithmic bytes of one decode layer-step at context `ctx` (uniform rank):
    the packed weights, K'/V' of ctx cached tokens, Q'/O' and x/y rows (bf16)."""
    ko = nh * r if ko is None else ko
    n_qkv = nh * r + 2 * nkv * r
    return {"a1": n_qkv * d * 2 + B * d * 2 + B * n_qkv * 2,
            "a3": B * nkv * ctx * 2 * r * 2 + 2 * B * nh * r * 2,
            "a5": d * ko * 2 + B * ko * 2 + B * d * 2}


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int, period_ms: int = 200):
        self.dev, self.proc, self.lines, self.period = dev, None, [], period_ms

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                          "-lms", str(self.period), "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout_s: float = 3.0):
        """Block until nvidia-smi has printed its first sample (it starts ~0.5 s late), so the
        timed region that follows is sampled from its start."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout_s:
            time.sleep(0.01)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for i, n in enumerate(names):
                if f[5 + i].lower().startswith("active"):
                    reasons.add(n)
        loaded = [s for s, p in zip(sm, pw) if p > 200.0] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------------------------ oracle baseline
def oracle_sample(n_decode: int = 16, prompt: int = 2048):
    """The fp64 oracle as it stands, on a bounded sample of the c2 workload: one layer's fold
    (untimed, like the GPU path's), one layer prefill of the full prompt, n_decode decode steps.
    BLAS threads are pinned (threadpoolctl) to the CPUs this process may run on.
    Returns (seconds_prefill_layer, seconds_per_decode_layer_step, cores) with cores =
    {"threads": BLAS threads used, "affinity": len(sched_getaffinity), "cpu_count": os.cpu_count()}."""
    import numpy as np
    import oracle as O
    import zdc_synth as Z
    dims = Z.dims_of(2, n_layers=1)
    plan = Z.plan_uniform(1, 64)
    w = Z.layer_weights(dims, 2, 0)
    xc = Z.calibration(dims, 2, 0, 4096)
    folded = O.fold_layer(dims, w.wq, w.wk, w.wv, w.wo, xc)
    x = Z.prompt(dims, 2, 1, prompt, seed=21)
    m = O.OracleModel(dims, plan, [folded])
    aff = len(os.sched_getaffinity(0))
    from threadpoolctl import threadpool_info, threadpool_limits
    with threadpool_limits(limits=aff):
        nthreads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
        t0 = time.perf_counter()
        m.prefill(x)
        t1 = time.perf_counter()
        for s in range(n_decode):
            m.decode(Z.decode_input(dims, 2, 1, s))
        t2 = time.perf_counter()
    cores = {"threads": nthreads, "affinity": aff, "cpu_count": os.cpu_count()}
    return t1 - t0, (t2 - t1) / n_decode, cores


def oracle_step_tok_s(t_pre_layer, t_dec_layer, L, S, T, B=1):
    step = L * t_pre_layer + L * T * t_dec_layer
    return B * (S + T) / step, step


# ------------------------------------------------------------------------------------ kernels alone
def _time_graph(torch, stream, fn, reps):
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps  # ms per launch


def isolated_kernels(zdc, torch, stream, dev, d, nh, nkv, r, S, T, B, L, step_ms):
    """Each kernel of the c2 step alone: achieved algorithmic bytes (decode, HBM-bound) or FLOPs
    (prefill, tensor-bound) per launch / average launch time.  Returns ({name: roofline}, {name:
    estimated share of the step = time alone x launches per step / step time})."""
    peaks = load_peaks()
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    g = torch.Generator(device=dev).manual_seed(77)
    bf = torch.bfloat16
    Nqkv = nh * r + 2 * nkv * r
    ko = ((nh * r + 63) // 64) * 64
    avg_ctx = int(S + (T + 1) / 2.0)
    cap = S + T
    res = {}
    # decode projections (B rows): 8 weight copies rotate (400 MB > L2)
    for name, N, K in (("a1_decode_gemv", Nqkv, d), ("a5_decode_gemv", d, ko)):
        ws = [torch.randn(N, K, device=dev, generator=g).to(bf) for _ in range(8)]
        x = torch.randn(B, K, device=dev, generator=g).to(bf)
        y = torch.empty(B, N, device=dev, dtype=bf)
        ms = _time_graph(torch, stream, lambda i: zdc.gemv_bf16(ws[i % 8], x, y), 64)
        res[name] = ("hbm", decode_layer_bytes(d, nh, nkv, r, B, avg_ctx, ko)["a1" if name.startswith("a1") else "a5"],
                     ms, L * T)
        del ws
    # decode attention at the average context of the 256 decode steps: 8 caches rotate
    caches = [(torch.randn(B, nkv, cap, r, device=dev, generator=g).to(bf),
               torch.randn(B, nkv, cap, r, device=dev, generator=g).to(bf)) for _ in range(8)]
    q = torch.randn(B, nh * r, device=dev, generator=g).to(bf)
    o = torch.empty_like(q)
    lse = torch.empty(B, nh, device=dev)
    wsp = zdc.decode_attention_bf16(q, caches[0][0], caches[0][1], o, avg_ctx, lse)
    ms = _time_graph(torch, stream, lambda i: zdc.decode_attention_bf16(
        q, caches[i % 8][0], caches[i % 8][1], o, avg_ctx, lse, workspace=wsp), 64)
    res["a3_decode_attention"] = ("hbm", decode_layer_bytes(d, nh, nkv, r, B, avg_ctx, ko)["a3"], ms, L * T)
    del caches
    # prefill (tensor-bound): the two projection GEMMs and the causal attention
    xa = torch.randn(B * S, d, device=dev, generator=g).to(bf)
    wq = torch.randn(Nqkv, d, device=dev, generator=g).to(bf)
    yq = torch.empty(B * S, Nqkv, device=dev, dtype=bf)
    ms = _time_graph(torch, stream, lambda i: zdc.gemm_bf16(xa, wq, yq), 10)
    pf = prefill_layer_flops(d, nh, nkv, r, B, S)
    res["a1_prefill_gemm"] = ("tensor", pf["a1"], ms, L)
    oa = torch.randn(B * S, ko, device=dev, generator=g).to(bf)
    wo = torch.randn(d, ko, device=dev, generator=g).to(bf)
    yo = torch.empty(B * S, d, device=dev, dtype=bf)
    ms = _time_graph(torch, stream, lambda i: zdc.gemm_bf16(oa, wo, yo), 10)
    res["a5_prefill_gemm"] = ("tensor", pf["a5"], ms, L)
    qa = torch.randn(B, S, nh * r, device=dev, generator=g).to(bf)
    ka = torch.randn(B, nkv, S, r, device=dev, generator=g).to(bf)
    va = torch.randn(B, nkv, S, r, device=dev, generator=g).to(bf)
    pa = torch.empty_like(qa)
    la = torch.empty(B, nh, S, device=dev)
    ms = _time_graph(torch, stream, lambda i: zdc.prefill_attention_bf16(qa, ka, va, pa, la,
                                                                         scale=1.0 / math.sqrt(128)), 10)
    res["a3_prefill_attention"] = ("tensor", pf["a3"], ms, L)
    kernels, shares = {}, {}
    for k, (bound, work, ms, per_step) in res.items():
        s = ms / 1e3
        if bound == "hbm":
            ach, peak, unit = work / s / 1e9, peaks["hbm"], "GB/s"
        else:
            # a kernel timed alone: the burst GEMM peak (MEASURED_PEAKS bf16_tflops)
            ach, peak, unit = work / s / 1e12, peaks["tf"], "TFLOP/s"
        kernels[k] = {"bound": bound, "achieved": round(ach, 1), "peak": peak, "unit": unit,
                      "frac": round(ach / peak, 4), "avg_us": round(ms * 1e3, 2), "launches_per_step": per_step,
                      "work_per_launch": work, "traffic": traffic.get(k)}
        shares[k] = ms * per_step / step_ms
        kernels[k]["est_share_of_step"] = round(shares[k], 4)
    return kernels, shares


# ------------------------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    L, S, T = args.layers, args.prompt, args.decode_steps
    vals = []
    for i in range(args.warmup + args.steps):
        tp, td, cores = oracle_sample(n_decode=4, prompt=512 if i < args.warmup else S)
        if i >= args.warmup:
            vals.append((tp, td))
    tp = statistics.median(v[0] for v in vals)
    td = statistics.median(v[1] for v in vals)
    v, step_s = oracle_step_tok_s(tp, td, L, S, T)
    sample = ("per step: 1 layer fp64 prefill of S=%d + 4 decode steps (oracle/); value extrapolated to %d layers "
              "x (prefill + %d decode steps) = %.1f s per full-workload step" % (S, L, T, step_s))
    sample_ms = (tp + 4 * td) * 1e3  # the timed part of one sample (prefill + 4 decode steps)
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tok/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup,
           # what was actually timed per step (the bounded sample, incl. its untimed fold); the
           # full-workload step time behind `value` is an extrapolation, labelled as such
           "ms_per_step": sample_ms,
           "ms_per_step_kind": "measured: the timed part of one bounded sample (1 layer prefill + 4 decode steps)",
           "ms_per_full_step_extrapolated": step_s * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": CONFIG_NAME, "layers": L, "prompt": S, "decode_steps": T, "batch": 1, "rank": 64},
           "cpu_baseline": {"value": v, "unit": "tok/s", "cores": cores["threads"], "cores_detail": cores,
                            "kind": "oracle", "sample": sample},
           "e2e": {"value": v, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------ SP (a6)
def sp_bench(args, zdc, torch, dist, rank, world, dev, stream, dataflow="allgather"):
    """Sequence-parallel prefill (configs[4], c5): the c2 layer stack over a S_total-token prompt
    sharded zigzag over the `world` ranks, compressed K'/V' all-gathered in place per layer with
    NCCL (zdc_sp_prefill).  Reports the SP prefill tok/s (S_total / max-over-ranks time), and the
    exchange GB/s per GPU = bytes received per layer / time of the all-gather alone (CUDA events
    around the NCCL call on the launch stream, nothing concurrent: NCCL's bus bandwidth)."""
    import zdc_synth as Z
    S_tot, Lsp, r = args.sp_seq, args.sp_layers, args.rank
    base = Z.dims_of(5)
    dims = Z.Dims(Lsp, base.d_model, base.n_heads, base.n_kv_heads, base.d_head)
    d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
    ctx = zdc.Context(dims, Z.plan_uniform(Lsp, r), 1, S_tot)
    g = torch.Generator(device=dev).manual_seed(4321)
    sc = 1.0 / math.sqrt(d)
    for l in range(Lsp):
        w = [torch.randn(d, nh * dh, device=dev, generator=g) * sc, torch.randn(d, nkv * dh, device=dev, generator=g) * sc,
             torch.randn(d, nkv * dh, device=dev, generator=g) * sc, torch.randn(nh * dh, d, device=dev, generator=g) * sc]
        ctx.load_folded_device(l, *[t.to(torch.bfloat16).contiguous() for t in w])
        del w
    uid = [zdc.comm_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    ctx.comm_init(uid[0], rank, world)
    n_local = S_tot // world
    x = torch.randn(1, n_local, d, device=dev, generator=g).to(torch.bfloat16)
    y = torch.empty_like(x)
    for _ in range(2):  # warm-up (NCCL connection set-up, kernel attributes)
        ctx.reset()
        ctx.sp_prefill(x, y, S_tot, layout=2 if dataflow == "allgather" else 1, stream=stream, dataflow=dataflow)
    torch.cuda.synchronize()
    reps = max(1, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    ms = 0.0
    for _ in range(reps):
        ctx.reset()
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.sp_prefill(x, y, S_tot, layout=2 if dataflow == "allgather" else 1, stream=stream, dataflow=dataflow)
        e1.record(stream)
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
    ms /= reps
    ctx.reset()
    st = ctx.sp_prefill(x, y, S_tot, layout=2 if dataflow == "allgather" else 1, stats=True, stream=stream, dataflow=dataflow)
    torch.cuda.synchronize()
    tt = torch.tensor([ms, st["exchange_ms"], -st["exchange_ms"]], device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms, ex_max, ex_min = float(tt[0]), float(tt[1]), -float(tt[2])
    per_layer_recv = st["bytes_recv"] / Lsp
    ctx.close()
    out = {"workload": "c5_sp_llama2_7b", "dataflow": dataflow, "S_total": S_tot, "layers": Lsp, "P": world,
           "layout": "zigzag, exchange overlapped on a comm stream (layout 2)" if dataflow == "allgather" else "zigzag",
           "rank": r, "ms": ms, "sp_prefill_tok_s": S_tot / (ms / 1e3),
           "bytes_recv_per_gpu_per_layer": per_layer_recv,
           "bytes_recv_uncompressed_per_gpu_per_layer": st["bytes_recv_uncompressed"] / Lsp,
           "compression": (st["bytes_recv"] / st["bytes_recv_uncompressed"]) if st["bytes_recv_uncompressed"] else None,
           "exchange_ms_per_layer_max": ex_max / Lsp, "exchange_fraction_of_prefill": ex_max / st["total_ms"]
           if st["total_ms"] else None}
    if world > 1 and ex_max > 0:
        out["exchange_GBps_per_gpu"] = st["bytes_recv"] / (ex_max / 1e3) / 1e9  # slowest rank
        out["exchange_GBps_per_gpu_best"] = st["bytes_recv"] / (ex_min / 1e3) / 1e9
        out["exchange_frac_of_nvlink_900"] = out["exchange_GBps_per_gpu"] / 900.0
    return out


# ------------------------------------------------------------------------------------ c3 / c4 layers
def config_bench(args, zdc, torch, dev, stream, cid, n_layers=4, T=48, importance_mode=0):
    """Per-layer prefill and decode of config `cid` (3: the whole Llama-2-13B-shaped stack, 40 layers,
    batch 32, prompt 1024, SURVEY.md §8(d)'s plan: 10 groups of 4 layers, g_bp = round(2500 +
    5000 k / 9) for group k, r^i = 96 / r^u = 32, importance mode raw (0) or per-key mean (1);
    4: Llama-2-70B shape, GQA 8 KV heads, batch 64, prompt 8192, r = 64, on `n_layers` layers) with
    timing-only weights (the ideal
    fold of SURVEY.md §8(d)), each layer called separately with the same x (as for c2).  Prefill:
    algorithmic FLOP / time against the bf16 peak; decode: algorithmic bytes (weights at the plan
    ranks + K'/V' at the realised per-token widths + append + x/y) per layer-step / time against
    the HBM peak.  The whole-model figures scale the per-layer time to the config's layer count
    (labelled extrapolated)."""
    import zdc_synth as Z
    cfg = Z.CONFIGS[cid]
    full = cfg["dims"]
    dims = Z.Dims(n_layers, full.d_model, full.n_heads, full.n_kv_heads, full.d_head)
    d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
    B, S, r = cfg["B"], cfg["S"], cfg["r"]
    if cid == 3:
        ru = cfg["r_u"]
        n_layers = full.n_layers
        dims = Z.Dims(n_layers, full.d_model, full.n_heads, full.n_kv_heads, full.d_head)
        plan = Z.c3_plan(n_layers, importance_mode)
    else:
        ru = r
        plan = Z.plan_uniform(n_layers, r)
    ctx = zdc.Context(dims, plan, B, S + T + 4)
    g = torch.Generator(device=dev).manual_seed(4321 + cid)
    sv = torch.tensor([10.0 ** (-2.0 * j / (dh - 1)) for j in range(dh)], device=dev)
    a = (4.0 * dh / float((sv ** 4).sum())) ** 0.25
    bta = math.sqrt(dh / float((sv ** 2).sum()))
    gam = math.sqrt(dh / (nh * float((sv ** 2).sum())))
    for l in range(n_layers):
        wq = (torch.randn(d, nh, dh, device=dev, generator=g) * (a * sv / math.sqrt(d))).reshape(d, nh * dh)
        wk = (torch.randn(d, nkv, dh, device=dev, generator=g) * (a * sv / math.sqrt(d))).reshape(d, nkv * dh)
        wv = (torch.randn(d, nkv, dh, device=dev, generator=g) * (bta * sv / math.sqrt(d))).reshape(d, nkv * dh)
        wo = (torch.randn(nh, dh, d, device=dev, generator=g) * (gam * sv[:, None] / math.sqrt(d))).reshape(nh * dh, d)
        ctx.load_folded_device(l, *[t.to(torch.bfloat16).contiguous() for t in (wq, wk, wv, wo)])
        del wq, wk, wv, wo
    x = torch.randn(B, S, d, device=dev, generator=g).to(torch.bfloat16)
    y = torch.empty_like(x)
    xd = torch.randn(T + 2, B, d, device=dev, generator=g).to(torch.bfloat16)
    xb = torch.empty(B, d, device=dev, dtype=torch.bfloat16)
    yb = torch.empty_like(xb)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def prefill(timed):
        ctx.reset()
        if timed:
            ev[0].record(stream)
        for l in range(n_layers):
            ctx.prefill(x, y, l, l + 1)
        if timed:
            ev[1].record(stream)

    def decode_steps(t0, n, timed):
        if timed:
            ev[2].record(stream)
        for t in range(t0, t0 + n):
            xb.copy_(xd[t])
            for l in range(n_layers):
                ctx.decode(xb, yb, l, l + 1)
        if timed:
            ev[3].record(stream)

    prefill(False)                 # warm-up (kernel attributes)
    decode_steps(0, 2, False)      # warm-up (decode graphs)
    torch.cuda.synchronize()
    prefill(True)
    decode_steps(0, 2, False)
    torch.cuda.synchronize()
    # Decode is timed in its own power regime: the max-power prefill GEMMs just before leave this
    # power-capped box at sw_power_cap with SM clocks of ~800-950 MHz for a while, which would
    # otherwise bleed into the decode window (profiles/r01/NOTES.md); clocks are sampled during it.
    time.sleep(0.5)
    # one decode step (the n_layers per-layer calls) captured as one CUDA graph, as for c2; the
    # device-side cache lengths make it replayable at every position
    g_step = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_step, stream=stream):
        for l in range(n_layers):
            ctx.decode(xb, yb, l, l + 1)
    torch.cuda.synchronize()
    clk = ClockSampler(dev.index if dev.index is not None else 0, period_ms=5)
    clk.start()
    time.sleep(0.1)
    ev[2].record(stream)
    for t in range(2, T + 2):
        xb.copy_(xd[t])
        g_step.replay()
    ev[3].record(stream)
    torch.cuda.synchronize()
    dec_clocks = clk.stop()
    ctx.cache_sync(stream)  # the replays advanced the device lengths only
    pre_ms = ev[0].elapsed_time(ev[1]) / n_layers
    dec_us = ev[2].elapsed_time(ev[3]) * 1e3 / (T * n_layers)
    per_class = None
    if os.environ.get("ZDC_BENCH_CLASS_PROFILE"):  # diagnostics: per-kernel-class time of 2 eager steps
        zdc.profile(True)
        zdc.profile_read()
        decode_steps(T + 2 - 2, 2, False)  # cache has room: S + T + 4 rows
        per_class = {k: (round(v[0] / (2 * n_layers) * 1e3, 1), v[1]) for k, v in zdc.profile_read().items() if v[1]}
        zdc.profile(False)
    # algorithmic work: unpadded ranks (multiples of 16 here: padding = 0)
    nq, nkvr = nh * r, nkv * r
    n_qkv = nq + 2 * nkvr
    flop = sum(prefill_layer_flops(d, nh, nkv, r, B, S).values())
    wbytes = (n_qkv * d + d * nq) * 2
    wI, wU = 2 * nkv * r * 2, 2 * nkv * ru * 2  # bytes per cached token per layer (K' + V')
    groups = None
    if cid == 3:
        kv, groups, imps = 0.0, [], {}
        for l in range(n_layers):
            rl = plan.group_rep[l]
            if rl not in imps:  # the classes the representative layer assigned (prompt + decode)
                imp = np.zeros((B, ctx.cache_length(rl)), dtype=np.uint8)
                zdc._check(zdc.lib().zdc_cache_export(ctx.h, rl, None, None, imp.ctypes.data_as(ctypes.c_void_p),
                                                      None, ctypes.c_void_p(stream.cuda_stream)), "zdc_cache_export")
                imps[rl] = imp
                groups.append({"layers": [rl, rl + 3], "g_bp": plan.g_bp[rl],
                               "important_prompt": round(float(imp[:, :S].mean()), 4),
                               "important_decode": round(float(imp[:, S:S + T + 2].mean()), 4)})
            cum = np.cumsum(imps[rl].astype(np.int64), axis=1)  # important tokens among the first j+1
            for t in range(2, T + 2):
                n_before = S + t  # cached rows the step-t query attends to (+ its own, appended)
                ni = cum[:, n_before - 1]
                kv += float((ni * wI + (n_before - ni) * wU).sum())
        kv /= T * n_layers  # per layer-step, averaged over the layers
        frac_imp_prompt = float(np.mean([v[:, :S].mean() for v in imps.values()]))
        frac_imp_decode = float(np.mean([v[:, S:S + T + 2].mean() for v in imps.values()]))
    else:
        kv = float(B * (S + 2 + (T - 1) / 2.0) * wI)
        frac_imp_prompt = frac_imp_decode = None
    dbytes = wbytes + kv + B * wI + 2 * B * d * 2
    peaks = load_peaks()
    out = {
        "workload": cfg["name"], "layers_measured": n_layers, "layers_model": full.n_layers, "batch": B,
        "prompt": S, "rank": r, "rank_unimportant": ru if cid == 3 else None,
        "prefill": {"ms_per_layer": round(pre_ms, 3), "flop_per_layer": flop,
                    "achieved_tflops": round(flop / (pre_ms / 1e3) / 1e12, 1), "peak": peaks["tf"],
                    "frac": round(flop / (pre_ms / 1e3) / 1e12 / peaks["tf"], 4),
                    # a long region of back-to-back GEMMs: the sustained bf16 peak is the roofline
                    "peak_sustained": peaks["tf_sus"],
                    "frac_sustained": round(flop / (pre_ms / 1e3) / 1e12 / peaks["tf_sus"], 4),
                    "tok_s_model_extrapolated": round(B * S / (pre_ms / 1e3 * full.n_layers), 1)},
        "decode": {"us_per_layer_step": round(dec_us, 2), "bytes_per_layer_step": dbytes,
                   "weight_bytes": wbytes, "kv_bytes_avg": kv,
                   "achieved_gbs": round(dbytes / (dec_us / 1e6) / 1e9, 1), "peak": peaks["hbm"],
                   "frac": round(dbytes / (dec_us / 1e6) / 1e9 / peaks["hbm"], 4), "steps_timed": T,
                   "tok_s_model_extrapolated": round(B / (dec_us / 1e6 * full.n_layers), 1),
                   "clocks": dec_clocks, "timing": "one CUDA graph per decode step, after a 0.5 s idle gap"},
    }
    if per_class:
        out["decode"]["per_class_us_per_layer"] = per_class
    if cid == 3:
        out["importance_mode"] = {0: "raw", 1: "mean"}[importance_mode]
        out["realised_important_fraction"] = {"prompt": round(frac_imp_prompt, 4),
                                              "decode": round(frac_imp_decode, 4), "groups": groups}
    ctx.close()
    del x, y, xd
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------------------------ r = d_h baseline
def _timing_weights(torch, dev, g, d, nh, nkv, dh):
    """Timing-only unfolded weights (the decaying-spectrum recipe of zdc_synth, generated on the device)."""
    sv = torch.tensor([10.0 ** (-2.0 * j / (dh - 1)) for j in range(dh)], device=dev)
    a = (4.0 * dh / float((sv ** 4).sum())) ** 0.25
    bta = math.sqrt(dh / float((sv ** 2).sum()))
    gam = math.sqrt(dh / (nh * float((sv ** 2).sum())))
    wq = (torch.randn(d, nh, dh, device=dev, generator=g) * (a * sv / math.sqrt(d))).reshape(d, nh * dh)
    wk = (torch.randn(d, nkv, dh, device=dev, generator=g) * (a * sv / math.sqrt(d))).reshape(d, nkv * dh)
    wv = (torch.randn(d, nkv, dh, device=dev, generator=g) * (bta * sv / math.sqrt(d))).reshape(d, nkv * dh)
    wo = (torch.randn(nh, dh, d, device=dev, generator=g) * (gam * sv[:, None] / math.sqrt(d))).reshape(nh * dh, d)
    return [t.to(torch.bfloat16).contiguous() for t in (wq, wk, wv, wo)]


def uncompressed_bench(args, zdc, torch, dev, stream, pre_ms_r, dec_ms_r, dec_bytes_r):
    """SURVEY.md §8(d) "Uncompressed baseline": the same kernels at r = d_h with R = I (folding with
    the identity is exact, pin P10), i.e. the uncompressed model run through the library, timed the
    same way as the c2 step (CUDA graphs of per-layer calls); plus each attention kernel alone at
    r and at d_h -- the B200 analogue of the paper's "attention time saved".
    Library comparison (report only, never on the product path): torch SDPA at head dim r / d_h and
    torch.matmul at the c2 projection shapes."""
    import torch.nn.functional as F
    import zdc_synth as Z
    L, S, T, r = args.layers, args.prompt, args.decode_steps, args.rank
    base = Z.dims_of(2)
    dims = Z.Dims(L, base.d_model, base.n_heads, base.n_kv_heads, base.d_head)
    d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
    ctx = zdc.Context(dims, Z.plan_uniform(L, dh), 1, S + T)
    g = torch.Generator(device=dev).manual_seed(999)
    for l in range(L):
        ctx.load_folded_device(l, *_timing_weights(torch, dev, g, d, nh, nkv, dh))
    xp = torch.randn(1, S, d, device=dev, generator=g).to(torch.bfloat16)
    xd = torch.randn(T, 1, d, device=dev, generator=g).to(torch.bfloat16)
    y = torch.empty_like(xp)
    xb = torch.empty(1, d, device=dev, dtype=torch.bfloat16)
    yb = torch.empty_like(xb)
    for l in range(L):  # warm-up (kernel attributes, decode graphs)
        ctx.prefill(xp, y, l, l + 1)
    for l in range(L):
        ctx.decode(xd[0], yb, l, l + 1)
    ctx.reset()
    gp = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gp, stream=stream):
        for l in range(L):
            ctx.prefill(xp, y, l, l + 1)
    gd = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gd, stream=stream):
        for l in range(L):
            ctx.decode(xb, yb, l, l + 1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    pre, dec = [], []
    for i in range(1 + max(1, args.steps)):
        ctx.reset()
        torch.cuda.synchronize()
        ev[0].record(stream)
        gp.replay()
        ev[1].record(stream)
        for t in range(T):
            xb.copy_(xd[t])
            gd.replay()
        ev[2].record(stream)
        torch.cuda.synchronize()
        if i:
            pre.append(ev[0].elapsed_time(ev[1]))
            dec.append(ev[1].elapsed_time(ev[2]))
    ctx.close()
    pre_ms, dec_ms = statistics.median(pre), statistics.median(dec)
    avg_ctx = int(S + (T + 1) / 2.0)
    dec_bytes_u = sum(decode_layer_bytes(d, nh, nkv, dh, 1, avg_ctx).values())
    # each attention kernel alone at r and at d_h (CUDA graph of back-to-back launches)
    attn = {}
    for rr in sorted({r, dh}):
        qa = torch.randn(1, S, nh * rr, device=dev, generator=g).to(torch.bfloat16)
        ka = torch.randn(1, nkv, S + T, rr, device=dev, generator=g).to(torch.bfloat16)
        va = torch.randn(1, nkv, S + T, rr, device=dev, generator=g).to(torch.bfloat16)
        pa = torch.empty_like(qa)
        la = torch.empty(1, nh, S, device=dev)
        ks, vs = ka[:, :, :S].contiguous(), va[:, :, :S].contiguous()
        t_pre = _time_graph(torch, stream, lambda i: zdc.prefill_attention_bf16(qa, ks, vs, pa, la,
                                                                                scale=1.0 / math.sqrt(dh)), 10)
        qd = torch.randn(1, nh * rr, device=dev, generator=g).to(torch.bfloat16)
        od = torch.empty_like(qd)
        ld = torch.empty(1, nh, device=dev)
        wsp = zdc.decode_attention_bf16(qd, ka, va, od, avg_ctx, ld)
        t_dec = _time_graph(torch, stream, lambda i: zdc.decode_attention_bf16(qd, ka, va, od, avg_ctx, ld,
                                                                               workspace=wsp), 64)
        # library comparison: torch SDPA (flash / cuDNN backend), causal, same scale
        qs = qa.view(1, S, nh, rr).transpose(1, 2).contiguous()
        kk = ks if nkv == nh else ks.repeat_interleave(nh // nkv, dim=1).contiguous()
        vv = vs if nkv == nh else vs.repeat_interleave(nh // nkv, dim=1).contiguous()
        try:
            t_sdpa = _time_graph(torch, stream, lambda i: F.scaled_dot_product_attention(
                qs, kk, vv, is_causal=True, scale=1.0 / math.sqrt(dh)), 10)
        except Exception as e:  # reported only
            t_sdpa = None
        flop = prefill_layer_flops(d, nh, nkv, rr, 1, S)["a3"]
        attn["r%d" % rr] = {"prefill_attention_us": round(t_pre * 1e3, 2),
                            "prefill_attention_tflops": round(flop / (t_pre / 1e3) / 1e12, 1),
                            "decode_attention_us": round(t_dec * 1e3, 2),
                            "torch_sdpa_prefill_us": round(t_sdpa * 1e3, 2) if t_sdpa else None,
                            "torch_sdpa_tflops": round(flop / (t_sdpa / 1e3) / 1e12, 1) if t_sdpa else None}
        del qa, ka, va, pa, qs, kk, vv, ks, vs
    # torch.matmul at the c2 projection shapes (report only)
    mm = {}
    for name, (M, N, K) in {"a1_qkv_r%d" % r: (S, nh * r + 2 * nkv * r, d), "a5_out_r%d" % r: (S, d, nh * r)}.items():
        A = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
        Bm = torch.randn(K, N, device=dev, generator=g).to(torch.bfloat16)
        Wt = Bm.t().contiguous()
        Cm = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        t_mm = _time_graph(torch, stream, lambda i: torch.matmul(A, Bm, out=Cm), 10)
        t_z = _time_graph(torch, stream, lambda i: zdc.gemm_bf16(A, Wt, Cm), 10)
        fl = 2.0 * M * N * K
        mm[name] = {"shape_MNK": [M, N, K], "torch_matmul_us": round(t_mm * 1e3, 2),
                    "torch_matmul_tflops": round(fl / (t_mm / 1e3) / 1e12, 1),
                    "zdc_gemm_us": round(t_z * 1e3, 2), "zdc_gemm_tflops": round(fl / (t_z / 1e3) / 1e12, 1)}
        del A, Bm, Wt, Cm
    torch.cuda.empty_cache()
    ar, ad = attn["r%d" % r], attn["r%d" % dh]
    return {
        "what": "same kernels at r = d_h = %d with R = I (uncompressed model), c2 step timed as the headline" % dh,
        "prefill_ms": round(pre_ms, 3), "decode_ms": round(dec_ms, 3),
        "prefill_tok_s": S / (pre_ms / 1e3), "decode_tok_s": T / (dec_ms / 1e3),
        "step_tok_s": (S + T) / ((pre_ms + dec_ms) / 1e3),
        "speedup_compressed_vs_uncompressed": {"prefill": round(pre_ms / pre_ms_r, 3), "decode": round(dec_ms / dec_ms_r, 3),
                                               "step": round((pre_ms + dec_ms) / (pre_ms_r + dec_ms_r), 3)},
        "decode_bytes_per_layer_step": {"r%d" % r: dec_bytes_r, "r%d" % dh: dec_bytes_u,
                                        "ratio": round(dec_bytes_r / dec_bytes_u, 4)},
        "sp_exchange_bytes_ratio": r / dh,
        "attention_time_saved": {"prefill": round(1.0 - ar["prefill_attention_us"] / ad["prefill_attention_us"], 4),
                                 "decode": round(1.0 - ar["decode_attention_us"] / ad["decode_attention_us"], 4),
                                 "paper": "21-28% -> 62-64% of attention time saved at p 0.3 -> 0.7 (PAPER.md:1971, A100)"},
        "attention_kernels": attn, "library_comparison_matmul": mm,
        "note": "library numbers are reported only; the product path never calls torch SDPA or matmul",
    }


# ------------------------------------------------------------------------------------ NEXT-4 FP8 cache
def _decode_step_us(zdc, torch, dev, stream, dims, plan, B, S, T=32):
    """Per-layer decode layer-step time (us) of `dims.n_layers` layers called one by one (same x),
    each step one CUDA graph, after a prefill of S tokens; timing-only weights."""
    L, d, nh, nkv, dh = dims.n_layers, dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
    ctx = zdc.Context(dims, plan, B, S + T + 4)
    g = torch.Generator(device=dev).manual_seed(77)
    for l in range(L):
        ctx.load_folded_device(l, *_timing_weights(torch, dev, g, d, nh, nkv, dh))
    x = torch.randn(B, S, d, device=dev, generator=g).to(torch.bfloat16)
    y = torch.empty_like(x)
    for l in range(L):
        ctx.prefill(x, y, l, l + 1)
    xb = torch.randn(B, d, device=dev, generator=g).to(torch.bfloat16)
    yb = torch.empty_like(xb)
    for l in range(L):
        ctx.decode(xb, yb, l, l + 1)
    gs = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gs, stream=stream):
        for l in range(L):
            ctx.decode(xb, yb, l, l + 1)
    gs.replay()
    torch.cuda.synchronize()
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(T - 2):
        gs.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ctx.close()
    return e0.elapsed_time(e1) * 1e3 / ((T - 2) * L)


def fp8_bench(zdc, torch, dev, stream):
    """NEXT-4 (GEAR-ZDC, P:1642 DEL): decode layer-step with the FP8 E4M3 compressed cache (r codes +
    f32 scale + 12 pad bytes per row) against the bf16 cache, at the c2 shape (B = 1, ctx 2048+) and
    at a c3-like uniform shape (B = 32, 40 heads, r = 96, ctx 1024+).  The FP8 cache runs the
    separate-kernel decode path (split-K FP8 attention); bf16 is shown on that path and, at B = 1,
    on the fused layer-step kernel the headline uses."""
    import zdc_synth as Z
    out = {}
    shapes = {"c2_B1": (Z.Dims(4, 4096, 32, 32, 128), 64, 1, 2048), "c3_uniform_B32": (Z.Dims(4, 5120, 40, 40, 128), 96, 32, 1024)}
    peaks = load_peaks()
    for name, (dims, r, B, S) in shapes.items():
        rec = {"rank": r, "batch": B, "prompt": S}
        wbytes = sum(decode_layer_bytes(dims.d_model, dims.n_heads, dims.n_kv_heads, r, B, 0).values())
        ctx_avg = S + 16
        for label, fp8, mode in (("bf16_fused", 0, "auto"), ("bf16_separate", 0, "separate"), ("fp8", 1, "separate")):
            if label == "bf16_fused" and B > 8:
                continue
            plan = Z.plan_uniform(dims.n_layers, r)
            plan.kv_fp8 = fp8
            old = zdc.decode_mode(mode)
            try:
                us = _decode_step_us(zdc, torch, dev, stream, dims, plan, B, S)
            finally:
                zdc.decode_mode(old)
            row = (r + 16) if fp8 else 2 * r
            kv = B * dims.n_kv_heads * ctx_avg * 2 * row
            rec[label] = {"us_per_layer_step": round(us, 2), "kv_bytes": kv, "bytes_per_layer_step": wbytes + kv,
                          "achieved_gbs": round((wbytes + kv) / (us / 1e6) / 1e9, 1),
                          "frac": round((wbytes + kv) / (us / 1e6) / 1e9 / peaks["hbm"], 4)}
        out[name] = rec
    # eviction (H2O-ZDC, reading c26): a c3 group (4 layers, g = 0.5, r^i = 96) with r^u = 32 (token
    # split) vs r^u = 0 (unimportant tokens evicted), per-key-mean importance (decode tokens ~g important)
    dims = Z.Dims(4, 5120, 40, 40, 128)
    rec = {"batch": 32, "prompt": 1024, "g_bp": 5000, "importance": "mean"}
    for label, ru in (("split_r32", 32), ("evict_r0", 0)):
        plan = Z.plan_split(4, 96, ru, [[0, 1, 2, 3]], [5000], importance_mode=1)
        old = zdc.decode_mode("auto")
        try:
            rec[label] = {"us_per_layer_step": round(_decode_step_us(zdc, torch, dev, stream, dims, plan, 32, 1024), 2)}
        finally:
            zdc.decode_mode(old)
    out["c3_group_eviction"] = rec
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------------------------ NEXT-3 fold
def fold_bench(zdc, torch, dev, stream, n_calib=32768, k=2048, iters=5):
    """NEXT-3: the offline fold of one c2-shaped layer on the GPU in fp64
    (calibration capture -> K-means of every Q^h / K^g / V^g block -> Gram + Jacobi -> fold), with
    n_calib calibration rows consolidated into k clusters by `iters` Lloyd rounds; plus the plain
    (no K-means) GPU fold and the host TSQR + Jacobi fold at 4096 rows.  Timing-only random inputs."""
    import zdc_synth as Z
    dims = Z.dims_of(2, n_layers=1)
    d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
    g = torch.Generator(device=dev).manual_seed(31)
    f64 = torch.float64
    w = [torch.randn(d, nh * dh, device=dev, generator=g, dtype=f64) / math.sqrt(d),
         torch.randn(d, nkv * dh, device=dev, generator=g, dtype=f64) / math.sqrt(d),
         torch.randn(d, nkv * dh, device=dev, generator=g, dtype=f64) / math.sqrt(d),
         torch.randn(nh * dh, d, device=dev, generator=g, dtype=f64) / math.sqrt(d)]
    xc = torch.randn(n_calib, d, device=dev, generator=g, dtype=f64)
    out = {"layer": "c2 (d 4096, 32 heads, d_h 128)"}
    for name, rows, kk, it in (("kmeans", n_calib, k, iters), ("plain", 4096, 0, 0)):
        zdc.fold_weights_gpu(dims, *w, xc[:rows], k_clusters=kk, kmeans_iters=it, return_device=True)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        zdc.fold_weights_gpu(dims, *w, xc[:rows], k_clusters=kk, kmeans_iters=it, return_device=True)
        torch.cuda.synchronize()
        out["gpu_%s" % name] = {"calib_rows": rows, "clusters": kk, "lloyd_rounds": it,
                                "seconds_per_layer": round(time.perf_counter() - t0, 3)}
    wh = [t.cpu().numpy() for t in w]
    xh = xc[:4096].cpu().numpy()
    t0 = time.perf_counter()
    zdc.fold_weights(dims, *wh, xh)
    out["host_plain"] = {"calib_rows": 4096, "seconds_per_layer": round(time.perf_counter() - t0, 3),
                         "threads": os.cpu_count()}
    out["gpu_kmeans"]["model_minutes_extrapolated"] = round(out["gpu_kmeans"]["seconds_per_layer"] * 32 / 60, 2)
    out["paper"] = "rotation-matrix computation 7.8-282 min per model (P:1897-1901; A100 cluster, up to 1M clusters)"
    del w, xc
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------------------------ zdc arm
def run_zdc(args):
    import torch
    import torch.distributed as dist
    import paper_2408_04107_b200 as zdc
    import zdc_synth as Z

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    zdc.decode_mode(args.decode_mode)

    L, S, T, r = args.layers, args.prompt, args.decode_steps, args.rank
    base = Z.dims_of(2)
    dims = Z.Dims(L, base.d_model, base.n_heads, base.n_kv_heads, base.d_head)
    d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
    B = 1
    plan = Z.plan_uniform(L, r)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = zdc.Context(dims, plan, B, S + T)

    # Timing-only weights (SURVEY.md §8(d) "ideal fold" shortcut): folded weights W^R = W R with
    # R = the generator's own basis, i.e. column j of W_Q^{R,h} is a * s_j * (orthonormal-like
    # column); generated on the device with a seeded generator, same shapes/bytes as a real fold.
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    s = torch.tensor([10.0 ** (-2.0 * j / (dh - 1)) for j in range(dh)], device=dev)
    a = (4.0 * dh / float((s ** 4).sum())) ** 0.25
    bta = math.sqrt(dh / float((s ** 2).sum()))
    gam = math.sqrt(dh / (nh * float((s ** 2).sum())))
    for l in range(L):
        wq = (torch.randn(d, nh, dh, device=dev, generator=g) * (a * s / math.sqrt(d))).reshape(d, nh * dh)
        wk = (torch.randn(d, nkv, dh, device=dev, generator=g) * (a * s / math.sqrt(d))).reshape(d, nkv * dh)
        wv = (torch.randn(d, nkv, dh, device=dev, generator=g) * (bta * s / math.sqrt(d))).reshape(d, nkv * dh)
        wo = (torch.randn(nh, dh, d, device=dev, generator=g) * (gam * s[:, None] / math.sqrt(d))).reshape(nh * dh, d)
        ctx.load_folded_device(l, *[t.to(torch.bfloat16).contiguous() for t in (wq, wk, wv, wo)])
        del wq, wk, wv, wo
    torch.cuda.synchronize()

    x_prompt = torch.randn(B, S, d, device=dev, generator=g).to(torch.bfloat16)
    x_dec = torch.randn(T, B, d, device=dev, generator=g).to(torch.bfloat16)
    y = torch.empty(B, S, d, device=dev, dtype=torch.bfloat16)
    x_buf = torch.empty(B, d, device=dev, dtype=torch.bfloat16)
    y_dec = torch.empty(B, d, device=dev, dtype=torch.bfloat16)
    y_all = torch.empty(T, B, d, device=dev, dtype=torch.bfloat16)

    def eager_step():
        ctx.reset()
        for l in range(L):
            ctx.prefill(x_prompt, y, l, l + 1)
        for t in range(T):
            x_buf.copy_(x_dec[t])
            for l in range(L):
                ctx.decode(x_buf, y_dec, l, l + 1)
            y_all[t].copy_(y_dec)

    # warm-up eagerly (kernel attributes, decode graphs of the library), then capture the step
    log("weights loaded; eager warm-up step")
    eager_step()
    torch.cuda.synchronize()
    log("eager step done")
    if args.profile_only:
        eager_step()
        torch.cuda.synchronize()
        return

    launches = {"prefill": 0, "decode": 0}
    ctx.reset()
    g_pre = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_pre, stream=stream):
        for l in range(L):
            ctx.prefill(x_prompt, y, l, l + 1)
            launches["prefill"] += zdc.last_launch_count()
    g_dec = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_dec, stream=stream):
        if args.decode_calls == "chain":
            ctx.decode(x_buf, y_dec, 0, L)  # the model's dataflow: y of layer l feeds layer l+1
            launches["decode"] += zdc.last_launch_count()
        else:
            for l in range(L):
                ctx.decode(x_buf, y_dec, l, l + 1)
                launches["decode"] += zdc.last_launch_count()
    torch.cuda.synchronize()
    log("graphs captured")
    kernels_per_step = launches["prefill"] + T * launches["decode"]

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

    def graph_step(times=None):
        ctx.reset()  # lengths only (the prefill graph sets them to S); host bookkeeping
        if times is not None:
            ev[0].record(stream)
        g_pre.replay()
        if times is not None:
            ev[1].record(stream)
        for t in range(T):
            x_buf.copy_(x_dec[t])
            g_dec.replay()
            y_all[t].copy_(y_dec)
        if times is not None:
            ev[2].record(stream)

    for _ in range(args.warmup):
        graph_step()
    torch.cuda.synchronize()
    log("graph warm-up done")
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local, period_ms=20)
    clk.start()
    clk.wait_first()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    pre_ms, dec_ms = [], []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_start.record(stream)
    for _ in range(args.steps):
        graph_step(times=True)
        # per-phase split from the last step's events (sync-free: read after the loop)
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    pre_ms.append(ev[0].elapsed_time(ev[1]))
    dec_ms.append(ev[1].elapsed_time(ev[2]))
    clocks = clk.stop()
    if world > 1:
        tt = torch.tensor([total_ms, pre_ms[-1], dec_ms[-1]], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, pre_ms[-1], dec_ms[-1] = [float(v) for v in tt]
    ms_per_step = total_ms / args.steps
    tok_per_step = B * (S + T)
    value = world * tok_per_step * args.steps / (total_ms / 1e3)

    # ---- per-kernel roofline: every kernel of the step timed ALONE at the bench shapes (a CUDA
    # graph of back-to-back launches through the kernel-level C-ABI entries, CUDA events on this
    # stream; weights / caches rotate through 8 copies so every launch streams from HBM).  Inside
    # the step the decode kernels overlap through PDL, so per-kernel times are only defined here.
    log("isolated kernel timing")
    kernels, shares = isolated_kernels(zdc, torch, stream, dev, d, nh, nkv, r, S, T, B, L,
                                       total_ms / args.steps)
    decode_layer_bytes = sum(kernels[k]["work_per_launch"] for k in
                             ("a1_decode_gemv", "a3_decode_attention", "a5_decode_gemv"))
    fused = launches["decode"] in (1, L)  # fused layer-step kernel(s) (decode_fused.cuh)
    if fused:
        # the decode step is L back-to-back launches of the fused layer kernel (a1+a2+a3+a5): its
        # average launch duration is measured LIVE, over the decode region of the timed step
        # (CUDA events on the launch stream; includes the two tiny x/y copies per step).  The
        # separate decode kernels are then not in the step: kept under "unfused_decode_kernels".
        unf = {k: kernels.pop(k) for k in ("a1_decode_gemv", "a3_decode_attention", "a5_decode_gemv")}
        for k in unf:
            shares.pop(k)
            unf[k]["est_share_of_step"] = 0.0
        per_launch = L if launches["decode"] == 1 else 1  # layers per fused launch
        n_launch = L * T // per_launch
        avg_s = dec_ms[-1] / 1e3 / n_launch
        ach = decode_layer_bytes * per_launch / avg_s / 1e9
        peaks = load_peaks()
        kernels["decode_layer_fused"] = {
            "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm"], "unit": "GB/s",
            "frac": round(ach / peaks["hbm"], 4), "avg_us": round(avg_s * 1e6, 2), "launches_per_step": n_launch,
            "layers_per_launch": per_launch, "work_per_launch": decode_layer_bytes * per_launch, "traffic": None,
            "timing": "live (timed region)",
            "est_share_of_step": round(dec_ms[-1] / (total_ms / args.steps), 4)}
        shares["decode_layer_fused"] = dec_ms[-1] / (total_ms / args.steps)
        traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(traffic_path):
            t = json.load(open(traffic_path)).get("decode_layer_fused")  # one layer-step, ncu
            kernels["decode_layer_fused"]["traffic"] = t * per_launch if t else None
    dom = max(kernels, key=lambda k: shares[k])
    roof = dict(kernels[dom])
    roof["kernel"] = dom

    # ---- end to end through the public API with host buffers (pinned), copies inside the region
    e2e = None
    if not args.no_e2e:
        hx = torch.empty(B, S, d, dtype=torch.bfloat16, pin_memory=True).copy_(x_prompt.cpu())
        hxd = torch.empty(T, B, d, dtype=torch.bfloat16, pin_memory=True).copy_(x_dec.cpu())
        hy = torch.empty(B, S, d, dtype=torch.bfloat16, pin_memory=True)
        hyd = torch.empty(T, B, d, dtype=torch.bfloat16, pin_memory=True)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            x_prompt.copy_(hx, non_blocking=True)
            x_dec.copy_(hxd, non_blocking=True)
            graph_step()
            hy.copy_(y, non_blocking=True)
            hyd.copy_(y_all, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([e_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt[0])
        bpe = 2
        e2e = {"value": world * tok_per_step * args.steps / (e_ms / 1e3), "unit": "tok/s",
               "h2d_bytes_per_step": (B * S * d + T * B * d) * bpe,
               "d2h_bytes_per_step": (B * S * d + T * B * d) * bpe}

    # ---- SP prefill with the compressed K'/V' all-gather (a6): N > 1 (or --sp at N = 1)
    sp = None
    if (world > 1 or args.sp) and not args.no_sp:
        log("SP prefill (c5) over %d rank(s)" % world)
        sp = {}
        for flow in ("allgather", "ulysses"):   # compressed K'/V' all-gather; the paper's Ulysses a2a
            try:
                sp[flow] = sp_bench(args, zdc, torch, dist, rank, world, dev, stream, dataflow=flow)
            except Exception as e:  # reported, never hides the main line
                sp[flow] = {"error": "%s: %s" % (type(e).__name__, e)}
    elif world == 1:
        sp = {"note": "the K'/V' exchange needs N > 1: bench.py --gpus N under torchrun (or --sp for P = 1)"}

    # ---- per-layer measurements of the other configs (c3 token split, c4 GQA KV-bound decode)
    other = None
    if world == 1 and args.configs:
        other = {}
        for name in [c for c in args.configs.split(",") if c]:
            log("config %s layers" % name)
            modes = (0, 1) if name == "c3" else (0,)
            for mode in modes:   # c3: both importance modes (reading c10)
                key = name if mode == 0 else name + "_mean"
                try:
                    other[key] = config_bench(args, zdc, torch, dev, stream, int(name.lstrip("c")),
                                              importance_mode=mode)
                except Exception as e:  # reported, never hides the main line
                    other[key] = {"error": "%s: %s" % (type(e).__name__, e)}

    # ---- uncompressed r = d_h baseline + library comparison (report only), N = 1
    unc = None
    if world == 1 and not args.no_uncompressed:
        log("uncompressed r = d_h baseline")
        try:
            unc = uncompressed_bench(args, zdc, torch, dev, stream, pre_ms[-1], dec_ms[-1], decode_layer_bytes)
        except Exception as e:  # reported, never hides the main line
            unc = {"error": "%s: %s" % (type(e).__name__, e)}

    # ---- NEXT-3: the offline fold on the GPU at calibration scale (N = 1)
    fold = None
    if world == 1 and not args.no_fold:
        log("offline fold on the GPU (NEXT-3)")
        try:
            fold = fold_bench(zdc, torch, dev, stream)
        except Exception as e:  # reported, never hides the main line
            fold = {"error": "%s: %s" % (type(e).__name__, e)}

    # ---- NEXT-4: FP8 compressed cache decode (N = 1)
    fp8 = None
    if world == 1 and not args.no_fp8:
        log("FP8 cache decode (NEXT-4)")
        try:
            fp8 = fp8_bench(zdc, torch, dev, stream)
        except Exception as e:  # reported, never hides the main line
            fp8 = {"error": "%s: %s" % (type(e).__name__, e)}

    # ---- CPU baseline (oracle as it stands), rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tp, td, cores = oracle_sample(n_decode=16, prompt=S)
        v, _ = oracle_step_tok_s(tp, td, L, S, T)
        cpu = {"value": v, "unit": "tok/s", "cores": cores["threads"], "cores_detail": cores, "kind": "oracle",
               "sample": "1 c2 layer fp64 prefill S=%d (%.2f s) + 16 decode steps (%.3f s/step), extrapolated to "
                         "%d layers x (prefill + %d decode steps)" % (S, tp, td, L, T)}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": CONFIG_NAME, "layers": L, "d_model": d, "n_heads": nh, "n_kv_heads": nkv,
                       "d_head": dh, "rank": r, "batch": B, "prompt": S, "decode_steps": T,
                       "tokens_per_step_per_gpu": tok_per_step, "parallelism": "replicas%d" % world,
                       "l2": "inputs larger than L2 (2.1 GB folded weights per step)",
                       "timing": "CUDA graphs of per-layer zdc_prefill / zdc_decode calls",
                       "decode_mode": args.decode_mode},
            "prefill_tok_s": world * B * S / (pre_ms[-1] / 1e3),
            "decode_tok_s": world * B * T / (dec_ms[-1] / 1e3),
            "prefill_ms": pre_ms[-1], "decode_ms": dec_ms[-1],
            "roofline": roof, "kernels": kernels, "peaks_source": load_peaks()["src"],
            "unfused_decode_kernels": unf if fused else None,
            "decode_layer_roofline": {
                "bound": "hbm", "unit": "GB/s", "peak": load_peaks()["hbm"],
                "achieved": round(decode_layer_bytes / (dec_ms[-1] / 1e3 / (L * T)) / 1e9, 1),
                "frac": round(decode_layer_bytes / (dec_ms[-1] / 1e3 / (L * T)) / 1e9 / load_peaks()["hbm"], 4),
                "bytes_per_layer_step": decode_layer_bytes,
                "note": "whole decode layer-step inside the graph-replayed step: algorithmic bytes (packed "
                        "weights + K'/V' at the average context + x/y) / measured time per layer-step"},
            "clocks": clocks, "gpu_launches": kernels_per_step * args.steps,
            "e2e": e2e, "cpu_baseline": cpu, "sp": sp, "other_configs": other, "baseline_uncompressed": unc, "offline_fold": fold, "kv_fp8": fp8,
        }
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------ launcher
def launch_command(argv, n_gpus, port):
    """`python bench.py --gpus N ...` without a torchrun environment: the same command once per GPU
    of this node through torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n_gpus),
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


def needs_launch(args, env) -> bool:
    return args.gpus > 1 and "WORLD_SIZE" not in env


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    args = parse()
    if needs_launch(args, os.environ):
        cmd = launch_command(sys.argv[1:], args.gpus, _free_port())
        log("launching %d ranks: %s" % (args.gpus, " ".join(cmd)))
        sys.exit(subprocess.call(cmd))
    if args.launch_probe:
        import torch
        import torch.distributed as dist
        rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
        total = rank
        if world > 1:
            dist.init_process_group("gloo")
            t = torch.tensor([rank])
            dist.all_reduce(t)
            total = int(t[0])
            dist.destroy_process_group()
        print(json.dumps({"rank": rank, "world": world, "rank_sum": total}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_zdc(args)


if __name__ == "__main__":
    main()
