"""The algorithmic work bench.py divides by ("Algorithmic counts" and the
per-kernel budget table): pinned to the figures §8(d) derives by hand for the configs."""
import os

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c2_prefill_flops():
    f = bench.prefill_layer_flops(4096, 32, 32, 64, 1, 2048)
    assert f["a1"] == 103079215104.0        # 103.1 GFLOP: M=2048 N=6144 K=4096
    assert f["a5"] == 34359738368.0         # 34.4 GFLOP: M=2048 N=4096 K=2048
    assert f["a3"] == 17188257792.0         # 17.2 GFLOP: 4 r N_h S(S+1)/2
    # whole c2 prefill (32 layers): 4.95e12 FLOP, projections 66 % / attention 11 % / output 22 %
    tot = 32 * sum(f.values())
    assert abs(tot - 4.95e12) / 4.95e12 < 0.01
    assert round(32 * f["a1"] / tot, 2) == 0.67 and round(32 * f["a3"] / tot, 2) == 0.11


def test_c2_decode_layer_bytes():
    b = bench.decode_layer_bytes(4096, 32, 32, 64, 1, 2176)  # average context of 256 steps after 2048
    assert b["a1"] == 50352128              # W_QKV 50.33 MB (+ x / Q'K'V' rows)
    assert b["a5"] == 16789504              # W_O 16.79 MB (+ O' / y rows)
    assert b["a3"] == 17833984              # K'/V' 8192 B per token x 2176 (+ q / o rows)
    assert sum(b.values()) == 84975616      # 84.98 MB per layer-step


def test_c3_c4_weight_and_kv_bytes():
    # c4 (70B, GQA 8, r = 64): weights 151 MB per layer; K'/V' 256 B per token per KV head
    b4 = bench.decode_layer_bytes(8192, 64, 8, 64, 64, 8320)
    w4 = b4["a1"] - 64 * 8192 * 2 - 64 * 5120 * 2 + b4["a5"] - 64 * 4096 * 2 - 64 * 8192 * 2
    assert w4 == 150994944
    assert abs(b4["a3"] - 1.09e9) / 1.09e9 < 0.01       # KV ~1.09 GB at average context 8320
    # c3 (13B, r^i = 96): weights 157 MB per layer at the important rank
    b3 = bench.decode_layer_bytes(5120, 40, 40, 96, 32, 1)
    w3 = b3["a1"] - 32 * 5120 * 2 - 32 * 11520 * 2 + b3["a5"] - 32 * 3840 * 2 - 32 * 5120 * 2
    assert w3 == 157286400


def test_bench_self_launch_command():
    """`bench.py --gpus N` without torchrun's environment relaunches itself once per GPU."""
    import argparse
    ns = argparse.Namespace(gpus=4)
    assert bench.needs_launch(ns, {})
    assert not bench.needs_launch(ns, {"WORLD_SIZE": "4"})
    assert not bench.needs_launch(argparse.Namespace(gpus=1), {})
    cmd = bench.launch_command(["--gpus", "4", "--steps", "2"], 4, 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert cmd[cmd.index("--nproc-per-node") + 1] == "4"
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_bench_self_launch_gloo_world2():
    """The real launcher path: two ranks rendezvous on 127.0.0.1 and all-reduce over gloo."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-probe"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    import re
    lines = [json.loads(x) for x in re.findall(r"\{[^{}]*\}", out.stdout)]
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert all(x["world"] == 2 and x["rank_sum"] == 1 for x in lines)
