"""Host logic of the sequence-parallel path (a6) with a real world_size-2 gloo process group on
CPU: the positions each rank holds (contiguous / zigzag) partition the sequence, match the golden
layouts, and the compressed-exchange byte count equals the closed form (P12)."""
import json
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2408_04107_b200 as zdc

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "sp_partition_examples.json")


def test_positions_golden():
    spec = json.load(open(GOLDEN))
    for c in spec["zigzag"]:
        assert zdc.sp_positions(c["S"], c["P"], c["rank"], 1).tolist() == c["positions"]
    with pytest.raises(zdc.ZdcError):
        zdc.sp_positions(30, 4, 0, 1)   # 30 not divisible by 2P
    assert zdc.sp_positions(12, 3, 1, 0).tolist() == [4, 5, 6, 7]


def _worker(rank, world, port, S, layout, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos = torch.from_numpy(zdc.sp_positions(S, world, rank, layout).astype(np.int64))
    gathered = [torch.zeros_like(pos) for _ in range(world)]
    dist.all_gather(gathered, pos)
    allpos = torch.cat(gathered).numpy()
    # every position exactly once; each rank's causal work balanced under zigzag
    ok_partition = sorted(allpos.tolist()) == list(range(S))
    work = torch.tensor([float(np.sum(pos.numpy() + 1))])
    works = [torch.zeros(1) for _ in range(world)]
    dist.all_gather(works, work)
    # bytes this rank receives in the all-gather of compressed K'/V' (B=1, N_kv=4, r=16):
    recv = (S - len(pos)) * 1 * 4 * (16 + 16) * 2
    out_q.put((rank, ok_partition, [float(w) for w in works], recv))
    dist.destroy_process_group()


@pytest.mark.parametrize("layout", [0, 1])
def test_gloo_world2_partition_and_bytes(layout):
    world, S = 2, 512
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + layout * 7 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, layout, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, works, recv in res:
        assert ok
        assert recv == O.sp_bytes_received(world, 1, S, 4, 16, 16)
        if layout == 1:   # zigzag balances the causal work exactly for P=2
            assert works[0] == works[1]
        else:
            assert works[0] < works[1]


def test_layer_groups_library_equals_oracle():
    """zdc_layer_groups (host C, NEXT-3 planner) is bit-exact with the oracle's layer_groups
    (reading c22) on random and near-threshold class sets."""
    import numpy as np
    import oracle as O
    import paper_2408_04107_b200 as zdc
    rng = np.random.default_rng(12)
    for trial in range(20):
        L, B, S = 6, 2, int(rng.integers(50, 400))
        base = rng.random((B, S)) < 0.5
        cls = []
        for l in range(L):
            flip = rng.random((B, S)) < float(rng.choice([0.0, 0.02, 0.049, 0.05, 0.051, 0.2]))
            cls.append(base ^ flip)
        cls = np.stack(cls)
        for thr in (9500, 9000, 9950, 0, 10000):
            assert zdc.layer_groups(cls, thr) == O.layer_groups(cls, thr), (trial, thr)
