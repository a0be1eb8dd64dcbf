"""zdc_sp_prefill on ONE GPU with P processes (one zdc_ctx each).  The exchange runs through the
library's test transport (zdc_sp_set_exchange_hook: a gloo all-gather over host memory) instead of
NCCL, which cannot put two ranks on one device; everything else is the production SP path: the a1
epilogue writes each rank's compressed K'/V' slot, attention maps key tiles to (owner, local row)
in the gather buffer, zigzag query chunks.  Checks (P11 layout invariance):
* every rank's y rows are BIT-IDENTICAL to the single-process zdc_prefill rows of its positions
  (same per-element GEMM K order and per-row key-tile order);
* and within 2e-2 of the fp64 oracle."""
import ctypes
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _cudart():
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    raise OSError("libcudart not found")


DIMS = {"mha": (2, 256, 4, 2, 64, 32), "gqa4": (2, 256, 8, 4, 64, 32), "split": (2, 256, 4, 2, 64, 32),
        "split_mean": (2, 256, 4, 2, 64, 32)}


def _plan(shape):
    import zdc_synth as Z
    r = DIMS[shape][5]
    if shape.startswith("split"):   # both layers one group, layer 0 the representative, g = 0.45
        return Z.plan_split(2, r, 16, [[0, 1]], [4500], importance_mode=1 if shape == "split_mean" else 0)
    return Z.plan_uniform(2, r)


def _worker(rank, world, port, layout, S, B, out_q, dataflow="allgather", shape="mha", T=0):
    import torch.distributed as dist
    import oracle as O  # noqa: F401
    import paper_2408_04107_b200 as zdc
    import zdc_synth as Z
    from zdc_testlib import fold_stack, load_lib_fold, to_dev_bf16
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dims = Z.Dims(*DIMS[shape][:5])
    plan = _plan(shape)
    _, folded = fold_stack(dims, 1, n_calib=256)
    ctx = zdc.Context(dims, plan, B, S + (S if T else 0))
    for l, f in enumerate(folded):
        load_lib_fold(ctx, l, f)
    x = Z.prompt(dims, 1, B, S + T, seed=41)
    pos = zdc.sp_positions(S, world, rank, layout)
    cudart = _cudart()
    cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    cudart.cudaStreamSynchronize.argtypes = [ctypes.c_void_p]

    def exchange(user, gbuf, chunk_bytes, r, P, stream):
        cudart.cudaStreamSynchronize(stream)
        mine = np.empty(chunk_bytes, dtype=np.uint8)
        cudart.cudaMemcpy(mine.ctypes.data, gbuf + r * chunk_bytes, chunk_bytes, 2)   # D2H
        parts = [torch.zeros(chunk_bytes, dtype=torch.uint8) for _ in range(P)]
        dist.all_gather(parts, torch.from_numpy(mine))
        for q in range(P):
            cudart.cudaMemcpy(gbuf + q * chunk_bytes, parts[q].numpy().ctypes.data, chunk_bytes, 1)  # H2D

    def alltoall(user, send, recv, chunk_bytes, r, P, stream):
        cudart.cudaStreamSynchronize(stream)
        mine = np.empty(P * chunk_bytes, dtype=np.uint8)
        cudart.cudaMemcpy(mine.ctypes.data, send, P * chunk_bytes, 2)   # D2H
        out = torch.empty(P * chunk_bytes, dtype=torch.uint8)
        dist.all_to_all_single(out, torch.from_numpy(mine))
        cudart.cudaMemcpy(recv, out.numpy().ctypes.data, P * chunk_bytes, 1)   # H2D

    cb = zdc.EXCHANGE_FN(exchange)
    ctx.set_exchange_hook(cb, rank, world)
    cb2 = zdc.ALLTOALL_FN(alltoall)
    ctx.set_alltoall_hook(cb2, rank, world)
    xl = to_dev_bf16(np.ascontiguousarray(x[:, pos]))
    yl = torch.empty_like(xl)
    stats = ctx.sp_prefill(xl, yl, S_total=S, layout=layout, stats=True, dataflow=dataflow)
    torch.cuda.synchronize()
    extra = None
    if shape.startswith("split"):
        extra = ctx.classes_export(0, B) + (ctx.scores_export(0, B),)
    if T:   # NEXT-2: decode over the sequence-sharded cache (partials merged by LSE across ranks)
        ys = []
        for t in range(T):
            xt = to_dev_bf16(np.ascontiguousarray(x[:, S + t]))
            yt = torch.empty_like(xt)
            ctx.sp_decode(xt, yt)
            ys.append(yt.float().cpu().numpy())
        extra = np.stack(ys, axis=1)
    out_q.put((rank, pos, yl.float().cpu().numpy(), stats, extra))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,layout,dataflow,shape", [
    (2, 0, "allgather", "mha"), (2, 1, "allgather", "mha"), (4, 1, "allgather", "mha"),
    (2, 0, "ulysses", "mha"), (2, 1, "ulysses", "mha"), (4, 1, "ulysses", "gqa4"),
    (2, 1, "allgather", "split"), (4, 1, "allgather", "split_mean"), (2, 0, "allgather", "split_mean"),
    (2, 2, "allgather", "mha"), (4, 2, "allgather", "mha")])   # layout 2: exchange overlapped on a comm stream
def test_sp_prefill_equals_single_gpu_rows(world, layout, dataflow, shape):
    import multiprocessing as pymp
    import oracle as O
    import paper_2408_04107_b200 as zdc
    import zdc_synth as Z
    from zdc_testlib import fold_stack, make_context, normwise, to_dev_bf16
    B = 2
    S = 256 * world * (2 if layout else 1)   # chunks of 128 (zigzag) / 256 (contiguous)
    ctx_mp = pymp.get_context("spawn")
    q = ctx_mp.Queue()
    port = 29600 + world * 10 + layout + (5 if dataflow == "ulysses" else 0) + os.getpid() % 500
    procs = [ctx_mp.Process(target=_worker, args=(r, world, port, layout, S, B, q, dataflow, shape))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single-process reference through zdc_prefill
    dims = Z.Dims(*DIMS[shape][:5])
    r = DIMS[shape][5]
    plan = _plan(shape)
    _, folded = fold_stack(dims, 1, n_calib=256)
    x = Z.prompt(dims, 1, B, S, seed=41)
    ctx = make_context(dims, plan, folded, B, S)
    xd = to_dev_bf16(x)
    y = torch.empty_like(xd)
    ctx.prefill(xd, y, 0, 1)
    y0 = torch.empty_like(xd)
    if shape.startswith("split"):   # the SP run chains layer 0 -> 1: the single run does the same
        ctx.prefill(y, y0, 1, 2)
        y, y0 = y0, y
    else:
        ctx.prefill(y, y0, 1, 2)
        y, y0 = y0, y
    torch.cuda.synchronize()
    y_single = y.float().cpu().numpy()
    if shape.startswith("split"):
        cls_single, tau_single = ctx.classes_export(0, B)
        sc_single = ctx.scores_export(0, B)
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    covered = []
    for rank, pos, yl, stats, extra in res:
        assert np.array_equal(yl, y_single[:, pos]), rank      # bit-identical rows
        if extra is not None:   # NEXT-2: the global top-g selection equals the single-GPU one
            cls_sp, tau_sp, sc_sp = extra
            assert np.array_equal(sc_sp, sc_single), rank
            assert np.array_equal(cls_sp, cls_single) and np.array_equal(tau_sp, tau_single), rank
            for b in range(B):
                c_o, t_o, _ = O.select_important(sc_sp[b], plan.g_bp[0])
                assert c_o.tolist() == cls_sp[b].tolist()
        assert normwise(yl, want[:, pos]) <= 2e-2
        covered += pos.tolist()
        nh, nkv, dh = dims.n_heads, dims.n_kv_heads, dims.d_head
        if dataflow == "allgather":
            # bytes received per rank and layer: (P-1)/P * B * S * N_kv * (r_k + r_v) * 2, two layers
            want_b = O.sp_bytes_received(world, B, S, nkv, r, r)
            want_u = O.sp_bytes_received(world, B, S, nkv, dh, dh)
            if extra is not None:   # + the representative's scores: (P-1) * B * S/P f32, once
                want_b += (world - 1) * B * (S // world) * 4 / 2
                want_u += (world - 1) * B * (S // world) * 4 / 2
        else:
            # both all-to-alls (compressed Q'/K'/V' of this rank's heads, then O' back)
            want_b = O.sp_bytes_received_ulysses(world, B, S, nh, nkv, r, r)
            want_u = O.sp_bytes_received_ulysses(world, B, S, nh, nkv, dh, dh)
        assert stats["bytes_recv"] == 2 * want_b
        # r / d_head = 32 / 64 of the uncompressed bytes
        assert stats["bytes_recv_uncompressed"] == 2 * want_u
    assert sorted(covered) == list(range(S))


def test_sp_prefill_nccl_world1():
    """The NCCL transport itself (libnccl resolved at runtime, ncclCommInitRank from a unique id):
    with one rank the communicator is real but the exchange is empty, and zdc_sp_prefill must
    equal zdc_prefill bit for bit; the stats report zero exchanged bytes."""
    import paper_2408_04107_b200 as zdc
    import zdc_synth as Z
    from zdc_testlib import fold_stack, from_dev, load_lib_fold, to_dev_bf16
    dims = Z.Dims(2, 256, 4, 2, 64)
    plan = Z.plan_uniform(2, 32)
    _, folded = fold_stack(dims, 1, n_calib=256)
    S = 256
    x = to_dev_bf16(Z.prompt(dims, 1, 1, S, seed=43))
    outs = []
    for sp in (None, "allgather", "ulysses"):
        ctx = zdc.Context(dims, plan, 1, S)
        for l, f in enumerate(folded):
            load_lib_fold(ctx, l, f)
        y = torch.empty_like(x)
        if sp:
            ctx.comm_init(zdc.comm_unique_id(), 0, 1)
            st = ctx.sp_prefill(x, y, S, layout=1, stats=True, dataflow=sp)
            assert st["bytes_recv"] == 0 and st["bytes_recv_uncompressed"] == 0
        else:
            ctx.prefill(x, y)
        torch.cuda.synchronize()
        outs.append(from_dev(y))
        ctx.close()
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("world,layout", [(2, 1), (4, 0)])
def test_sp_decode_over_sharded_cache(world, layout):
    """NEXT-2: after an all-gather SP prefill, zdc_sp_decode appends decode token j on rank j mod P
    only and merges the ranks' partial attention by LSE; every rank's y equals the oracle's rows
    (P7) within the north-star tolerance, and all ranks agree."""
    import multiprocessing as pymp
    import oracle as O
    import zdc_synth as Z
    from zdc_testlib import fold_stack, normwise
    B, T = 2, 7
    S = 256 * world * (2 if layout else 1)
    ctx_mp = pymp.get_context("spawn")
    q = ctx_mp.Queue()
    port = 29700 + world * 10 + layout + os.getpid() % 500
    procs = [ctx_mp.Process(target=_worker, args=(r, world, port, layout, S, B, q, "allgather", "mha", T))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dims = Z.Dims(*DIMS["mha"][:5])
    plan = _plan("mha")
    _, folded = fold_stack(dims, 1, n_calib=256)
    x = Z.prompt(dims, 1, B, S + T, seed=41)
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)[:, S:]
    ys = [r[4] for r in res]
    for yd in ys:
        assert normwise(yd, want) <= 2e-2
        assert np.array_equal(yd, ys[0])     # every rank computes the same merged rows
