"""zdc_decode parity vs the fp64 oracle for each decode kernel family (zdc_decode_mode):
the persistent fused layer-step (decode_fused.cuh), the cluster layer-step (decode_cluster.cuh:
one thread-block cluster per KV group, DSMEM exchanges, f32 y accumulation across groups) and
the separate kernels.  By pin P7 T decode steps from an empty cache equal the rows
of a prefill over the same T tokens; decode after a prefill continues the same rows."""
import numpy as np
import pytest

import oracle as O
import zdc_synth as Z
from zdc_synth import Dims, plan_uniform
from zdc_testlib import fold_stack, from_dev, make_context, normwise, to_dev_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2
MODES = ["fused", "cluster", "separate"]


@pytest.fixture
def mode(request):
    import paper_2408_04107_b200 as zdc
    old = zdc.decode_mode(request.param)
    yield request.param
    zdc.decode_mode(old)


def _decode_steps(ctx, x_steps, stream=None):
    ys = []
    s = stream or torch.cuda.current_stream()
    with torch.cuda.stream(s):
        for t in range(x_steps.shape[1]):
            x = to_dev_bf16(x_steps[:, t])
            y = torch.empty_like(x)
            ctx.decode(x, y)
            ys.append(y)
    s.synchronize()
    return np.stack([from_dev(v) for v in ys], axis=1)


@pytest.mark.parametrize("mode", MODES, indirect=True)
@pytest.mark.parametrize("dims,r,B", [
    (Dims(1, 64, 2, 2, 32), 16, 1),      # c1 shape
    (Dims(1, 64, 2, 2, 32), 16, 3),      # ragged batch (NB = 4)
    (Dims(2, 128, 4, 2, 64), 32, 2),     # GQA G = 2, 2-layer chain
    (Dims(1, 256, 8, 1, 128), 64, 5),    # G = 8 (cluster: G r > 256 -> fused fallback)
    (Dims(1, 384, 4, 4, 96), 96, 8),     # r = 96 (three 32-wide chunks), NB = 8
    (Dims(1, 256, 2, 2, 128), 128, 1),   # full rank r = d_h
])
def test_decode_modes_small(mode, dims, r, B):
    plan = plan_uniform(dims.n_layers, r)
    _, folded = fold_stack(dims, 1, n_calib=max(256, 2 * dims.d_head))
    T = 37
    x = Z.prompt(dims, 1, B, T, seed=21)
    ctx = make_context(dims, plan, folded, B, T + 2)
    y = _decode_steps(ctx, x)
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    assert normwise(y, want) <= TOL
    # the cache holds K'/V' of every token (a2) and the device length advanced once per step
    k, v, _, _ = ctx.cache_export(0, B)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    m.prefill(x)
    assert k.shape[1] == T
    assert normwise(k.transpose(0, 2, 1, 3), m.K[0]) <= 1e-2
    assert normwise(v.transpose(0, 2, 1, 3), m.V[0]) <= 1e-2
    ctx.close()


@pytest.mark.parametrize("mode", ["fused", "cluster"], indirect=True)
def test_decode_modes_c2_after_prefill(mode):
    """c2 layer shape (d=4096, 32 heads, r=64): prefill 1000 tokens, then 40 decode steps on a
    side stream (CUDA graphs + PDL); the cluster kernel splits 1000..1039 cached rows over its 4
    CTAs with ragged slots.  Sampled rows against the oracle."""
    dims = Z.dims_of(2, n_layers=1)
    plan = plan_uniform(1, 64)
    _, folded = fold_stack(dims, 2, n_calib=1024)
    S, T = 1000, 40
    x = Z.prompt(dims, 2, 1, S + T, seed=22)
    ctx = make_context(dims, plan, folded, 1, S + T + 4)
    y0 = torch.empty(1, S, dims.d_model, dtype=torch.bfloat16, device="cuda")
    ctx.prefill(to_dev_bf16(x[:, :S]), y0)
    y = _decode_steps(ctx, x[:, S:], stream=torch.cuda.Stream())
    m = O.OracleModel(dims, plan, folded, faithful=True)
    rows = np.array([S, S + 1, S + 17, S + T - 1])
    want = m.prefill_rows(0, x, rows)
    assert normwise(y[:, rows - S], want) <= TOL
    ctx.close()


@pytest.mark.parametrize("mode", ["cluster"], indirect=True)
def test_decode_cluster_graph_layers(mode):
    """Per-layer calls on a side stream (one graph per call shape, PDL between the cluster
    launches, the y accumulator and counters re-zeroed by each launch's last group) and one
    chained call over 8 layers; both equal the oracle."""
    dims = Dims(8, 256, 4, 4, 64)
    plan = plan_uniform(8, 32)
    _, folded = fold_stack(dims, 1, n_calib=256)
    T = 24
    x = Z.prompt(dims, 1, 2, T, seed=23)
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    ctx = make_context(dims, plan, folded, 2, T + 4)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        bufs = [torch.empty(2, 256, device="cuda", dtype=torch.bfloat16) for _ in range(9)]
        ys = []
        for t in range(T):
            bufs[0].copy_(to_dev_bf16(x[:, t]))
            for l in range(8):
                ctx.decode(bufs[l], bufs[l + 1], l, l + 1)
            ys.append(bufs[8].clone())
    s.synchronize()
    assert normwise(np.stack([from_dev(v) for v in ys], 1), want) <= TOL
    ctx.reset()
    with torch.cuda.stream(s):
        xb = torch.empty(2, 256, device="cuda", dtype=torch.bfloat16)
        yb = torch.empty_like(xb)
        ys = []
        for t in range(T):
            xb.copy_(to_dev_bf16(x[:, t]))
            ctx.decode(xb, yb, 0, 8)
            ys.append(yb.clone())
    s.synchronize()
    assert normwise(np.stack([from_dev(v) for v in ys], 1), want) <= TOL
    ctx.close()


@pytest.mark.parametrize("mode", ["auto"], indirect=True)
def test_decode_in_caller_graph_and_cache_sync(mode):
    """zdc_decode captured inside the CALLER's CUDA graph and replayed per step (device-side cache
    lengths make one graph valid at every position): rows equal the oracle's, and after
    zdc_cache_sync the host lengths agree with the device (P7)."""
    dims = Dims(2, 256, 4, 4, 64)
    plan = plan_uniform(2, 32)
    _, folded = fold_stack(dims, 1, n_calib=256)
    T = 12
    x = Z.prompt(dims, 1, 2, T, seed=24)
    ctx = make_context(dims, plan, folded, 2, T + 2)
    s = torch.cuda.Stream()
    xb = torch.empty(2, 256, device="cuda", dtype=torch.bfloat16)
    yb = torch.empty_like(xb)
    ys = []
    with torch.cuda.stream(s):
        xb.copy_(to_dev_bf16(x[:, 0]))
        ctx.decode(xb, yb, 0, 2)  # eager first step (also warms the library)
        ys.append(yb.clone())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ctx.decode(xb, yb, 0, 2)
        for t in range(1, T):
            xb.copy_(to_dev_bf16(x[:, t]))
            g.replay()
            ys.append(yb.clone())
    s.synchronize()
    got = np.stack([from_dev(v) for v in ys], axis=1)
    want = O.OracleModel(dims, plan, folded, faithful=True).prefill(x)
    assert normwise(got, want) <= TOL
    ctx.cache_sync(s)
    assert ctx.cache_length(0) == T and ctx.cache_length(1) == T
    ctx.close()


@pytest.mark.parametrize("mode,dims,B", [("fused", Dims(1, 256, 4, 4, 64), 2), ("cluster", Dims(1, 256, 4, 4, 64), 2),
                                         ("separate", Dims(1, 256, 4, 4, 64), 2),
                                         ("auto", Dims(1, 512, 16, 2, 64), 10)],   # GEMM + TC attention path
                         indirect=["mode"])
def test_decode_graph_replays_past_max_seq_are_flagged(mode, dims, B):
    """Each replay of a caller-captured decode graph uses one cache row.  Replaying past max_seq
    must not write outside the layer's rows: the overflowing steps rewrite the last row, the length
    saturates at max_seq and zdc_cache_sync reports ZDC_ERR_CAPACITY."""
    import paper_2408_04107_b200 as zdc
    r = 64 if dims.n_kv_heads == 2 else 32
    plan = plan_uniform(1, r)
    _, folded = fold_stack(dims, 1, n_calib=256)
    cap = 6
    x = Z.prompt(dims, 1, B, cap + 6, seed=25)
    ctx = make_context(dims, plan, folded, B, cap)
    s = torch.cuda.Stream()
    xb = torch.empty(B, dims.d_model, device="cuda", dtype=torch.bfloat16)
    yb = torch.empty_like(xb)
    with torch.cuda.stream(s):
        xb.copy_(to_dev_bf16(x[:, 0]))
        ctx.decode(xb, yb)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ctx.decode(xb, yb)
        for t in range(1, cap + 6):
            xb.copy_(to_dev_bf16(x[:, t]))
            g.replay()
    s.synchronize()
    with pytest.raises(zdc.ZdcError) as e:
        ctx.cache_sync(s)
    assert e.value.status == -5
    assert ctx.cache_length(0) == cap
    # rows 0 .. cap-2 still hold tokens 0 .. cap-2 of every (sequence, KV head): nothing spilled
    # into a neighbouring block
    k, v, _, _ = ctx.cache_export(0, B)
    m = O.OracleModel(dims, plan, folded, faithful=True)
    m.prefill(x[:, :cap - 1])
    assert normwise(k[:, :cap - 1].transpose(0, 2, 1, 3), m.K[0]) <= 1e-2
    assert normwise(v[:, :cap - 1].transpose(0, 2, 1, 3), m.V[0]) <= 1e-2
    ctx.reset(s)
    ctx.cache_sync(s)
    ctx.close()
