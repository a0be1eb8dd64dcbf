"""Kernel-level numerics (through the C ABI) against plain PyTorch fp32 references of the same op:
the tcgen05 causal attention (a3 prefill), the split-K decode attention (a3 decode) and the decode
projection GEMV (a1 / a5 decode).  Shapes span several tiles, ragged tails and GQA groups."""
import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ref_attention(q, k, v, causal_pos, scale):
    """q [Tq][r] f32, k/v [Tk][r] f32; row i sees keys j <= causal_pos[i]."""
    s = (q @ k.t()) * scale
    j = torch.arange(k.shape[0], device=q.device)[None, :]
    s = s.masked_fill(j > causal_pos[:, None], float("-inf"))
    lse = torch.logsumexp(s, dim=1)
    return torch.softmax(s, dim=1) @ v, lse


def _normwise(a, b):
    return float((a - b).abs().max() / b.abs().max())


@pytest.mark.parametrize("B,S,Nh,Nkv,r", [(1, 128, 2, 2, 16), (2, 300, 4, 2, 64), (1, 257, 8, 1, 32),
                                          (1, 1024, 4, 4, 64), (1, 200, 2, 1, 96), (2, 150, 2, 2, 128)])
def test_prefill_attention_kernel_vs_torch(B, S, Nh, Nkv, r):
    import paper_2408_04107_b200 as zdc
    g = torch.Generator(device="cuda").manual_seed(S + r)
    q = (torch.randn(B, S, Nh * r, device="cuda", generator=g) * 0.3).to(torch.bfloat16)
    k = (torch.randn(B, Nkv, S, r, device="cuda", generator=g) * 0.3).to(torch.bfloat16)
    v = torch.randn(B, Nkv, S, r, device="cuda", generator=g).to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty(B, Nh, S, device="cuda", dtype=torch.float32)
    scale = 1.0 / math.sqrt(128)
    zdc.prefill_attention_bf16(q, k, v, o, lse, scale=scale)
    torch.cuda.synchronize()
    G = Nh // Nkv
    pos = torch.arange(S, device="cuda")
    for b in range(B):
        for h in range(Nh):
            ref, ref_lse = _ref_attention(q[b, :, h * r:(h + 1) * r].float(), k[b, h // G].float(),
                                          v[b, h // G].float(), pos, scale)
            assert _normwise(o[b, :, h * r:(h + 1) * r].float(), ref) <= 1e-2
            assert float((lse[b, h] - ref_lse).abs().max()) <= 2e-2


@pytest.mark.parametrize("B,Nh,Nkv,r,length,cap", [(1, 32, 32, 64, 2049, 2304), (2, 8, 1, 128, 700, 800),
                                                   (3, 4, 2, 48, 1, 16), (1, 64, 8, 64, 8448, 8448)])
def test_decode_attention_kernel_vs_torch(B, Nh, Nkv, r, length, cap):
    import paper_2408_04107_b200 as zdc
    g = torch.Generator(device="cuda").manual_seed(length)
    q = (torch.randn(B, Nh * r, device="cuda", generator=g) * 0.3).to(torch.bfloat16)
    k = (torch.randn(B, Nkv, cap, r, device="cuda", generator=g) * 0.3).to(torch.bfloat16)
    v = torch.randn(B, Nkv, cap, r, device="cuda", generator=g).to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty(B, Nh, device="cuda", dtype=torch.float32)
    scale = 1.0 / math.sqrt(128)
    ws = zdc.decode_attention_bf16(q, k, v, o, length, lse, scale=scale)
    zdc.decode_attention_bf16(q, k, v, o, length, lse, scale=scale, workspace=ws)  # counters reusable
    torch.cuda.synchronize()
    G = Nh // Nkv
    pos = torch.tensor([length - 1], device="cuda")
    for b in range(B):
        for h in range(Nh):
            ref, ref_lse = _ref_attention(q[b:b + 1, h * r:(h + 1) * r].float(), k[b, h // G, :length].float(),
                                          v[b, h // G, :length].float(), pos, scale)
            assert _normwise(o[b:b + 1, h * r:(h + 1) * r].float(), ref) <= 1e-2
            assert abs(float(lse[b, h]) - float(ref_lse[0])) <= 2e-2


@pytest.mark.parametrize("B,N,K", [(1, 6144, 4096), (1, 4096, 2048), (3, 1000, 512), (8, 96, 64), (2, 5120, 8192)])
def test_gemv_kernel_vs_torch(B, N, K):
    import paper_2408_04107_b200 as zdc
    g = torch.Generator(device="cuda").manual_seed(N + K)
    w = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    x = torch.randn(B, K, device="cuda", generator=g).to(torch.bfloat16)
    y = torch.empty(B, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):   # back-to-back launches (programmatic dependent launch)
        zdc.gemv_bf16(w, x, y)
    torch.cuda.synchronize()
    ref = x.float() @ w.float().t()
    err = (y.float() - ref).abs()
    assert bool((err <= ref.abs() * 2.0 ** -8 + 1e-3 * ref.abs().max()).all())
