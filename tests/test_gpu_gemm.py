"""tcgen05 projection GEMM (a1 / a5 engine) vs a plain PyTorch fp32 reference of the same op,
through the C-ABI entry zdc_gemm_bf16.  Shapes span several tiles, ragged M/N tails, both
tile widths (BN = 128 / 256) and the c2 projection shapes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [
    (128, 256, 64), (1, 96, 64), (300, 520, 128), (257, 136, 192), (128, 128, 4096),
    (2048, 6144, 4096),   # c2 QKV projection (a1)
    (2048, 4096, 2048),   # c2 output projection (a5)
    (777, 1000, 320),
])
def test_gemm_vs_torch_fp32(M, N, K):
    import paper_2408_04107_b200 as zdc
    g = torch.Generator(device="cuda").manual_seed(M * 131 + N * 7 + K)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    d = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    zdc.gemm_bf16(a, b, d)
    torch.cuda.synchronize()
    ref = a.float() @ b.float().t()
    err = (d.float() - ref).abs()
    # bf16 output rounding (2^-9 relative) + f32 accumulation-order differences
    tol = ref.abs() * 2.0 ** -8 + 1e-4 * ref.abs().max() + 1e-3
    assert torch.isfinite(d.float()).all()
    assert bool((err <= tol).all()), float((err / (ref.abs() + 1e-3)).max())
    assert zdc.last_launch_count() == 1
