"""GPU: the tcgen05 stream-K skinny GEMM (a4/a7-a10's contraction, split-bf16
activation operand, R28) against a plain PyTorch fp32 matmul of the
bf16 weights and the fp32 activations."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,K,R", [(128, 64, 1), (256, 64, 16), (1000, 4096, 17), (6144, 4096, 32),
                                   (4096, 14336, 5), (300, 192, 3), (2048, 8192, 9)])
def test_gemm_matches_torch(N, K, R):
    from paper_2505_01572_b200.stage import test_gemm
    g = torch.Generator(device="cuda").manual_seed(N * 7 + K + R)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    X = torch.randn(32, K, device="cuda", generator=g)
    out = test_gemm(W, X, R)
    ref = (X[:R].double() @ W.double().T).float()
    err = (out - ref).abs().max().item()
    # split operand: ~2^-16 relative per element -> far below a bf16 operand's 2^-8
    assert err <= 2e-5 * max(1.0, ref.abs().max().item()) + 1e-5, err


def test_gemm_row_invariance():
    """Row r's result does not depend on R (16- vs 32-row buckets): bit-exact."""
    from paper_2505_01572_b200.stage import test_gemm
    g = torch.Generator(device="cuda").manual_seed(1)
    W = (torch.randn(4096, 4096, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    X = torch.randn(32, 4096, device="cuda", generator=g)
    a = test_gemm(W, X, 1)
    b = test_gemm(W, X, 17)
    c = test_gemm(W, X, 32)
    assert torch.equal(a[0], b[0]) and torch.equal(b, c[:17])
