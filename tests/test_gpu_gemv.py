"""Decode GEMM (tcgen05 weight-streaming kernel, glmx_gemv_run) against a PyTorch fp32 reference:
y (+)= x @ w.T for n <= 64 token rows, the Llama-3-8B decode shapes (split-K with the
last-arriving-CTA reduction for the narrow ones) and the tiny model's.  bf16 inputs, fp32
accumulation: |err| <= 2e-2 + 1e-2 |ref| on outputs of unit scale."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2511_01633_b200.ops import gemv  # noqa: E402

SHAPES = [(4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096), (512, 1024), (4096, 128256)]


@pytest.mark.parametrize("K,N", SHAPES)
@pytest.mark.parametrize("n", [1, 7, 64])
def test_gemv_matches_fp32(K, N, n):
    g = torch.Generator(device="cpu").manual_seed(K + N + n)
    x = torch.randn((n, K), generator=g).to(torch.bfloat16).cuda()
    w = (torch.randn((N, K), generator=g) / K ** 0.5).to(torch.bfloat16).cuda()
    ref = x.float() @ w.float().T
    y = torch.full((n, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    gemv(x, w, y, mode=0)
    err = (y.float() - ref).abs()
    assert (err <= 2e-2 + 1e-2 * ref.abs()).all(), err.max().item()
    y32 = torch.full((n, N), float("nan"), dtype=torch.float32, device="cuda")
    gemv(x, w, y32, mode=1)
    assert ((y32 - ref).abs() <= 2e-3 + 1e-3 * ref.abs()).all()
    base = torch.randn((n, N), generator=g).cuda()
    y_acc = base.clone()
    gemv(x, w, y_acc, mode=2)
    gemv(x, w, y_acc, mode=2)  # counters reset by the last CTA: a second launch is exact too
    assert ((y_acc - (base + 2 * ref)).abs() <= 4e-3 + 1e-3 * ref.abs()).all()
