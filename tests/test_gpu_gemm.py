"""NEXT-3 projection GEMM (dmha_linear, tcgen05 kernel gemm_sm100.cu) against a
plain PyTorch reference of the same op: y = x @ w with bf16 inputs, computed
in fp64 on the device from the same bf16 values.

Bound per element: the bf16 round-to-nearest-even of the output (2^-9 |ref|,
taken as 2^-8 for slack) plus the fp32 accumulation error of K products,
K * 2^-24 * (|x| @ |w|).
"""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2302_06218_b200 import dmha  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _lib():
    dmha.init(1, 0, None, 0, "bf16", "contiguous")
    yield
    dmha.finalize()


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (1, 8, 8), (300, 264, 72), (777, 520, 1000),
                                   (4096, 2048, 2048), (1000, 1024, 4096), (33000, 512, 256)])
def test_linear_matches_fp64(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    x = torch.randn((M, K), generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn((K, N), generator=g, device="cuda") / K ** 0.5).to(torch.bfloat16)
    y = dmha.linear(x, w)
    torch.cuda.synchronize()
    ref = x.double() @ w.double()
    mag = x.double().abs() @ w.double().abs()
    err = (y.double() - ref).abs()
    bound = 2.0 ** -8 * ref.abs() + K * 2.0 ** -24 * mag + 1e-30
    assert bool((err <= bound).all()), f"max err {err.max().item():.3e}, worst ratio {(err / bound).max().item():.2f}"


def test_linear_empty_and_errors():
    x = torch.zeros((0, 64), dtype=torch.bfloat16, device="cuda")
    w = torch.zeros((64, 128), dtype=torch.bfloat16, device="cuda")
    y = dmha.linear(x, w)
    assert y.shape == (0, 128)
    with pytest.raises(dmha.DmhaError):  # N not a multiple of 8
        dmha.linear(torch.zeros((4, 64), dtype=torch.bfloat16, device="cuda"),
                    torch.zeros((64, 12), dtype=torch.bfloat16, device="cuda"))


def test_linear_is_deterministic():
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((2048, 1024), generator=g, device="cuda").to(torch.bfloat16)
    w = torch.randn((1024, 768), generator=g, device="cuda").to(torch.bfloat16)
    a = dmha.linear(x, w)
    b = dmha.linear(x, w)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
