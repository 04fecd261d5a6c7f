"""tcgen05 GEMM parity against a plain PyTorch fp32/fp64 reference of the same op."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(a, b, bias=None, residual=None, gelu=False):
    v = (a.double() @ b.double().T).float()
    if bias is not None:
        v = v + bias
    if gelu:
        v = v * (0.5 * (1.0 + torch.erf(v * 0.7071067811865476)))
    if residual is not None:
        v = residual + v
    return v


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (300, 384, 768), (12608, 2304, 768),
                                   (3200, 768, 3072), (64, 1000, 768), (77, 136, 24)])
def test_gemm_bf16(cuda, M, N, K):
    from paper_2505_19342_b200 import kernels
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    b = torch.randn(N, K, device=cuda, generator=g).to(torch.bfloat16)
    out = torch.empty(M, N, device=cuda)
    kernels.gemm(a, b, out_f32=out)
    ref = _ref(a.float(), b.float())
    err = (out - ref).abs().max().item()
    assert err <= 1e-4 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("M,N,K", [(300, 384, 768), (3200, 3072, 768), (256, 768, 3072)])
def test_gemm_split3_fp32_class(cuda, M, N, K):
    from paper_2505_19342_b200 import kernels
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(M, K, device=cuda, generator=g)
    b = torch.randn(N, K, device=cuda, generator=g) * 0.02
    ah, al = kernels.split_bf16(a)
    bh, bl = kernels.split_bf16(b)
    bias = torch.randn(N, device=cuda, generator=g) * 0.1
    res = torch.randn(M, N, device=cuda, generator=g)
    out = torch.empty(M, N, device=cuda)
    hi = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    lo = torch.empty_like(hi)
    kernels.gemm(ah, bh, a_lo=al, b_lo=bl, bias=bias, residual=res, gelu=True, out_f32=out,
                 out_hi=hi, out_lo=lo)
    ref = _ref(a, b, bias, res, gelu=True)
    scale = (a.double().abs() @ b.double().abs().T).float()
    rel = ((out - ref).abs() / (scale + 1e-30)).max().item()
    assert rel < 2e-5, rel
    # hi/lo outputs reproduce the fp32 value to 2^-16
    assert ((hi.float() + lo.float()) - out).abs().max().item() <= 2 ** -15 * out.abs().max().item()


@pytest.mark.parametrize("cluster", ["1", "2", "4"])
@pytest.mark.parametrize("M,N,K", [(12608, 768, 768), (1000, 3072, 768), (300, 900, 256)])
def test_gemm_cluster_shapes(cuda, monkeypatch, cluster, M, N, K):
    """Every CTA-cluster shape of the persistent GEMM (single CTA, CTA pair, 2x2 with A
    multicast) on ragged shapes, with the fused bias + residual epilogue."""
    from paper_2505_19342_b200 import kernels
    monkeypatch.setenv("ASTRA_GEMM_CLUSTER", cluster)
    g = torch.Generator(device="cuda").manual_seed(2)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    b = torch.randn(N, K, device=cuda, generator=g).to(torch.bfloat16)
    bias = torch.randn(N, device=cuda, generator=g)
    res = torch.randn(M, N, device=cuda, generator=g)
    out = torch.empty(M, N, device=cuda)
    kernels.gemm(a, b, bias=bias, residual=res, out_f32=out)
    ref = _ref(a.float(), b.float(), bias=bias, residual=res)
    err = (out - ref).abs().max().item()
    assert err <= 1e-4 * max(1.0, ref.abs().max().item()), err
