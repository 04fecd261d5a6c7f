"""One W1-shaped GEMM with the forward's fused epilogue (+b1, fast GELU, bf16 out) for ncu."""
import sys, torch
sys.path.insert(0, ".")
from paper_2505_19342_b200 import kernels
M, N, K = 12608, 3072, 768
a = torch.randn(M, K, device="cuda").to(torch.bfloat16); b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
outh = torch.empty(M, N, device="cuda", dtype=torch.bfloat16); bias = torch.randn(N, device="cuda")
for _ in range(3):
    kernels.gemm(a, b, bias=bias, gelu=2, out_hi=outh)
torch.cuda.synchronize()
