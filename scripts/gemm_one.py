"""Run one astra_gemm configuration a few times (for ncu captures)."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_19342_b200 import kernels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=12608)
ap.add_argument("--N", type=int, default=3072)
ap.add_argument("--K", type=int, default=768)
ap.add_argument("--gelu", action="store_true")
ap.add_argument("--residual", action="store_true")
ap.add_argument("--f32", action="store_true")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
A = torch.randn(a.M, a.K, device="cuda").to(torch.bfloat16)
B = torch.randn(a.N, a.K, device="cuda").to(torch.bfloat16)
bias = torch.randn(a.N, device="cuda")
res = torch.randn(a.M, a.N, device="cuda") if a.residual else None
of = torch.empty(a.M, a.N, device="cuda") if (a.f32 or a.residual) else None
oh = None if of is not None else torch.empty(a.M, a.N, device="cuda", dtype=torch.bfloat16)
for _ in range(a.iters):
    kernels.gemm(A, B, bias=bias, gelu=a.gelu, residual=res, out_f32=of, out_hi=oh)
torch.cuda.synchronize()
