"""Tile-choice sweep for the per-rank GEMM shapes at N = 8 (M ~ 1664 rows)."""
import os, sys, torch
sys.path.insert(0, ".")
from paper_2505_19342_b200 import kernels

def bench(fn, iters=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1664
for N, K in [(2304, 768), (768, 768), (3072, 768), (768, 3072)]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16); b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    outh = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    res = {}
    os.environ.pop("ASTRA_GEMM_BN", None); os.environ.pop("ASTRA_GEMM_CLUSTER", None)
    res["default"] = bench(lambda: kernels.gemm(a, b, out_hi=outh))
    for c in ("1", "2"):
        for bn in ("128", "192", "256"):
            os.environ["ASTRA_GEMM_BN"] = bn; os.environ["ASTRA_GEMM_CLUSTER"] = c
            res[f"c{c}bn{bn}"] = bench(lambda: kernels.gemm(a, b, out_hi=outh))
    os.environ.pop("ASTRA_GEMM_BN", None); os.environ.pop("ASTRA_GEMM_CLUSTER", None)
    tc = bench(lambda: torch.matmul(a, b.T))
    print(f"{M}x{N}x{K}: " + " ".join(f"{k} {v:.1f}" for k, v in res.items()) + f" | cublas {tc:.1f} us", flush=True)
