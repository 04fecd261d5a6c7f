"""GEMM bottleneck isolation: per shape, time with UMMAs skipped / epilogue skipped
(ASTRA_GEMM_DEBUG, read once per process: run once per mode)."""
import os, sys, torch
sys.path.insert(0, ".")
from paper_2505_19342_b200 import kernels

def bench(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3

mode = os.environ.get("ASTRA_GEMM_DEBUG", "0")
for M, N, K in [(12608, 2304, 768), (12608, 768, 768), (12608, 3072, 768), (12608, 768, 3072)]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16); b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    outh = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t = bench(lambda: kernels.gemm(a, b, out_hi=outh))
    print(f"mode {mode} {M}x{N}x{K}: {t*1e6:.1f} us  {2*M*N*K/t/1e12:.0f} TF/s", flush=True)
