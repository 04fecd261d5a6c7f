"""Microbenchmark of astra_gemm vs torch.matmul (cuBLAS) on the block's GEMM shapes."""
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

shapes = [(12608, 2304, 768), (12608, 768, 768), (12608, 3072, 768), (12608, 768, 3072), (12544, 1024, 768), (3200, 768, 768)]
for M, N, K in shapes:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16); b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    al = torch.randn(M, K, device="cuda").to(torch.bfloat16); bl = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda"); outh = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2 * M * N * K
    t1 = bench(lambda: kernels.gemm(a, b, out_hi=outh))
    cl = {}
    for bn in ("128", "192", "256"):
        os.environ["ASTRA_GEMM_BN"] = bn
        cl[bn] = bench(lambda: kernels.gemm(a, b, out_hi=outh))
    del os.environ["ASTRA_GEMM_BN"]
    print("   " + " | ".join(f"BN{k} {v*1e6:.1f}us {fl/v/1e12:.0f} TF/s" for k, v in cl.items()), flush=True)
    t3 = bench(lambda: kernels.gemm(a, b, a_lo=al, b_lo=bl, out_f32=out))
    tc = bench(lambda: torch.matmul(a, b.T))
    bias = torch.randn(N, device="cuda")
    tg = bench(lambda: kernels.gemm(a, b, bias=bias, gelu=2, out_hi=outh))
    res = torch.randn(M, N, device="cuda")
    tr = bench(lambda: kernels.gemm(a, b, bias=bias, residual=res, out_f32=out))
    # the same fused outputs from cuBLAS + torch elementwise ops (what an unfused path launches)
    tcg = bench(lambda: torch.nn.functional.gelu(torch.addmm(bias.to(torch.bfloat16), a, b.T)))
    tcr = bench(lambda: torch.add(torch.matmul(a, b.T).float(), res).add_(bias))
    print(f"   +bias+gelu->bf16 {tg*1e6:.1f}us (cublas+torch {tcg*1e6:.1f}us) | +bias+residual->f32 {tr*1e6:.1f}us (cublas+torch {tcr*1e6:.1f}us)", flush=True)
    print(f"{M}x{N}x{K}: bf16 {t1*1e6:.1f}us {fl/t1/1e12:.0f} TF/s | bf16x3 {t3*1e6:.1f}us {3*fl/t3/1e12:.0f} TF/s(eff x3) | cublas {tc*1e6:.1f}us {fl/tc/1e12:.0f} TF/s", flush=True)
