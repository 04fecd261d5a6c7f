"""GEMM epilogue cost on the block shapes: plain bf16 out vs the fused epilogues the forward uses
(QKV: bf16; Wo / W2: +bias +fp32 residual -> fp32; W1: +bias +GELU -> bf16), each also with
ASTRA_GEMM_DEBUG (read once per process; run the script once per mode: 0 full, 1 no UMMA)."""
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

mode = os.environ.get("ASTRA_GEMM_DEBUG", "0")
M = 12608
for name, N, K, kind in [("wo", 768, 768, "res"), ("w2", 768, 3072, "res"), ("w1", 3072, 768, "gelu"), ("qkv", 2304, 768, "plain")]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16); b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    outh = torch.empty(M, N, device="cuda", dtype=torch.bfloat16); out = torch.empty(M, N, device="cuda")
    bias = torch.randn(N, device="cuda"); res = torch.randn(M, N, device="cuda")
    r = {"plain": bench(lambda: kernels.gemm(a, b, out_hi=outh)),
         "bias": bench(lambda: kernels.gemm(a, b, bias=bias, out_hi=outh)),
         "f32": bench(lambda: kernels.gemm(a, b, out_f32=out))}
    if kind == "res":
        r["res_f32"] = bench(lambda: kernels.gemm(a, b, residual=res, out_f32=out))
        r["bias_res_f32"] = bench(lambda: kernels.gemm(a, b, bias=bias, residual=res, out_f32=out))
        r["bias_res_inplace"] = bench(lambda: kernels.gemm(a, b, bias=bias, residual=out, out_f32=out))
    if kind == "gelu":
        r["bias_gelu"] = bench(lambda: kernels.gemm(a, b, bias=bias, gelu=2, out_hi=outh))
        r["gelu"] = bench(lambda: kernels.gemm(a, b, gelu=2, out_hi=outh))
    print(f"mode {mode} {name} {M}x{N}x{K}: " + " | ".join(f"{k} {v:.1f}" for k, v in r.items()), flush=True)
