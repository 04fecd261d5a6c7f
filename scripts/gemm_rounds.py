import sys, torch
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
for N in (2304, 3072):
    for M in (11264, 11776, 12288, 12608, 13056, 13568):
        a = torch.randn(M, 768, device="cuda").to(torch.bfloat16); b = torch.randn(N, 768, device="cuda").to(torch.bfloat16)
        o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t = bench(lambda: kernels.gemm(a, b, out_hi=o))
        tiles = ((M + 255) // 256) * ((N + 255) // 256)
        print(f"N={N} M={M}: tiles {tiles} rounds {tiles/74:.2f} -> {t:.1f} us, {t/((tiles+73)//74):.2f} us/round")
