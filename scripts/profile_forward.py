"""One eager ViT-B/16 Astra forward (B=64, N given) for ncu / launch-list capture.

Codebooks: 8 Lloyd iterations (setup, outside the profiler range); the kernel sequence is
the same as bench.py's.  Only the --iters forwards run between cudaProfilerStart/Stop, so
pass `--profile-from-start off` to ncu.  Usage: python scripts/profile_forward.py [--n 1] [--fast|--parity]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_19342_b200 import cluster, data, model, vq  # noqa: E402
from paper_2505_19342_b200.runtime import AstraRuntime, LoopbackExchange  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--parity", action="store_true")
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--rank-of", type=int, default=0,
                help="profile ONE rank (the last) of an N-way split, loopback exchange")
args = ap.parse_args()

cfg = model.ModelConfig(layers=12, hidden=768, heads=12, vocab_or_classes=1000, max_tokens=197,
                        causal=False, codebook_size=1024, groups=1)
params = model.init_params(cfg, seed=0)
xs = data.make_classify_batch(768, 196, args.batch, seed=1)
from paper_2505_19342_b200 import codebooks  # noqa: E402
codebooks.fit_codebooks(params, data.make_classify_batch(768, 196, 8, seed=0), iterations=8)
n = args.rank_of or args.n
plan = cluster.partition_tokens(196, n)
comm = LoopbackExchange(n - 1, n) if args.rank_of > 1 else None
rt = AstraRuntime(params, plan, batch=args.batch, precision="parity" if args.parity else "fast",
                  comm=comm)
rt.stage_input(xs)
torch.cuda.synchronize()
rt.forward()                       # warm-up (module load, first-touch)
torch.cuda.synchronize()
# only the timed forwards are inside the profiler range: run ncu with --profile-from-start off
torch.cuda.cudart().cudaProfilerStart()
for _ in range(args.iters):
    rt.forward()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("logits", rt.logits[:2, :4].cpu().numpy())
