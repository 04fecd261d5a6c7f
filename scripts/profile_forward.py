"""One eager Astra forward of a bench.py workload for ncu / launch-list capture.

Weights, codebooks and inputs come from bench.py's setup (the same kernel sequence as the
bench).  Only the --iters forwards run between cudaProfilerStart/Stop, so pass
`--profile-from-start off` to ncu.

    python scripts/profile_forward.py [--config vitb|vitl|gpt2s|gpt2m] [--groups G]
        [--codebook K] [--n N | --rank-of N] [--parity] [--iters I]
"""
import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2505_19342_b200 import cluster  # noqa: E402
from paper_2505_19342_b200.runtime import AstraRuntime, LoopbackExchange  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="vitb", choices=sorted(bench.WORKLOADS))
ap.add_argument("--groups", type=int, default=0)
ap.add_argument("--codebook", type=int, default=0)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--parity", action="store_true")
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--rank-of", type=int, default=0,
                help="profile ONE rank (the last) of an N-way split, loopback exchange")
args = ap.parse_args()

w = bench._workload(args)
params, xs, _ = bench._setup_params(w)
n = args.rank_of or args.n
plan = cluster.partition_tokens(w.T, n, class_replication=w.kind != "prefill")
comm = LoopbackExchange(n - 1, n) if args.rank_of > 1 else None
rt = AstraRuntime(params, plan, batch=w.B, precision="parity" if args.parity else "fast",
                  comm=comm, mode="generate" if w.kind == "prefill" else "classify")
if w.kind == "prefill":
    rt.set_ids(xs)
else:
    rt.stage_input(xs)
torch.cuda.synchronize()
rt.forward()                       # warm-up (module load, first-touch)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(args.iters):
    rt.forward()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", args)
