"""Per-rank device time of the Astra forward on ONE B200 for the configs of BASELINE.json:
the rank's own shard of an N-way sequence split, with the packed-code all-gather replaced by
a loopback (runtime.LoopbackExchange) — i.e. every kernel an N-GPU rank runs, minus the NCCL
transfer.  Synthetic inputs, seeded weights, sampled codebooks (timing only).

    python scripts/bench_ranks.py [--config vitb|gpt2s|vitl] [--n 1 2 4 8] [--steps 20]
Prints one JSON line per (config, N).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_19342_b200 import cluster, data, model, vq  # noqa: E402
from paper_2505_19342_b200.runtime import AstraRuntime, LoopbackExchange  # noqa: E402

CONFIGS = {
    # name: (layers, hidden, heads, classes/vocab, tokens, batch, codebook K, groups, causal)
    "vitb": (12, 768, 12, 1000, 196, 64, 1024, 1, False),
    "gpt2s": (12, 768, 12, 50257, 1024, 4, 1024, 1, True),
    "vitl": (24, 1024, 16, 1000, 576, 32, 1024, 1, False),
    "vitl_g16": (24, 1024, 16, 1000, 576, 32, 1024, 16, False),
    "vitl_g32": (24, 1024, 16, 1000, 576, 32, 1024, 32, False),
    "gpt2m": (24, 1024, 16, 50257, 4096, 2, 1024, 1, True),   # BASELINE config #5
}


def run(name, n, steps, warmup, rank=None):
    L, D, H, C, T, B, K, G, causal = CONFIGS[name]
    cfg = model.ModelConfig(layers=L, hidden=D, heads=H, vocab_or_classes=C,
                            max_tokens=T + (0 if causal else 1) + (8 if causal else 0),
                            causal=causal, codebook_size=K, groups=G)
    params = model.init_params(cfg, seed=0)
    rng = np.random.default_rng(0)
    sample = rng.standard_normal((4096, D)).astype(np.float32) * 0.5
    for i, b in enumerate(params.blocks):
        cents = sample[rng.choice(4096, K, replace=False)]
        b.codebook = vq.Codebook(layer_id=i, groups=G,
                                 centroids=[np.ascontiguousarray(c) for c in np.split(cents, G, axis=1)])
    plan = cluster.partition_tokens(T, n, class_replication=not causal)
    rank = n - 1 if rank is None else rank
    comm = LoopbackExchange(rank, n) if n > 1 else None
    rt = AstraRuntime(params, plan, batch=B, mode="generate" if causal else "classify",
                      precision="fast", comm=comm)
    if causal:
        rt.set_ids(rng.integers(0, C, size=(B, T)))
    else:
        rt.stage_input(data.make_classify_batch(D, T, B, seed=1))
    torch.cuda.synchronize()
    try:
        rt.capture(warmup=1)
        graphed = True
    except Exception:
        torch.cuda.synchronize()
        rt.graph, graphed = None, False
    for _ in range(warmup):
        rt.run() if not causal else rt.forward()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        rt.run() if (graphed or not causal) else rt.forward()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    unit = "tokens/s (prefill)" if causal else "images/s"
    per_rank_items = B * (T if causal else 1)
    return {"config": name, "n": n, "rank": rank, "ms_per_step": round(ms, 4),
            "per_layer_ms": round(ms / L, 4), "batch": B, "tokens": T,
            "box_rate_if_ranks_parallel": round(per_rank_items / (ms / 1000), 1), "unit": unit,
            "cuda_graph": graphed, "exchange": "loopback (no NCCL)" if n > 1 else "none"}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", nargs="+", default=["vitb"])
    ap.add_argument("--n", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    for name in args.config:
        for n in args.n:
            print(json.dumps(run(name, n, args.steps, args.warmup)), flush=True)
