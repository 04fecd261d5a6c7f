"""Per-op device time (eager, ops serialised, CUDA events; bench._profile) of ONE rank of an
N-way split with the loopback exchange — which ops sit on the N > 1 critical path.

    python scripts/rank_ops.py [--config vitb] [--n 2 4 8]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))
import bench  # noqa: E402
import bench_ranks  # noqa: E402
from paper_2505_19342_b200 import cluster, data, model, vq  # noqa: E402
from paper_2505_19342_b200.runtime import AstraRuntime, LoopbackExchange  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="vitb")
    ap.add_argument("--n", type=int, nargs="+", default=[2, 4, 8])
    a = ap.parse_args()
    L, D, H, C, T, B, K, G, causal = bench_ranks.CONFIGS[a.config]
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
    for n in a.n:
        plan = cluster.partition_tokens(T, n, class_replication=not causal)
        rt = AstraRuntime(params, plan, batch=B, mode="generate" if causal else "classify",
                          precision="fast", comm=LoopbackExchange(n - 1, n) if n > 1 else None)
        if causal:
            rt.set_ids(rng.integers(0, C, size=(B, T)))
        else:
            rt.stage_input(data.make_classify_batch(D, T, B, seed=1))
        rt.forward()
        torch.cuda.synchronize()
        prof = bench._profile(rt, steps=3)
        print(json.dumps({"config": a.config, "n": n,
                          "ops_us": {k: round(v["avg_ms"] * 1000, 2) for k, v in prof.items()}}), flush=True)
        del rt


if __name__ == "__main__":
    main()
