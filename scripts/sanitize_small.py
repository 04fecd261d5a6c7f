"""Small forwards for compute-sanitizer: ViT-width model (2 layers, D=768) at N=1 and N=4 in both
precision modes (and B=12 at N=1: the 256-code records tiles), a grouped-codebook run (G=16, K=4096: overflow scans) and a causal generate."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_19342_b200 import cluster, data, model, vq  # noqa: E402
from paper_2505_19342_b200.runtime import AstraRuntime  # noqa: E402

rng = np.random.default_rng(0)
# (B = 12 at N = 1: 2364 rows, enough row blocks for the 256-code records tiles and the
# half-warp finalize)
for causal, G, K, T, B, ns in ((False, 1, 1024, 196, 4, (1, 4)), (False, 1, 1024, 196, 12, (1,)),
                               (False, 16, 4096, 196, 2, (1, 4)), (True, 1, 256, 128, 2, (1, 4))):
    cfg = model.ModelConfig(layers=2, hidden=768, heads=12, vocab_or_classes=100,
                            max_tokens=T + (8 if causal else 1), causal=causal, codebook_size=K,
                            groups=G)
    params = model.init_params(cfg, seed=0)
    sample = rng.standard_normal((8192, 768)).astype(np.float32) * 0.5
    for i, b in enumerate(params.blocks):
        c = sample[rng.choice(8192, K, replace=False)]
        b.codebook = vq.Codebook(layer_id=i, groups=G, centroids=[np.ascontiguousarray(x) for x in np.split(c, G, axis=1)])
    for n in ns:
        for prec in ("fast", "parity"):
            plan = cluster.partition_tokens(T, n, class_replication=not causal)
            rt = AstraRuntime(params, plan, batch=B, precision=prec,
                              mode="generate" if causal else "classify")
            if causal:
                rt.set_ids(rng.integers(0, 100, size=(B, T)))
            else:
                rt.stage_input(data.make_classify_batch(768, T, B, seed=1))
            rt.forward()
            torch.cuda.synchronize()
            rt.check_errors()
            print("ok", causal, G, K, n, prec, flush=True)
