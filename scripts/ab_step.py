"""A/B helper: graphed step time and per-op eager times of the B=64 ViT-B forward for the
library named by ASTRA_B200_LIB (run once per library, alternating, on the same box)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_19342_b200 import cluster, data, model, vq  # noqa: E402
from paper_2505_19342_b200.runtime import AstraRuntime  # noqa: E402

cfg = model.ModelConfig(layers=12, hidden=768, heads=12, vocab_or_classes=1000, max_tokens=197,
                        causal=False, codebook_size=1024, groups=1)
params = model.init_params(cfg, seed=0)
xs = data.make_classify_batch(768, 196, 64, seed=1)
rng = np.random.default_rng(0)
flat = xs.reshape(-1, 768)
for i, b in enumerate(params.blocks):
    b.codebook = vq.Codebook(layer_id=i, groups=1, centroids=[flat[rng.choice(len(flat), 1024, replace=False)]])
rt = AstraRuntime(params, cluster.partition_tokens(196, 1), batch=64, precision="fast")
rt.stage_input(xs)
rt.capture(warmup=2)
for _ in range(20):
    rt.run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(200):
    rt.run()
e.record()
torch.cuda.synchronize()
step = s.elapsed_time(e) / 200
rt.overlap_vq = False
rt.profile = {}
for _ in range(5):
    rt.forward()
torch.cuda.synchronize()
ops = {k: np.median([a.elapsed_time(b) for a, b in v]) * 1000 for k, v in rt.profile.items()}
print(f"{Path(os.environ.get('ASTRA_B200_LIB', 'default')).name}: step {step:.4f} ms | " +
      " ".join(f"{k} {v:.1f}" for k, v in ops.items() if k.startswith("gemm")))
