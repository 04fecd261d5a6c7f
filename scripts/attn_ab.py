"""A/B of the attention kernel variants on the ViT-B/16 B=64 workload: the runtime's own
astra_attention call (layer 0 arguments) replayed back to back, CUDA-event timed."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_19342_b200 import _native, cluster, data, model, vq  # noqa: E402
from paper_2505_19342_b200.runtime import AstraRuntime, LoopbackExchange  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = model.ModelConfig(layers=1, hidden=768, heads=12, vocab_or_classes=1000, max_tokens=197,
                        causal=False, codebook_size=1024, groups=1)
params = model.init_params(cfg, seed=0)
xs = data.make_classify_batch(768, 196, 64, seed=1)
rng = np.random.default_rng(0)
for i, b in enumerate(params.blocks):
    c = xs.reshape(-1, 768)[rng.choice(64 * 196, 1024, replace=False)]
    b.codebook = vq.Codebook(layer_id=i, groups=1, centroids=[c])
comm = LoopbackExchange(n - 1, n) if n > 1 else None   # one rank (the last) of an N-way split
rt = AstraRuntime(params, cluster.partition_tokens(196, n), batch=64, precision="fast", comm=comm)
rt.stage_input(xs)
calls = []
orig = _native.call


def spy(name, *args):
    if name == "astra_attention":
        calls.append(args)
    return orig(name, *args)


_native.call = spy
rt.forward()
torch.cuda.synchronize()
_native.call = orig
args = calls[0]
lib = _native.load()
res = {}
for rep in range(3):
    for v in (0, 2, 1, "simt"):
        lib.astra_attention_force_simt(int(v == "simt"))
        lib.astra_attention_variant(0 if v == "simt" else v)
        for _ in range(5):
            lib.astra_attention(*args)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50):
            lib.astra_attention(*args)
        e.record()
        torch.cuda.synchronize()
        res.setdefault(v, []).append(s.elapsed_time(e) / 50 * 1000)
lib.astra_attention_variant(0)
lib.astra_attention_force_simt(0)
for v, t in res.items():
    print(f"variant {v}: {' '.join('%.1f' % x for x in t)} us per launch")
