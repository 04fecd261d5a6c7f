"""Timeline of the persistent attention kernel (CTA 0) on the ViT-B/16 B=64 workload:
per unit, globaltimer stamps of the loader / MMA / softmax events (debug aid)."""
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
rt.forward()
torch.cuda.synchronize()
buf = torch.zeros(512 + 2 * 1024, dtype=torch.int64, device="cuda")
lib = _native.load()
lib.astra_attention_trace(buf.data_ptr())
rt.profile = {}
rt.forward()
torch.cuda.synchronize()
lib.astra_attention_trace(None)
ms = [s.elapsed_time(e) for s, e in rt.profile["attention"]]
print("attention ms", ms)
allb = buf.cpu().numpy().astype(np.int64)
t = allb[:512].reshape(32, 16)
se = allb[512:].reshape(-1, 2)
se = se[se[:, 0] > 0]
c0 = se[:, 0].min()
st, en = (se[:, 0] - c0) / 1000, (se[:, 1] - c0) / 1000
print(f"CTAs {len(se)}: start min/med/max {st.min():.2f}/{np.median(st):.2f}/{st.max():.2f} us, "
      f"end min/med/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f} us")
print("end histogram (us):", np.histogram(en, bins=8)[0].tolist(), np.round(np.histogram(en, bins=8)[1], 1).tolist())
t0 = t[t > 0].min()
names = ["0p2end", "0S", "0PV", "0sm_st", "0sm_end", "0Sdone", "0p1end", "0top", "1p2end", "1S", "1PV", "1sm_st", "1sm_end", "1Sdone", "1p1end", "1top"]
print("unit " + " ".join(f"{x:>8s}" for x in names))
for u in range(32):
    if t[u].max() == 0:
        break
    print(f"{u:4d} " + " ".join(f"{(v - t0) / 1000:8.2f}" if v else "       -" for v in t[u]))
