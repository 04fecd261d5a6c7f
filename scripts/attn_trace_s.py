"""Timeline of the single-pipeline attention kernel (CTA 0), ViT-B/16 B=64 (debug aid)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_19342_b200 import _native, cluster, data, model, vq  # noqa: E402
from paper_2505_19342_b200.runtime import AstraRuntime  # noqa: E402

cfg = model.ModelConfig(layers=1, hidden=768, heads=12, vocab_or_classes=1000, max_tokens=197,
                        causal=False, codebook_size=1024, groups=1)
params = model.init_params(cfg, seed=0)
xs = data.make_classify_batch(768, 196, 64, seed=1)
rng = np.random.default_rng(0)
for i, b in enumerate(params.blocks):
    c = xs.reshape(-1, 768)[rng.choice(64 * 196, 1024, replace=False)]
    b.codebook = vq.Codebook(layer_id=i, groups=1, centroids=[c])
rt = AstraRuntime(params, cluster.partition_tokens(196, 1), batch=64, precision="fast")
rt.stage_input(xs)
rt.forward()
torch.cuda.synchronize()
buf = torch.zeros(512 + 2 * 1024, dtype=torch.int64, device="cuda")
lib = _native.load()
lib.astra_attention_variant(2)
rt.forward()
torch.cuda.synchronize()
lib.astra_attention_trace(buf.data_ptr())
rt.forward()
torch.cuda.synchronize()
lib.astra_attention_trace(None)
allb = buf.cpu().numpy().astype(np.int64)
t = allb[:512].reshape(32, 16)
cta = allb[512:].reshape(-1, 2)
cta = cta[cta[:, 0] > 0]
t0 = t[t > 0].min()
names = ["S_tempty", "S_iss", "PV_iss", "sm_st", "p_full", "ld_v", "p1bar", "o_full", "drained",
         "S_qkfull", "PV_pfull", "PV_vfull", "sm_top", "sfull_ok", "est_done", "-"]
print("unit " + " ".join(f"{x:>8s}" for x in names))
for u in range(32):
    if t[u].max() == 0:
        break
    print(f"{u:4d} " + " ".join(f"{(t[u][k] - t0) / 1000:8.2f}" if t[u][k] else "       -" for k in range(16)))

c0 = cta[:, 0].min()
st, en = (cta[:, 0] - c0) / 1000, (cta[:, 1] - c0) / 1000
print(f"CTAs {len(cta)}: start min/med/max {st.min():.2f}/{np.median(st):.2f}/{st.max():.2f}  end min/med/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f} us")
print("end-time histogram (us):", np.histogram(en, bins=8))
print("CTA0 first stamp vs CTA start:", (t[t > 0].min() - cta[0, 0]) / 1000)
