"""BASELINE config #4 golden fixtures (ViT-L/16@384 with grouped codebooks), produced by running
the REFERENCE (seqvq 0.1.0).  Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=8 python tests/golden/make_golden_vitl.py

ViT-L/16@384 shape (L=24, D=1024, H=16, T=576, 1000 classes), G=16 groups of 64 dims, K=256
codes per group, seed 0, the reference recipe:

* weights   init_params(cfg, seed=0)                                   (model.py:126-160)
* codebooks initialize_codebooks(params, make_classify_data(1024, 576, 4, seed=0,
            task_seed=0), "classify", 256, 16, seed=0)                  (train.py:176-189)
* inputs    make_classify_data(1024, 576, 2, seed=1, task_seed=0)      (train.py:66-90)

Outputs (next to this script): ``vitl_g16k256_codebooks.npz`` (the reference's centroids, fp32
[24, 16, 256, 64], with SHA-256) and ``golden_vitl.npz`` (for N in {1, 4}: ``run_inference``
logits and every layer's VQ indices in global token order, int16 [images, L * T * G]).
tests/test_config4_gpu.py checks the GPU runtime against them.
"""

from __future__ import annotations

import hashlib
import importlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

model = importlib.import_module("seqvq.model")
cluster = importlib.import_module("seqvq.cluster")
train = importlib.import_module("seqvq.train")

L, D, H, T, K, G, IMAGES, FIT = 24, 1024, 16, 576, 256, 16, 2, 4


def _capture_run(params, plan, x):
    caps = []
    orig = cluster.quantize

    def q(cb, xx):
        res = orig(cb, xx)
        caps.append(res[0].indices.copy())
        return res

    cluster.quantize = q
    try:
        r = cluster.run_inference(params, plan, x, "classify", workers=1)
    finally:
        cluster.quantize = orig
    return r, np.concatenate([c.reshape(-1) for c in caps]).astype(np.int16)


def main(ns=(1, 4)):
    t0 = time.time()
    mcfg = model.ModelConfig(layers=L, hidden=D, heads=H, vocab_or_classes=1000,
                             max_tokens=T + 1, causal=False, codebook_size=K, groups=G)
    params = model.init_params(mcfg, seed=0)
    fit = train.make_classify_data(D, T, FIT, seed=0, task_seed=0)
    train.initialize_codebooks(params, fit, "classify", K, G, seed=0)
    print(f"codebooks fitted in {time.time() - t0:.1f} s", flush=True)
    cents = np.stack([np.stack(b.codebook.centroids) for b in params.blocks]).astype(np.float32)
    np.savez(OUT / "vitl_g16k256_codebooks.npz", centroids=cents,
             centroids_sha256=np.array(hashlib.sha256(cents.tobytes()).hexdigest()))
    xs = train.make_classify_data(D, T, IMAGES, seed=1, task_seed=0)[0]
    out = {}
    meta = {"images": IMAGES, "ns": list(ns), "L": L, "D": D, "H": H, "T": T, "K": K, "G": G,
            "fit_images": FIT, "centroids_sha256": hashlib.sha256(cents.tobytes()).hexdigest(),
            "inputs_sha256": hashlib.sha256(np.stack(xs).tobytes()).hexdigest()}
    for n in ns:
        plan = cluster.partition_tokens(T, n)
        logits = np.zeros((IMAGES, 1000), np.float32)
        idx = np.zeros((IMAGES, L * T * G), np.int16)
        for b in range(IMAGES):
            r, caps = _capture_run(params, plan, xs[b])
            logits[b] = np.asarray(r.output).reshape(-1)
            idx[b] = caps
            if b == 0:
                meta[f"n{n}_ledger"] = r.ledger.to_csv()
        out[f"n{n}_logits"] = logits
        out[f"n{n}_indices"] = idx
        meta[f"n{n}_top1"] = logits.argmax(1).tolist()
        print(f"N={n}: {IMAGES} images done at {time.time() - t0:.0f} s", flush=True)
    np.savez_compressed(OUT / "golden_vitl.npz", **out)
    (OUT / "golden_vitl_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
