"""Headline-config golden fixtures, produced by running the REFERENCE (seqvq 0.1.0).

Run in the build container, where /root/reference exists (≈10 min on 8 cores):

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=8 python tests/golden/make_golden_vitb.py

BASELINE configs #1/#2: ViT-B/16 shape (L=12, D=768, H=12, T=196, 1000 classes), K=1024,
G=1, seed 0 — exactly the CLI's `_prepared_params` recipe (cli.py:83-105):

* weights   init_params(cfg, seed=0)                                   (model.py:126-160)
* codebooks initialize_codebooks(params, make_classify_data(768, 196, 8, seed=0,
            task_seed=0), "classify", 1024, 1, seed=0)                  (train.py:176-189)
* inputs    make_classify_data(768, 196, 64, seed=1, task_seed=0)       (train.py:66-90);
            image 0 is config #1's input (cli.py:126-128).

Outputs (next to this script):

* ``vitb16_codebooks.npz`` — the reference's fitted centroids, fp32 [12, G=1, 1024, 768]
  (the AVQ1 blobs' centroid sections, vq.py:328-339; the fp64 EMA accumulators are not
  needed for inference and would triple the size), plus the SHA-256 of every full AVQ1
  blob the reference wrote and of the centroid bytes.
* ``golden_vitb.npz`` — for N in {1, 2, 4, 8} and all 64 images: ``run_inference`` logits
  and every layer's VQ indices (cluster.py:272-275 captures, global token order).
* ``golden_vitb_meta.json`` — ledgers per N and config #1's headline (predicted class).

bench.py loads the codebooks for both arms; tests/test_headline_gpu.py checks the GPU
forward against the logits/indices at L=12 in both precision modes.
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

vq = importlib.import_module("seqvq.vq")
model = importlib.import_module("seqvq.model")
cluster = importlib.import_module("seqvq.cluster")
train = importlib.import_module("seqvq.train")

L, D, H, T, K, G, B = 12, 768, 12, 196, 1024, 1, 64


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


def main(ns=(1, 2, 4, 8), images=B):
    t0 = time.time()
    mcfg = model.ModelConfig(layers=L, hidden=D, heads=H, vocab_or_classes=1000, max_tokens=197,
                             causal=False, codebook_size=K, groups=G)
    params = model.init_params(mcfg, seed=0)
    fit = train.make_classify_data(D, T, 8, seed=0, task_seed=0)
    train.initialize_codebooks(params, fit, "classify", K, G, seed=0)
    print(f"codebooks fitted in {time.time() - t0:.1f} s", flush=True)
    cents = np.stack([np.stack(b.codebook.centroids) for b in params.blocks]).astype(np.float32)
    avq = [hashlib.sha256(vq.save_codebook(b.codebook)).hexdigest() for b in params.blocks]
    np.savez(OUT / "vitb16_codebooks.npz", centroids=cents,
             centroids_sha256=np.array(hashlib.sha256(cents.tobytes()).hexdigest()),
             avq1_sha256=np.array(avq))
    xs = train.make_classify_data(D, T, images, seed=1, task_seed=0)[0]
    out, meta = {}, {"images": images, "ns": list(ns),
                     "centroids_sha256": hashlib.sha256(cents.tobytes()).hexdigest(),
                     "avq1_sha256": avq,
                     "inputs_sha256": hashlib.sha256(np.stack(xs).tobytes()).hexdigest()}
    for n in ns:
        plan = cluster.partition_tokens(T, n)
        logits = np.zeros((images, 1000), np.float32)
        idx = np.zeros((images, L * T), np.int16)
        for b in range(images):
            r, caps = _capture_run(params, plan, xs[b])
            logits[b] = np.asarray(r.output).reshape(-1)
            idx[b] = caps
            if b == 0:
                meta[f"n{n}_ledger"] = r.ledger.to_csv()
                meta[f"n{n}_bits_per_token"] = r.ledger.bits_per_token(T)
        out[f"n{n}_logits"] = logits
        out[f"n{n}_indices"] = idx
        meta[f"n{n}_top1"] = logits.argmax(1).tolist()
        print(f"N={n}: {images} images done at {time.time() - t0:.0f} s; "
              f"image0 predicted={int(logits[0].argmax())}", flush=True)
    meta["config1_predicted"] = int(out["n4_logits"][0].argmax()) if 4 in ns else None
    np.savez_compressed(OUT / "golden_vitb.npz", **out)
    (OUT / "golden_vitb_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
