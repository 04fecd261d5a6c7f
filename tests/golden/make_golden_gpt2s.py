"""BASELINE config #3 golden fixtures (GPT-2-small causal prefill + greedy decode), produced by
running the REFERENCE (seqvq 0.1.0).  Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=8 python tests/golden/make_golden_gpt2s.py

GPT-2-small shape (L=12, D=768, H=12, vocab 50,257, causal), prompt T=1024, K=1024, G=1, seed 0:

* weights   init_params(cfg, seed=0)                                     (model.py:126-160)
* codebooks initialize_codebooks(params, 2 sequences of 1025 ids from the named stream
            (0, "gpt2-ids"), "lm", 1024, 1, seed=0)                      (train.py:176-189)
* prompts   2 x 1024 ids from the named stream (1, "gpt2-ids")          (rng.py:24-37)

Outputs (next to this script): ``gpt2s_codebooks.npz`` (the reference's centroids, fp32
[12, 1, 1024, 768], with SHA-256) and ``golden_gpt2s.npz`` (for N in {1, 4}: the 4 tokens
``run_inference(..., "generate", steps=4)`` returns and every layer's prefill VQ indices in
global token order).  tests/test_config3_gpu.py checks the GPU runtime against them.
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
rng = importlib.import_module("seqvq.rng")

L, D, H, V, T, K, G, SEQS, STEPS = 12, 768, 12, 50257, 1024, 1024, 1, 2, 4


def _capture_run(params, plan, ids):
    caps = []
    orig = cluster.quantize

    def q(cb, xx):
        res = orig(cb, xx)
        caps.append(res[0].indices.copy())
        return res

    cluster.quantize = q
    try:
        r = cluster.run_inference(params, plan, ids, "generate", steps=STEPS, workers=1)
    finally:
        cluster.quantize = orig
    return r, np.concatenate([c.reshape(-1) for c in caps]).astype(np.int16)


def main(ns=(1, 4)):
    t0 = time.time()
    mcfg = model.ModelConfig(layers=L, hidden=D, heads=H, vocab_or_classes=V,
                             max_tokens=T + STEPS, causal=True, codebook_size=K, groups=G)
    params = model.init_params(mcfg, seed=0)
    fit = list(rng.generator(0, "gpt2-ids").integers(0, V, size=(2, T + 1)))
    train.initialize_codebooks(params, fit, "lm", K, G, seed=0)
    print(f"codebooks fitted in {time.time() - t0:.1f} s", flush=True)
    cents = np.stack([np.stack(b.codebook.centroids) for b in params.blocks]).astype(np.float32)
    np.savez(OUT / "gpt2s_codebooks.npz", centroids=cents,
             centroids_sha256=np.array(hashlib.sha256(cents.tobytes()).hexdigest()))
    prompts = rng.generator(1, "gpt2-ids").integers(0, V, size=(SEQS, T))
    out = {"prompts": prompts.astype(np.int32)}
    meta = {"seqs": SEQS, "ns": list(ns), "L": L, "D": D, "H": H, "V": V, "T": T, "K": K, "G": G,
            "steps": STEPS, "centroids_sha256": hashlib.sha256(cents.tobytes()).hexdigest()}
    for n in ns:
        plan = cluster.partition_tokens(T, n, class_replication=False)
        toks = np.zeros((SEQS, STEPS), np.int32)
        idx = np.zeros((SEQS, L * T * G), np.int16)
        for b in range(SEQS):
            r, caps = _capture_run(params, plan, prompts[b])
            toks[b] = r.output
            idx[b] = caps
            if b == 0:
                meta[f"n{n}_ledger"] = r.ledger.to_csv()
        out[f"n{n}_tokens"] = toks
        out[f"n{n}_indices"] = idx
        print(f"N={n}: {SEQS} prompts done at {time.time() - t0:.0f} s: {toks.tolist()}", flush=True)
    np.savez_compressed(OUT / "golden_gpt2s.npz", **out)
    (OUT / "golden_gpt2s_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
