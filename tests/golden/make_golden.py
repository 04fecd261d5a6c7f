"""Generate golden fixtures by running the REFERENCE (seqvq 0.1.0) itself.

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The fixtures (small .npz files next to this script) pin oracle/astra_oracle.py
(the CPU restatement) to the reference's own outputs; the GPU parity tests
then compare the CUDA path with the oracle and with these fixtures.  Nothing
at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import importlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parents[1]))

from tests.golden.cases import ATT_CASES, VQ_CASES, att_case_inputs, vq_case_inputs  # noqa: E402

vq = importlib.import_module("seqvq.vq")
att = importlib.import_module("seqvq.attention")
model = importlib.import_module("seqvq.model")
cluster = importlib.import_module("seqvq.cluster")
train = importlib.import_module("seqvq.train")
tensor = importlib.import_module("seqvq.tensor")


def _codebook(cents):
    g = len(cents)
    k = cents[0].shape[0]
    return vq.Codebook(layer_id=0, groups=g, centroids=[c.astype(np.float32) for c in cents],
                       ema_counts=np.ones((g, k)), ema_sums=[c.astype(np.float64) for c in cents])


def make_vq():
    out = {}
    for i, (k, d, g, m) in enumerate(VQ_CASES):
        if i == len(VQ_CASES) - 1:   # equidistant tie -> lowest index (test_vq.py:68-73)
            cents = [np.array([[1.0, 0.0], [-1.0, 0.0]], np.float32)]
            x = np.zeros((m, d), np.float32)
        else:
            cents, x = vq_case_inputs(i, k, d, g, m)
        q, x_hat = vq.quantize(_codebook(cents), x)
        out[f"c{i}_idx"] = q.indices
        out[f"c{i}_xhat_sha256"] = np.frombuffer(
            hashlib.sha256(np.ascontiguousarray(x_hat).tobytes()).digest(), np.uint8)
        out[f"c{i}_bits"] = np.array([q.bits_per_token])
    out["ncases"] = np.array([len(VQ_CASES)])
    np.savez_compressed(OUT / "golden_vq.npz", **out)


def make_attention():
    out = {}
    cases = ATT_CASES
    for i, (r, c, d, h, p) in enumerate(cases):
        q, k, v, mask = att_case_inputs(i, r, c, d, p)
        o = att.multihead_attention(tensor.constant(q), tensor.constant(k), tensor.constant(v),
                                    mask, h)
        out.update({f"c{i}_heads": np.array([h]), f"c{i}_out": o.data})
    out["ncases"] = np.array([len(cases)])
    np.savez_compressed(OUT / "golden_attention.npz", **out)


def _capture_run(params, plan, inputs, mode, steps=0, cls_mode="distributed"):
    caps = []
    orig = cluster.quantize

    def q(cb, x):
        res = orig(cb, x)
        caps.append(res[0].indices.copy())
        return res

    cluster.quantize = q
    try:
        r = cluster.run_inference(params, plan, inputs, mode, steps=steps, cls_mode=cls_mode)
    finally:
        cluster.quantize = orig
    return r, caps


def _cb_digest(params):
    h = hashlib.sha256()
    for b in params.blocks:
        for c in b.codebook.centroids:
            h.update(np.ascontiguousarray(c, "<f4").tobytes())
    return h.hexdigest()


def make_infer():
    """CLI-equivalent runs (cli.py:83-157) of the shipped configs plus ViT-B-width cases."""
    out = {}
    meta = {}
    specs = [
        # name, model kwargs, tokens, devices list, seed, cls modes, mode, steps
        ("toy", dict(layers=2, hidden=32, heads=4, vocab_or_classes=4, codebook_size=8,
                     max_tokens=512, causal=False), 16, [1, 2, 4], 0, ["distributed", "single"],
         "classify", 0),
        ("toyg2", dict(layers=2, hidden=32, heads=4, vocab_or_classes=4, codebook_size=16,
                       groups=4, max_tokens=512, causal=False), 16, [1, 3, 4], 1, ["distributed"],
         "classify", 0),
        ("gen", dict(layers=2, hidden=32, heads=4, vocab_or_classes=16, codebook_size=8,
                     max_tokens=17, causal=True), 8, [1, 2, 4], 0, [None], "generate", 6),
        ("vitb2", dict(layers=2, hidden=768, heads=12, vocab_or_classes=1000,
                       codebook_size=1024, max_tokens=197, causal=False), 196, [1, 4, 8], 0,
         ["distributed"], "classify", 0),
    ]
    for name, mk, tokens, devs, seed, modes, mode, steps in specs:
        mcfg = model.ModelConfig(**mk)
        params = model.init_params(mcfg, seed=seed)
        if mcfg.causal:
            data = train.make_lm_data(mcfg.vocab_or_classes, tokens, 8, seed=seed, task_seed=seed)
            train.initialize_codebooks(params, data, "lm", mcfg.codebook_size, mcfg.groups,
                                       seed=seed)
            inputs = train.make_lm_data(mcfg.vocab_or_classes, tokens, 1, seed=seed + 1,
                                        task_seed=seed)[0][:tokens]
        else:
            data = train.make_classify_data(mcfg.hidden, tokens, 8, seed=seed, task_seed=seed)
            train.initialize_codebooks(params, data, "classify", mcfg.codebook_size, mcfg.groups,
                                       seed=seed)
            inputs = train.make_classify_data(mcfg.hidden, tokens, 1, seed=seed + 1,
                                              task_seed=seed)[0][0]
        meta[name] = dict(model=mk, tokens=tokens, devices=devs, seed=seed, mode=mode,
                          steps=steps, codebook_sha256=_cb_digest(params))
        if mcfg.hidden <= 64:
            out[f"{name}_codebooks"] = np.stack([np.stack(b.codebook.centroids)
                                                 for b in params.blocks])
            out[f"{name}_inputs"] = np.asarray(inputs)
        for n in devs:
            plan = cluster.partition_tokens(tokens, n, class_replication=not mcfg.causal)
            for cm in modes:
                tag = f"{name}_n{n}" + (f"_{cm}" if cm else "")
                r, caps = _capture_run(params, plan, inputs, mode, steps=steps,
                                       cls_mode=cm or "distributed")
                out[f"{tag}_output"] = np.asarray(r.output)
                out[f"{tag}_indices"] = np.concatenate([c.reshape(-1) for c in caps])
                meta[f"{tag}_ledger"] = r.ledger.to_csv()
    np.savez_compressed(OUT / "golden_infer.npz", **out)
    (OUT / "golden_infer_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


if __name__ == "__main__":
    make_vq()
    make_attention()
    make_infer()
    for p in sorted(OUT.glob("golden_*")):
        print(p.name, p.stat().st_size)
