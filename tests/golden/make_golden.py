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


def make_model_api():
    """Model-level API (model.py:198-432) outputs of the reference on toy configs, plus the
    inputs/outputs of acceptance criterion 3 (test_acceptance.py:114-150)."""
    out = {}
    # encoder toy (the shipped infer_classify.json model)
    mk = dict(layers=2, hidden=32, heads=4, vocab_or_classes=4, codebook_size=8, max_tokens=512,
              causal=False)
    params = model.init_params(model.ModelConfig(**mk), seed=0)
    data = train.make_classify_data(32, 16, 8, seed=0, task_seed=0)
    train.initialize_codebooks(params, data, "classify", 8, 1, seed=0)
    x = train.make_classify_data(32, 16, 1, seed=1, task_seed=0)[0][0]
    out["enc_codebooks"] = np.stack([np.stack(b.codebook.centroids) for b in params.blocks])
    out["enc_x"] = x
    for n in (1, 2, 4):
        for cm in ("distributed", "single"):
            plan = cluster.partition_tokens(16, n)
            out[f"enc_classify_n{n}_{cm}"] = model.classify(params, plan, x, cls_mode=cm).data
    plan4 = cluster.partition_tokens(16, 4)
    x0 = model.embed_classifier_inputs(params, x)
    out["enc_embed"] = x0.data
    infos = []
    content, reps = model.run_blocks(params, plan4, x0, on_layer=lambda i, info: infos.append(info))
    out["enc_blocks_content"], out["enc_blocks_replicas"] = content.data, reps.data
    for i, info in enumerate(infos):
        for k in ("x_in", "x_hat", "k_full", "v_full", "k_hat", "v_hat"):
            out[f"enc_info{i}_{k}"] = np.asarray(info[k])
        out[f"enc_info{i}_q"] = info["q"].indices
    out["enc_aggregate"] = model.aggregate_class_tokens(reps).data
    books = model.exact_codebooks_from_reference(params, cluster.partition_tokens(16, 1), x)
    out["enc_exact_books"] = np.stack([np.stack(b.centroids) for b in books])
    # causal toy (the shipped infer_generate.json model)
    mk = dict(layers=2, hidden=32, heads=4, vocab_or_classes=16, codebook_size=8, max_tokens=17,
              causal=True)
    params = model.init_params(model.ModelConfig(**mk), seed=0)
    data = train.make_lm_data(16, 8, 8, seed=0, task_seed=0)
    train.initialize_codebooks(params, data, "lm", 8, 1, seed=0)
    ids = train.make_lm_data(16, 8, 1, seed=1, task_seed=0)[0][:8]
    out["dec_codebooks"] = np.stack([np.stack(b.codebook.centroids) for b in params.blocks])
    out["dec_ids"] = ids
    out["dec_embed"] = model.embed_lm_inputs(params, ids, offset=3).data
    for n in (1, 2, 4):
        plan = cluster.partition_tokens(8, n, class_replication=False)
        out[f"dec_lm_logits_n{n}"] = model.lm_logits(params, plan, ids).data
        out[f"dec_generate_n{n}"] = np.array(model.generate(params, plan, ids, 6))
        st, first = model.prefill_decode_state(params, plan, ids)
        out[f"dec_prefill_first_n{n}"] = np.array([first])
        for i in range(len(st.k)):
            out[f"dec_prefill_n{n}_k{i}"], out[f"dec_prefill_n{n}_v{i}"] = st.k[i], st.v[i]
    # acceptance criterion 3: same draws as test_acceptance.py:114-150
    draw = np.random.default_rng(7)
    for trial in range(100):
        causal = bool(draw.integers(0, 2))
        layers = int(draw.integers(1, 4))
        heads = int(draw.choice([1, 2]))
        hidden = int(draw.choice([4, 8, 12, 16]))
        groups = int(draw.choice([1, 2]))
        devices = int(draw.choice([1, 2, 4]))
        tokens = int(draw.integers(max(devices, 2), 33))
        cfg = model.ModelConfig(layers=layers, hidden=hidden, heads=heads,
                                vocab_or_classes=int(draw.integers(3, 9)), max_tokens=tokens + 1,
                                causal=causal, codebook_size=4, groups=groups)
        params = model.init_params(cfg, seed=trial)
        plan1 = cluster.partition_tokens(tokens, 1)
        plan_n = cluster.partition_tokens(tokens, devices, class_replication=not causal)
        if causal:
            inputs = draw.integers(0, cfg.vocab_or_classes, size=tokens)
            reference = model.lm_logits(params, plan1, inputs).data
        else:
            inputs = draw.normal(size=(tokens, hidden)).astype(np.float32)
            reference = model.classify(params, plan1, inputs).data
        books = model.exact_codebooks_from_reference(params, plan1, inputs)
        for b, cb in zip(params.blocks, books):
            b.codebook = cb
        if causal:
            got = model.lm_logits(params, plan_n, inputs).data
        else:
            got = cluster.run_inference(params, plan_n, inputs, mode="classify").output
        out[f"c3_{trial}_cfg"] = np.array([int(causal), layers, heads, hidden, groups, devices,
                                           tokens, cfg.vocab_or_classes])
        out[f"c3_{trial}_inputs"] = inputs
        out[f"c3_{trial}_reference"] = reference
        out[f"c3_{trial}_got"] = np.asarray(got)
    np.savez_compressed(OUT / "golden_model.npz", **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["model"]:
        make_model_api()
        sys.exit(0)
    make_vq()
    make_attention()
    make_infer()
    make_model_api()
    for p in sorted(OUT.glob("golden_*")):
        print(p.name, p.stat().st_size)
