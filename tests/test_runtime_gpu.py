"""End-to-end parity of the GPU Astra forward (cluster.run_inference) against the
reference's golden runs and the CPU oracle, at the same device count N."""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import astra_oracle as O

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
META = json.loads((G / "golden_infer_meta.json").read_text())
GOLD = np.load(G / "golden_infer.npz")
_CACHE = {}


def _setup(name):
    """Our params (same seeded init as the reference) + the oracle's k-means codebooks."""
    if name in _CACHE:
        return _CACHE[name]
    from paper_2505_19342_b200 import model, vq
    m = META[name]
    cfg = model.ModelConfig(**m["model"])
    params = model.init_params(cfg, seed=m["seed"])
    ocfg = O.Config(**m["model"])
    op = O.init_params(ocfg, seed=m["seed"])
    t, seed = m["tokens"], m["seed"]
    if cfg.causal:
        data = O.make_lm_data(cfg.vocab_or_classes, t, 8, seed=seed, task_seed=seed)
        O.initialize_codebooks(op, data, "lm", seed=seed)
        inputs = O.make_lm_data(cfg.vocab_or_classes, t, 1, seed=seed + 1, task_seed=seed)[0][:t]
    else:
        xs, _ = O.make_classify_data(cfg.hidden, t, 8, seed=seed, task_seed=seed)
        O.initialize_codebooks(op, xs, "classify", seed=seed)
        inputs = O.make_classify_data(cfg.hidden, t, 1, seed=seed + 1, task_seed=seed)[0][0]
    for i, b in enumerate(params.blocks):
        b.codebook = vq.Codebook(layer_id=i, groups=cfg.groups, centroids=op.codebooks[i])
    _CACHE[name] = (params, op, inputs)
    return _CACHE[name]


CLASSIFY = [("toy", n, cm) for n in (1, 2, 4) for cm in ("distributed", "single")] + \
           [("toyg2", n, "distributed") for n in (1, 3, 4)] + \
           [("vitb2", n, "distributed") for n in (1, 4, 8)]


@pytest.mark.parametrize("name,n,cls_mode", CLASSIFY)
def test_classify_parity_vs_reference(cuda, name, n, cls_mode):
    from paper_2505_19342_b200 import cluster
    from paper_2505_19342_b200.runtime import AstraRuntime
    params, op, inputs = _setup(name)
    plan = cluster.partition_tokens(META[name]["tokens"], n)
    tag = f"{name}_n{n}_{cls_mode}"
    res = cluster.run_inference(params, plan, inputs, "classify", cls_mode=cls_mode)
    want = GOLD[f"{tag}_output"]
    err = np.abs(res.output - want).max()
    assert err <= 1e-4, err                       # parity-mode tolerance (logits, absolute)
    assert int(res.output.argmax()) == int(want.argmax())
    assert res.ledger.to_csv() == META[f"{tag}_ledger"]
    # VQ indices of every device at every layer are bit-identical to the reference's
    rt = AstraRuntime(params, plan, batch=1, cls_mode=cls_mode, precision="parity")
    rt.trace = []
    rt.classify_numpy(np.asarray(inputs, np.float32)[None])
    got = np.concatenate([t.cpu().numpy().reshape(-1) for t in rt.trace])
    np.testing.assert_array_equal(got, GOLD[f"{tag}_indices"])


@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("precision", ["parity", "fast"])
def test_generate_matches_reference(cuda, n, precision):
    """Causal SP prefill + greedy decode on device N-1 (cluster.py:243-308): same tokens."""
    from paper_2505_19342_b200 import cluster
    params, op, inputs = _setup("gen")
    m = META["gen"]
    plan = cluster.partition_tokens(m["tokens"], n, class_replication=False)
    res = cluster.run_inference(params, plan, inputs, "generate", steps=m["steps"],
                                precision=precision)
    tag = f"gen_n{n}"
    assert res.output == [int(t) for t in GOLD[f"{tag}_output"]]
    assert res.ledger.to_csv() == META[f"{tag}_ledger"]
    assert cluster.run_inference(params, plan, inputs, "generate", steps=0).output == []


def test_generate_gpt2_width_vs_oracle(cuda):
    """GPT-2 block width (D=768, H=12) causal prefill over 4 devices + 5 decode steps."""
    from paper_2505_19342_b200 import cluster, model, vq
    kw = dict(layers=2, hidden=768, heads=12, vocab_or_classes=300, max_tokens=80, causal=True,
              codebook_size=64)
    params = model.init_params(model.ModelConfig(**kw), seed=5)
    op = O.init_params(O.Config(**kw), seed=5)
    rng = np.random.default_rng(5)
    data = [rng.integers(0, 300, size=65) for _ in range(4)]
    O.initialize_codebooks(op, data, "lm", seed=5, iterations=4)
    for i, b in enumerate(params.blocks):
        b.codebook = vq.Codebook(layer_id=i, groups=1, centroids=op.codebooks[i])
    ids = rng.integers(0, 300, size=64)
    ranges = O.partition_tokens(64, 4)
    ref = O.run_inference(op, ranges, ids, "generate", steps=5)
    plan = cluster.partition_tokens(64, 4, class_replication=False)
    got = cluster.run_inference(params, plan, ids, "generate", steps=5)
    assert got.output == ref.output


@pytest.mark.parametrize("n", [1, 4])
def test_classify_fast_mode_tolerance(cuda, n):
    from paper_2505_19342_b200 import cluster
    params, op, inputs = _setup("vitb2")
    plan = cluster.partition_tokens(196, n)
    res = cluster.run_inference(params, plan, inputs, "classify", precision="fast")
    want = GOLD[f"vitb2_n{n}_distributed_output"]
    assert np.abs(res.output - want).max() <= 3e-2      # bf16 tolerance (SURVEY 8a')
    assert int(res.output.argmax()) == int(want.argmax())


def test_batch_equals_single_image(cuda):
    """Per-image results do not depend on the batch they ride in (bitwise)."""
    from paper_2505_19342_b200 import cluster
    from paper_2505_19342_b200.runtime import AstraRuntime
    params, op, _ = _setup("vitb2")
    xs = np.stack(O.make_classify_data(768, 196, 3, seed=7, task_seed=0)[0])
    plan = cluster.partition_tokens(196, 4)
    rt3 = AstraRuntime(params, plan, batch=3, precision="parity")
    out3 = rt3.classify_numpy(xs)
    rt1 = AstraRuntime(params, plan, batch=1, precision="parity")
    for b in range(3):
        np.testing.assert_array_equal(rt1.classify_numpy(xs[b:b + 1]), out3[b:b + 1])
    # and they match the oracle at fp32 tolerance
    ranges = O.partition_tokens(196, 4)
    for b in range(3):
        ref = O.run_inference(op, ranges, xs[b]).output
        assert np.abs(out3[b:b + 1] - ref).max() <= 1e-4


def test_cuda_graph_replay_matches_eager(cuda):
    from paper_2505_19342_b200 import cluster
    from paper_2505_19342_b200.runtime import AstraRuntime
    params, op, _ = _setup("vitb2")
    xs = np.stack(O.make_classify_data(768, 196, 2, seed=9, task_seed=0)[0])
    plan = cluster.partition_tokens(196, 2)
    rt = AstraRuntime(params, plan, batch=2, precision="fast")
    eager = rt.classify_numpy(xs)
    rt.capture()
    rt.stage_input(xs)
    rt.graph.replay()
    np.testing.assert_array_equal(rt.logits.cpu().numpy(), eager)


@pytest.mark.parametrize("precision,tol", [("parity", 1e-4), ("fast", 3e-2)])
def test_grouped_remote_rows_fused_decode_vs_oracle(cuda, precision, tol):
    """G = 16 codebooks at ViT-B width, N = 4: the received rows go through the fused decode+LN1
    kernel and the K|V GEMM; logits match the oracle's run_inference on the same codebooks."""
    from paper_2505_19342_b200 import cluster, model, vq
    from paper_2505_19342_b200.runtime import AstraRuntime
    cfg = model.ModelConfig(layers=2, hidden=768, heads=12, vocab_or_classes=10, max_tokens=65,
                            causal=False, codebook_size=64, groups=16)
    params = model.init_params(cfg, seed=2)
    ocfg = O.Config(layers=2, hidden=768, heads=12, vocab_or_classes=10, max_tokens=65,
                    causal=False, codebook_size=64, groups=16)
    op = O.init_params(ocfg, seed=2)
    xs, _ = O.make_classify_data(768, 64, 3, seed=5, task_seed=0)
    O.initialize_codebooks(op, xs[:2], "classify", seed=0, iterations=4)
    for i, b in enumerate(params.blocks):
        b.codebook = vq.Codebook(layer_id=i, groups=16, centroids=op.codebooks[i])
    plan = cluster.partition_tokens(64, 4)
    rt = AstraRuntime(params, plan, batch=1, precision=precision)
    assert rt.fused_decode
    x = xs[2]
    got = np.asarray(rt.classify_numpy(x[None])).reshape(-1)
    want = np.asarray(O.run_inference(op, O.partition_tokens(64, 4), x).output).reshape(-1)
    err = np.abs(got - want).max()
    assert err <= tol, err
    assert int(np.argmax(got)) == int(np.argmax(want))
