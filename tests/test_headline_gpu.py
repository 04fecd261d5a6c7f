"""Parity at the headline configuration (BASELINE configs #1/#2): ViT-B/16 shape, 12 layers,
K=1024, G=1, the reference's own k-means codebooks, 64 synthetic images, N = 1/2/4/8.

The expected values are the reference's outputs (tests/golden/make_golden_vitb.py runs
seqvq.cluster.run_inference on the same weights, codebooks and images).

* parity mode (fp32-class): every VQ index of every layer and device bit-identical, logits
  within 1e-4 (SURVEY 8a' suggested tolerance), top-1 identical;
* fast mode (bf16 operands, fp32 accumulation): logits within 3e-2, top-1 agreement and
  per-layer index agreement reported and bounded below.
"""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
L, D, H, T, K, B = 12, 768, 12, 196, 1024, 64


@pytest.fixture(scope="module")
def headline():
    from paper_2505_19342_b200 import codebooks, data, model
    cfg = model.ModelConfig(layers=L, hidden=D, heads=H, vocab_or_classes=1000, max_tokens=197,
                            causal=False, codebook_size=K, groups=1)
    params = model.init_params(cfg, seed=0)
    codebooks.load_codebook_tables(G / "vitb16_codebooks.npz", params)
    xs = data.make_classify_batch(D, T, B, seed=1, task_seed=0)
    gold = np.load(G / "golden_vitb.npz")
    meta = json.loads((G / "golden_vitb_meta.json").read_text())
    return params, xs, gold, meta


def _run(params, xs, n, precision):
    from paper_2505_19342_b200.cluster import partition_tokens
    from paper_2505_19342_b200.runtime import AstraRuntime
    rt = AstraRuntime(params, partition_tokens(T, n), batch=len(xs), precision=precision)
    rt.trace = []
    logits = rt.classify_numpy(xs)
    codes = np.stack([rt.codes_by_image(t)[:, :, 0] for t in rt.trace], axis=1)  # [B, L, T]
    return logits, codes.reshape(len(xs), L * T)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_parity_mode_bitwise_indices_all_layers(cuda, headline, n):
    params, xs, gold, _ = headline
    logits, codes = _run(params, xs, n, "parity")
    want_logits, want_idx = gold[f"n{n}_logits"], gold[f"n{n}_indices"]
    np.testing.assert_array_equal(codes, want_idx)           # 64 images x 12 layers x 196
    err = np.abs(logits - want_logits).max()
    assert err <= 1e-4, err
    np.testing.assert_array_equal(logits.argmax(1), want_logits.argmax(1))


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_fast_mode_tolerance_top1_and_index_agreement(cuda, headline, n):
    params, xs, gold, _ = headline
    logits, codes = _run(params, xs, n, "fast")
    want_logits, want_idx = gold[f"n{n}_logits"], gold[f"n{n}_indices"]
    err = np.abs(logits - want_logits).max()
    top1 = (logits.argmax(1) == want_logits.argmax(1)).mean()
    per_layer = (codes.reshape(B, L, T) == want_idx.reshape(B, L, T)).mean(axis=(0, 2))
    print(f"N={n} fast: max|dlogit| {err:.3e}, top-1 {top1:.4f}, "
          f"min layer index agreement {per_layer.min():.5f}")
    assert err <= 3e-2, err                      # bf16 tolerance (SURVEY 8a')
    assert top1 >= 0.98, top1
    assert per_layer[0] == 1.0                   # layer 0 sees identical inputs
    assert per_layer.min() >= 0.99, per_layer


def test_config1_cli_equivalent_run(cuda, headline):
    """BASELINE config #1: `seqvq infer` with the ViT-B overrides (cli.py:108-157) —
    predicted=392, ledger 23,520 bits — through the drop-in run_inference."""
    from paper_2505_19342_b200 import cluster
    params, xs, gold, meta = headline
    plan = cluster.partition_tokens(T, 4)
    res = cluster.run_inference(params, plan, xs[0], "classify", workers=2)
    assert int(np.argmax(res.output)) == meta["config1_predicted"] == 392
    assert res.ledger.to_csv() == meta["n4_ledger"]
    assert res.ledger.total_bits_sent() == 23520
    assert np.abs(res.output - gold["n4_logits"][:1]).max() <= 1e-4
