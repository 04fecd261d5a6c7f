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


def _run(params, xs, n, precision, capture=False):
    from paper_2505_19342_b200.cluster import partition_tokens
    from paper_2505_19342_b200.runtime import AstraRuntime
    rt = AstraRuntime(params, partition_tokens(T, n), batch=len(xs), precision=precision)
    rt.trace = []
    if capture:
        rt.capture_inputs = []
    logits = rt.classify_numpy(xs)
    codes = np.stack([rt.codes_by_image(t)[:, :, 0] for t in rt.trace], axis=1)  # [B, L, T]
    xin = [rt.codes_by_image(x, D) for x in rt.capture_inputs] if capture else None
    return logits, codes.reshape(len(xs), L * T), xin


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_parity_mode_indices_logits_vs_reference(cuda, headline, n):
    """Every index equal except documented near-ties.  The VQ encode is exact for its input;
    the fp32-class (bf16x3) forward lands within ~1e-6 of the reference's fp64-accumulate
    forward, so a token whose two best codes are closer than that can flip (gaps down to 5e-9
    of |x|^2 occur — below fp32 resolution, unresolvable by any fp32 forward).  At N > 1 a
    flipped code changes the other devices' dequantized K/V of that token, so it can cascade
    within that image.  Checked:
      * at most 1e-4 of all codes differ, and the EARLIEST mismatch of each affected image is a
        tie: on the GPU's own layer input our code is the fp64 argmin and the reference's code
        scores within 4e-6 * |x|^2 of it (the bf16x3 operand split is exact to 2^-17);
      * images without any flipped code: logits within 1e-4 (SURVEY 8a' parity tolerance);
      * every image: top-1 identical, logits within the bf16-class 3e-2."""
    params, xs, gold, _ = headline
    logits, codes, xin = _run(params, xs, n, "parity", capture=True)
    want_logits, want_idx = gold[f"n{n}_logits"], gold[f"n{n}_indices"]
    bad = np.argwhere(codes != want_idx)
    assert len(bad) <= codes.size // 10000, len(bad)
    first = {}
    for b, j in bad:
        first.setdefault(int(b), int(j))      # argwhere is row-major: earliest layer first
    gaps = []
    for b, j in first.items():
        l, t = divmod(j, T)
        x = xin[l][b, t].astype(np.float64)
        c = np.asarray(params.blocks[l].codebook.centroids[0], np.float64)
        d_ours = ((x - c[codes[b, j]]) ** 2).sum()
        d_ref = ((x - c[want_idx[b, j]]) ** 2).sum()
        assert d_ours <= d_ref
        gaps.append((d_ref - d_ours) / (x @ x))
    clean = np.setdiff1d(np.arange(len(xs)), list(first))
    err_clean = np.abs(logits[clean] - want_logits[clean]).max()
    err_all = np.abs(logits - want_logits).max()
    print(f"N={n} parity: {len(bad)} / {codes.size} code mismatches in {len(first)} image(s), "
          f"first-mismatch gaps {['%.1e' % g for g in gaps]}; max|dlogit| clean images "
          f"{err_clean:.2e}, all {err_all:.2e}")
    assert all(g <= 4e-6 for g in gaps), gaps
    assert err_clean <= 1e-4, err_clean
    assert err_all <= 3e-2, err_all
    np.testing.assert_array_equal(logits.argmax(1), want_logits.argmax(1))


def test_parity_mode_two_layer_fixtures_bitwise(cuda, headline):
    """The first two layers of the headline config are bitwise (no drift yet to flip a tie)."""
    params, xs, gold, _ = headline
    _, codes, _ = _run(params, xs[:16], 4, "parity")
    np.testing.assert_array_equal(codes[:, :2 * T], gold["n4_indices"][:16, :2 * T])


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_fast_mode_tolerance_top1_and_index_agreement(cuda, headline, n):
    params, xs, gold, _ = headline
    logits, codes, _ = _run(params, xs, n, "fast")
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
