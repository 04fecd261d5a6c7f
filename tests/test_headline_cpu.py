"""CPU pins of the headline-config fixtures (no GPU): the committed codebooks are the
reference's own k-means output, and the oracle reproduces the reference's 12-layer ViT-B/16
forward on them (tests/golden/make_golden_vitb.py produced both by running seqvq)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import astra_oracle as O

G = Path(__file__).resolve().parent / "golden"
L, D, H, T, K = 12, 768, 12, 196, 1024
META = json.loads((G / "golden_vitb_meta.json").read_text())


def _oracle_params():
    cfg = O.Config(layers=L, hidden=D, heads=H, vocab_or_classes=1000, max_tokens=197,
                   causal=False, codebook_size=K, groups=1)
    return O.init_params(cfg, seed=0)


def test_codebook_archive_is_the_reference_output():
    from paper_2505_19342_b200 import codebooks
    books = codebooks.load_codebook_tables(G / "vitb16_codebooks.npz")   # checks its own sha256
    cents = np.stack([np.stack(b.centroids) for b in books]).astype(np.float32)
    assert hashlib.sha256(cents.tobytes()).hexdigest() == META["centroids_sha256"]
    assert cents.shape == (L, 1, K, D)


def test_oracle_reproduces_reference_vitb_forward():
    """Config #1 (N=4, image 0) and N=8 (image 1): logits and every layer's indices."""
    from paper_2505_19342_b200 import codebooks, data
    op = _oracle_params()
    op.codebooks = [[np.asarray(c) for c in b.centroids]
                    for b in codebooks.load_codebook_tables(G / "vitb16_codebooks.npz")]
    xs = data.make_classify_batch(D, T, 2, seed=1, task_seed=0)
    gold = np.load(G / "golden_vitb.npz")
    for n, b in ((4, 0), (8, 1)):
        r = O.run_inference(op, O.partition_tokens(T, n), xs[b])
        np.testing.assert_allclose(r.output.reshape(-1), gold[f"n{n}_logits"][b], atol=1e-6)
        got = np.concatenate([np.concatenate([i.reshape(-1) for i in layer]) for layer in r.indices])
        np.testing.assert_array_equal(got, gold[f"n{n}_indices"][b])
    assert int(np.argmax(gold["n4_logits"][0])) == META["config1_predicted"] == 392


@pytest.mark.slow
def test_oracle_kmeans_reproduces_reference_codebooks():
    """The oracle's initialize_codebooks (train.py:176-189) on the recipe's 8 images gives the
    reference's centroids bit for bit (same host BLAS)."""
    op = _oracle_params()
    fit, _ = O.make_classify_data(D, T, 8, seed=0, task_seed=0)
    O.initialize_codebooks(op, fit, "classify", seed=0)
    cents = np.stack([np.stack(c) for c in op.codebooks]).astype(np.float32)
    assert hashlib.sha256(cents.tobytes()).hexdigest() == META["centroids_sha256"]
