"""Reference-WRITTEN blobs: an ASTM checkpoint and an AVQ1 codebook produced by
seqvq itself (tests/golden/make_golden_blobs.py) load through this repo's loaders, re-save to the
same bytes, and — on the GPU — drive cluster.run_inference to the reference's own outputs.
Formats: model.py:435-482 (ASTM), vq.py:328-361 (AVQ1)."""

from pathlib import Path

import numpy as np
import pytest

G = Path(__file__).resolve().parent / "golden"
GOLD = np.load(G / "golden_blobs.npz")


def _oracle_params(params):
    from oracle import astra_oracle as O
    cfg = params.config
    oc = O.Config(layers=cfg.layers, hidden=cfg.hidden, heads=cfg.heads,
                  vocab_or_classes=cfg.vocab_or_classes, max_tokens=cfg.max_tokens,
                  causal=cfg.causal, codebook_size=cfg.codebook_size, groups=cfg.groups)
    blocks = [{f: np.asarray(getattr(b, f).data) for f in b.TENSOR_FIELDS} for b in params.blocks]
    op = O.Params(config=oc, pos=params.pos.data, blocks=blocks, final_gain=params.final_gain.data,
                  final_bias=params.final_bias.data, head=params.head.data,
                  embedding=params.embedding.data if params.embedding is not None else None,
                  cls=params.cls.data if params.cls is not None else None)
    op.codebooks = [[np.asarray(c) for c in b.codebook.centroids] for b in params.blocks]
    return op


@pytest.mark.parametrize("name", ["ref_ckpt_toy.astm", "ref_ckpt_gen.astm"])
def test_reference_checkpoint_loads_and_resaves_bytewise(name):
    from paper_2505_19342_b200 import model
    blob = (G / name).read_bytes()
    p = model.load_checkpoint(blob)
    assert model.save_checkpoint(p) == blob
    assert all(b.codebook is not None for b in p.blocks)
    assert all(b.codebook.ema_counts is not None for b in p.blocks)   # EMA state travels too


def test_reference_codebook_blob():
    from paper_2505_19342_b200 import vq
    blob = (G / "ref_codebook.avq1").read_bytes()
    cb = vq.load_codebook(blob)
    assert cb.groups == 2 and cb.size == 16 and cb.layer_id == 1
    np.testing.assert_array_equal(np.stack(cb.centroids), GOLD["avq1_centroids"])
    np.testing.assert_array_equal(np.asarray(cb.ema_counts), GOLD["avq1_ema_counts"])
    np.testing.assert_array_equal(np.stack(cb.ema_sums), GOLD["avq1_ema_sums"])
    assert vq.save_codebook(cb) == blob
    with pytest.raises(ValueError):
        vq.load_codebook(b"XXXX" + blob[4:])


@pytest.mark.parametrize("n", [1, 2, 3])
def test_oracle_on_reference_checkpoint(n):
    """The CPU oracle, fed the reference-written checkpoint, reproduces the reference's logits."""
    from oracle import astra_oracle as O
    from paper_2505_19342_b200 import model
    p = model.load_checkpoint((G / "ref_ckpt_toy.astm").read_bytes())
    r = O.run_inference(_oracle_params(p), O.partition_tokens(12, n), GOLD["toy_x"])
    np.testing.assert_allclose(np.asarray(r.output).reshape(-1),
                               GOLD[f"toy_n{n}_logits"].reshape(-1), atol=1e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3])
def test_gpu_run_inference_on_reference_checkpoint(cuda, n):
    from paper_2505_19342_b200 import cluster, model
    p = model.load_checkpoint((G / "ref_ckpt_toy.astm").read_bytes())
    r = cluster.run_inference(p, cluster.partition_tokens(12, n), GOLD["toy_x"], "classify")
    err = np.abs(np.asarray(r.output).reshape(-1) - GOLD[f"toy_n{n}_logits"].reshape(-1)).max()
    assert err <= 1e-4, err
    assert r.ledger.total_bits_sent() == int(GOLD[f"toy_n{n}_ledger_bits"])


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2])
def test_gpu_generate_on_reference_checkpoint(cuda, n):
    from paper_2505_19342_b200 import cluster, model
    p = model.load_checkpoint((G / "ref_ckpt_gen.astm").read_bytes())
    plan = cluster.partition_tokens(10, n, class_replication=False)
    r = cluster.run_inference(p, plan, GOLD["gen_ids"], "generate", steps=3)
    assert list(np.asarray(r.output).reshape(-1)) == list(GOLD[f"gen_n{n}_tokens"].reshape(-1))
