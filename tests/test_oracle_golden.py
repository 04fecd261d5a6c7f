"""Pin the CPU oracle (oracle/astra_oracle.py) to golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import astra_oracle as O
from tests.golden.cases import ATT_CASES, VQ_CASES, att_case_inputs, vq_case_inputs

G = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def gvq():
    return np.load(G / "golden_vq.npz")


@pytest.fixture(scope="module")
def gatt():
    return np.load(G / "golden_attention.npz")


@pytest.fixture(scope="module")
def ginf():
    return np.load(G / "golden_infer.npz"), json.loads((G / "golden_infer_meta.json").read_text())


def test_index_bits_table():
    # test_vq.py:38-43
    assert [O.index_bits(k) for k in (1, 2, 3, 16, 1024)] == [0, 1, 2, 4, 10]


@pytest.mark.parametrize("i", range(len(VQ_CASES)))
def test_oracle_quantize_matches_reference(gvq, i):
    k, d, g, m = VQ_CASES[i]
    if i == len(VQ_CASES) - 1:
        cents = [np.array([[1.0, 0.0], [-1.0, 0.0]], np.float32)]
        x = np.zeros((m, d), np.float32)
    else:
        cents, x = vq_case_inputs(i, k, d, g, m)
    idx = O.quantize(cents, x)
    np.testing.assert_array_equal(idx, gvq[f"c{i}_idx"])
    xhat = O.dequantize(cents, idx)
    assert hashlib.sha256(np.ascontiguousarray(xhat).tobytes()).digest() == \
        gvq[f"c{i}_xhat_sha256"].tobytes()


@pytest.mark.parametrize("i", range(len(ATT_CASES)))
def test_oracle_attention_matches_reference(gatt, i):
    r, c, d, h, p = ATT_CASES[i]
    q, k, v, mask = att_case_inputs(i, r, c, d, p)
    out = O.multihead_attention(q, k, v, mask, h)
    ref = gatt[f"c{i}_out"]
    np.testing.assert_allclose(out, ref, atol=1e-6)   # test_attention.py:50 tolerance
    assert np.array_equal(out, ref)                   # and in fact bitwise on this host


def _oracle_setup(meta, name):
    m = meta[name]
    mk = dict(m["model"])
    cfg = O.Config(**mk)
    params = O.init_params(cfg, seed=m["seed"])
    t, seed = m["tokens"], m["seed"]
    if cfg.causal:
        data = O.make_lm_data(cfg.vocab_or_classes, t, 8, seed=seed, task_seed=seed)
        O.initialize_codebooks(params, data, "lm", seed=seed)
        inputs = O.make_lm_data(cfg.vocab_or_classes, t, 1, seed=seed + 1, task_seed=seed)[0][:t]
    else:
        xs, _ = O.make_classify_data(cfg.hidden, t, 8, seed=seed, task_seed=seed)
        O.initialize_codebooks(params, xs, "classify", seed=seed)
        inputs = O.make_classify_data(cfg.hidden, t, 1, seed=seed + 1, task_seed=seed)[0][0]
    return params, inputs


def _digest(params):
    h = hashlib.sha256()
    for books in params.codebooks:
        for c in books:
            h.update(np.ascontiguousarray(c, "<f4").tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["toy", "toyg2", "gen", "vitb2"])
def test_oracle_inference_matches_reference(ginf, name):
    arrs, meta = ginf
    params, inputs = _oracle_setup(meta, name)
    # weights, synthetic data and k-means codebooks reproduce the reference bit for bit
    assert _digest(params) == meta[name]["codebook_sha256"]
    if f"{name}_inputs" in arrs:
        np.testing.assert_array_equal(np.asarray(inputs), arrs[f"{name}_inputs"])
    m = meta[name]
    modes = ["distributed", "single"] if name == "toy" else ([None] if m["mode"] == "generate"
                                                             else ["distributed"])
    for n in m["devices"]:
        ranges = O.partition_tokens(m["tokens"], n)
        for cm in modes:
            tag = f"{name}_n{n}" + (f"_{cm}" if cm else "")
            res = O.run_inference(params, ranges, inputs, m["mode"], steps=m["steps"],
                                  cls_mode=cm or "distributed")
            got = np.asarray(res.output)
            want = arrs[f"{tag}_output"]
            if m["mode"] == "generate":
                np.testing.assert_array_equal(got, want)
            else:
                np.testing.assert_allclose(got, want, atol=1e-5, rtol=0)  # test_cluster.py:194
                assert np.array_equal(got, want)                         # bitwise on this host
            idx = np.concatenate([i.reshape(-1) for layer in res.indices for i in layer])
            np.testing.assert_array_equal(idx, arrs[f"{tag}_indices"])
            assert res.ledger.to_csv() == meta[f"{tag}_ledger"]


def test_partition_remainder_trailing():
    # test_cluster.py:44-50
    assert O.partition_tokens(10, 4) == ((0, 2), (2, 4), (4, 7), (7, 10))
    assert [e - s for s, e in O.partition_tokens(196, 8)] == [24] * 4 + [25] * 4


def test_pack_indices_lsb_first():
    idx = np.array([1, 2, 1023, 0, 512], dtype=np.int32)
    words = O.pack_indices(idx, 10)
    bits = 0
    for i, w in enumerate(words):
        bits |= int(w) << (32 * i)
    for i, v in enumerate(idx):
        assert (bits >> (10 * i)) & 1023 == v
