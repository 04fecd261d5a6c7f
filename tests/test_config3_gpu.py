"""BASELINE config #3 parity: GPT-2-small (L=12, D=768, H=12, vocab 50,257) causal prefill of
T=1024 tokens + greedy decode, K=1024 codebooks fitted by the reference, against the
reference's own run_inference(..., "generate", steps=4) at N=1 and N=4
(tests/golden/make_golden_gpt2s.py).

* parity mode: the 4 generated tokens identical; at most 1e-4 of the prefill VQ codes differ and
  the first differing code of a sequence is a near-tie (our code is the fp64 argmin on our layer
  input, the reference's within 1e-5 |x|^2 of it);
* fast mode: the first token identical, per-layer index agreement >= 0.98.
"""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def config3():
    from paper_2505_19342_b200 import codebooks, model
    meta = json.loads((GD / "golden_gpt2s_meta.json").read_text())
    cfg = model.ModelConfig(layers=meta["L"], hidden=meta["D"], heads=meta["H"],
                            vocab_or_classes=meta["V"], max_tokens=meta["T"] + meta["steps"],
                            causal=True, codebook_size=meta["K"], groups=meta["G"])
    params = model.init_params(cfg, seed=0)
    codebooks.load_codebook_tables(GD / "gpt2s_codebooks.npz", params)
    gold = np.load(GD / "golden_gpt2s.npz")
    prompts = gold["prompts"].astype(np.int64)
    want = model.generator(1, "gpt2-ids").integers(0, meta["V"], size=prompts.shape)
    np.testing.assert_array_equal(prompts, want)      # same named stream as the reference
    return params, prompts, gold, meta


def _run(params, prompts, meta, n, precision):
    from paper_2505_19342_b200.cluster import partition_tokens
    from paper_2505_19342_b200.runtime import AstraRuntime
    plan = partition_tokens(meta["T"], n, class_replication=False)
    rt = AstraRuntime(params, plan, batch=len(prompts), mode="generate", precision=precision)
    rt.trace, rt.capture_inputs = [], []
    toks = np.asarray(rt.generate(prompts, meta["steps"]))
    codes = np.stack([rt.codes_by_image(t) for t in rt.trace[:meta["L"]]], axis=1)
    xin = [rt.codes_by_image(x, meta["D"]) for x in rt.capture_inputs[:meta["L"]]]
    return toks, codes.reshape(len(prompts), -1), xin


@pytest.mark.parametrize("n", [1, 4])
def test_config3_parity_mode(cuda, config3, n):
    params, prompts, gold, meta = config3
    T, G, D = meta["T"], meta["G"], meta["D"]
    toks, codes, xin = _run(params, prompts, meta, n, "parity")
    want = gold[f"n{n}_indices"].astype(np.int64)
    np.testing.assert_array_equal(toks, gold[f"n{n}_tokens"])
    bad = np.argwhere(codes != want)
    # (at N > 1 a flipped code changes the other devices' dequantized K/V of that token, so a
    # near-tie can cascade into a few later codes of the same sequence)
    assert len(bad) <= max(8, codes.size // 10000), len(bad)
    first = {}
    for b, j in bad:
        first.setdefault(int(b), int(j))
    gaps = []
    for b, j in first.items():
        l, rem = divmod(j, T * G)
        t, g = divmod(rem, G)
        gd = D // G
        x = xin[l][b, t, g * gd:(g + 1) * gd].astype(np.float64)
        c = np.asarray(params.blocks[l].codebook.centroids[g], np.float64)
        d_ours = ((x - c[codes[b, j]]) ** 2).sum()
        d_ref = ((x - c[want[b, j]]) ** 2).sum()
        assert d_ours <= d_ref
        gaps.append((d_ref - d_ours) / (x @ x))
    print(f"N={n} parity: tokens {toks.tolist()}, {len(bad)} / {codes.size} code mismatches, "
          f"first-mismatch gaps {['%.1e' % v for v in gaps]}")
    assert all(v <= 1e-5 for v in gaps), gaps


@pytest.mark.parametrize("n", [1, 4])
def test_config3_fast_mode(cuda, config3, n):
    params, prompts, gold, meta = config3
    L, T, G = meta["L"], meta["T"], meta["G"]
    toks, codes, _ = _run(params, prompts, meta, n, "fast")
    want = gold[f"n{n}_indices"]
    per_layer = (codes.reshape(len(prompts), L, -1) == want.reshape(len(prompts), L, -1)).mean(axis=(0, 2))
    print(f"N={n} fast: tokens {toks.tolist()} vs {gold[f'n{n}_tokens'].tolist()}, "
          f"min layer index agreement {per_layer.min():.5f}")
    np.testing.assert_array_equal(toks[:, 0], gold[f"n{n}_tokens"][:, 0])
    assert per_layer[0] == 1.0
    assert per_layer.min() >= 0.98, per_layer
