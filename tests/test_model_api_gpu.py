"""Model-level drop-in API (seqvq model.py:198-432) on the GPU runtime: run_blocks, classify,
lm_logits, generate, prefill_decode_state / DecodeState, aggregate_class_tokens, the embed
helpers and exact_codebooks_from_reference — against the reference's own outputs
(tests/golden/golden_model.npz from make_golden.py) and ports of the reference's tests
(test_model.py:100-275, test_cluster.py:187-226, acceptance criterion 3)."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = np.load(Path(__file__).resolve().parent / "golden" / "golden_model.npz")
RNG = np.random.default_rng(20)


def _attach(params, books):
    from paper_2505_19342_b200 import vq
    for i, b in enumerate(params.blocks):
        b.codebook = vq.Codebook(layer_id=i, groups=books.shape[1],
                                 centroids=[np.ascontiguousarray(c) for c in books[i]])
    return params


def _enc():
    from paper_2505_19342_b200 import model
    p = model.init_params(model.ModelConfig(layers=2, hidden=32, heads=4, vocab_or_classes=4,
                                            codebook_size=8, max_tokens=512, causal=False), seed=0)
    return _attach(p, GOLD["enc_codebooks"])


def _dec():
    from paper_2505_19342_b200 import model
    p = model.init_params(model.ModelConfig(layers=2, hidden=32, heads=4, vocab_or_classes=16,
                                            codebook_size=8, max_tokens=17, causal=True), seed=0)
    return _attach(p, GOLD["dec_codebooks"])


@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("cls_mode", ["distributed", "single"])
def test_classify_matches_reference(cuda, n, cls_mode):
    from paper_2505_19342_b200 import model
    from paper_2505_19342_b200.cluster import partition_tokens
    got = model.classify(_enc(), partition_tokens(16, n), GOLD["enc_x"], cls_mode=cls_mode)
    np.testing.assert_allclose(got.data, GOLD[f"enc_classify_n{n}_{cls_mode}"], atol=1e-5)


def test_run_blocks_and_on_layer_info_match_reference(cuda):
    from paper_2505_19342_b200 import model
    from paper_2505_19342_b200.cluster import partition_tokens
    params = _enc()
    x0 = model.embed_classifier_inputs(params, GOLD["enc_x"])
    np.testing.assert_array_equal(x0.data, GOLD["enc_embed"])
    infos = []
    content, reps = model.run_blocks(params, partition_tokens(16, 4), x0,
                                     on_layer=lambda i, info: infos.append((i, info)))
    np.testing.assert_allclose(content.data, GOLD["enc_blocks_content"], atol=1e-5)
    np.testing.assert_allclose(reps.data, GOLD["enc_blocks_replicas"], atol=1e-5)
    assert [i for i, _ in infos] == [0, 1]
    for i, info in infos:
        np.testing.assert_array_equal(info["q"].indices, GOLD[f"enc_info{i}_q"])
        np.testing.assert_array_equal(info["x_hat"], GOLD[f"enc_info{i}_x_hat"])
        for k in ("x_in", "k_full", "v_full", "k_hat", "v_hat"):
            np.testing.assert_allclose(info[k], GOLD[f"enc_info{i}_{k}"], atol=1e-5, err_msg=k)
    agg = model.aggregate_class_tokens(reps)
    np.testing.assert_allclose(agg.data, GOLD["enc_aggregate"], atol=1e-6)


def test_exact_codebooks_match_reference_capture(cuda):
    from paper_2505_19342_b200 import model
    from paper_2505_19342_b200.cluster import partition_tokens
    books = model.exact_codebooks_from_reference(_enc(), partition_tokens(16, 1), GOLD["enc_x"])
    got = np.stack([np.stack(b.centroids) for b in books])
    np.testing.assert_allclose(got, GOLD["enc_exact_books"], atol=1e-5)
    with pytest.raises(ValueError):
        model.exact_codebooks_from_reference(_enc(), partition_tokens(16, 2), GOLD["enc_x"])


@pytest.mark.parametrize("n", [1, 2, 4])
def test_lm_logits_generate_prefill_match_reference(cuda, n):
    from paper_2505_19342_b200 import model
    from paper_2505_19342_b200.cluster import partition_tokens
    params, ids = _dec(), GOLD["dec_ids"]
    plan = partition_tokens(8, n, class_replication=False)
    np.testing.assert_array_equal(model.embed_lm_inputs(params, ids, offset=3).data,
                                  GOLD["dec_embed"])
    lg = model.lm_logits(params, plan, ids)
    np.testing.assert_allclose(lg.data, GOLD[f"dec_lm_logits_n{n}"], atol=1e-5)
    assert model.generate(params, plan, ids, 6) == GOLD[f"dec_generate_n{n}"].tolist()
    st, first = model.prefill_decode_state(params, plan, ids)
    assert first == int(GOLD[f"dec_prefill_first_n{n}"][0])
    for i in range(len(st.k)):
        np.testing.assert_allclose(st.k[i], GOLD[f"dec_prefill_n{n}_k{i}"], atol=1e-5)
        np.testing.assert_allclose(st.v[i], GOLD[f"dec_prefill_n{n}_v{i}"], atol=1e-5)
    st.append(0, st.k[0][:1], st.v[0][:1])
    assert st.k[0].shape[0] == 9


def test_acceptance_criterion_03_identity_quantization(cuda):
    """test_acceptance.py:114-150 over the same 100 random configs (hidden 4..16, heads 1..2,
    G 1..2, N 1/2/4, encoder and causal): with exact codebooks the N-device output equals the
    single-device output within 1e-5; both also match the reference's own numbers."""
    from paper_2505_19342_b200 import cluster, model
    worst = worst_ref = 0.0
    for trial in range(100):
        causal, layers, heads, hidden, groups, devices, tokens, vocab = \
            (int(v) for v in GOLD[f"c3_{trial}_cfg"])
        cfg = model.ModelConfig(layers=layers, hidden=hidden, heads=heads, vocab_or_classes=vocab,
                                max_tokens=tokens + 1, causal=bool(causal), codebook_size=4,
                                groups=groups)
        params = model.init_params(cfg, seed=trial)
        plan1 = cluster.partition_tokens(tokens, 1)
        plan_n = cluster.partition_tokens(tokens, devices, class_replication=not causal)
        inputs = GOLD[f"c3_{trial}_inputs"]
        if causal:
            reference = model.lm_logits(params, plan1, inputs).data
        else:
            reference = model.classify(params, plan1, inputs).data
        books = model.exact_codebooks_from_reference(params, plan1, inputs)
        for b, cb in zip(params.blocks, books):
            b.codebook = cb
        if causal:
            got = model.lm_logits(params, plan_n, inputs).data
        else:
            got = cluster.run_inference(params, plan_n, inputs, mode="classify").output
        worst = max(worst, float(np.abs(got - reference).max()))
        worst_ref = max(worst_ref, float(np.abs(reference - GOLD[f"c3_{trial}_reference"]).max()),
                        float(np.abs(got - GOLD[f"c3_{trial}_got"]).max()))
    assert worst < 1e-5, worst
    assert worst_ref < 1e-5, worst_ref


def test_causality_future_tokens_do_not_affect_past_logits(cuda):
    from paper_2505_19342_b200 import model
    from paper_2505_19342_b200.cluster import partition_tokens
    params = _dec()
    for b in params.blocks:
        b.codebook = None
    plan = partition_tokens(6, 1)
    a = model.lm_logits(params, plan, [0, 1, 2, 3, 4, 0]).data
    b = model.lm_logits(params, plan, [0, 1, 2, 4, 3, 1]).data
    np.testing.assert_array_equal(a[:3], b[:3])
    assert np.abs(a[3:] - b[3:]).max() > 0


def test_generate_matches_sequential_full_forward(cuda):
    from paper_2505_19342_b200 import model
    from paper_2505_19342_b200.cluster import partition_tokens
    params = model.init_params(model.ModelConfig(layers=2, hidden=8, heads=2, vocab_or_classes=6,
                                                 max_tokens=16, causal=True), seed=0)
    prompt = [0, 3, 1, 5, 2]
    got = model.generate(params, partition_tokens(5, 1), prompt, steps=4)
    ids, want = list(prompt), []
    for _ in range(4):
        logits = model.lm_logits(params, partition_tokens(len(ids), 1), ids).data
        want.append(int(np.argmax(logits[-1])))
        ids.append(want[-1])
    assert got == want


def test_generate_zero_head_picks_lowest_id_and_validation(cuda):
    from paper_2505_19342_b200 import model
    from paper_2505_19342_b200.cluster import partition_tokens
    from paper_2505_19342_b200.errors import ShapeError
    params = model.init_params(model.ModelConfig(layers=2, hidden=8, heads=2, vocab_or_classes=5,
                                                 max_tokens=8, causal=True), seed=1)
    params.assign("head", np.zeros_like(params.head.data))
    plan = partition_tokens(4, 1)
    assert model.generate(params, plan, [1, 2, 3, 4], steps=3) == [0, 0, 0]
    with pytest.raises(ValueError):
        model.generate(params, plan, [0, 1, 2, 3], steps=-1)
    assert model.generate(params, plan, [0, 1, 2, 3], steps=0) == []
    with pytest.raises(ShapeError):
        model.generate(params, plan, [0, 1, 2, 3], steps=5)


@pytest.mark.parametrize("devices,cls_mode,want", [(4, "distributed", 4), (4, "single", 1),
                                                   (1, "distributed", 1)])
def test_class_replica_counts(cuda, devices, cls_mode, want):
    from paper_2505_19342_b200 import model
    from paper_2505_19342_b200.cluster import partition_tokens
    params = _enc()
    x = RNG.normal(size=(16, 32)).astype(np.float32)
    _, c = model.run_blocks(params, partition_tokens(16, devices),
                            model.embed_classifier_inputs(params, x), cls_mode=cls_mode)
    assert c.data.shape[0] == want


def test_lifecycle_and_config_errors(cuda):
    from paper_2505_19342_b200 import model, vq
    from paper_2505_19342_b200.cluster import partition_tokens
    from paper_2505_19342_b200.errors import LifecycleError, ShapeError
    enc = model.init_params(model.ModelConfig(layers=2, hidden=8, heads=2, vocab_or_classes=3,
                                              max_tokens=7, causal=False), seed=0)
    x = RNG.normal(size=(6, 8)).astype(np.float32)
    with pytest.raises(LifecycleError):
        model.classify(enc, partition_tokens(6, 2), x)          # multi-device needs codebooks
    enc.blocks[0].codebook = vq.Codebook(layer_id=0, groups=1,
                                         centroids=[RNG.normal(size=(4, 8)).astype(np.float32)])
    with pytest.raises(LifecycleError):
        model.classify(enc, partition_tokens(6, 2), x)          # partial codebooks
    enc.blocks[0].codebook = None
    with pytest.raises(ValueError):
        model.classify(enc, partition_tokens(6, 1), x, cls_mode="triple")
    with pytest.raises(ShapeError):
        model.classify(enc, partition_tokens(9, 1), np.zeros((9, 8), np.float32))
    with pytest.raises(ValueError):
        model.lm_logits(enc, partition_tokens(4, 1), [0, 1, 2, 0])
    dec = model.init_params(model.ModelConfig(layers=1, hidden=8, heads=2, vocab_or_classes=5,
                                              max_tokens=8, causal=True), seed=0)
    with pytest.raises(ValueError):
        model.classify(dec, partition_tokens(4, 1), np.zeros((4, 8), np.float32))
    a = model.classify(enc, partition_tokens(6, 1), x, cls_mode="distributed").data
    b = model.classify(enc, partition_tokens(6, 1), x, cls_mode="single").data
    np.testing.assert_array_equal(a, b)
