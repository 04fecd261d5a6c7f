"""Host-side logic on CPU: parameter generation, shard plans, ledger, checkpoint
formats, runtime layout, and the C-ABI library's exported symbols (no compute)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import astra_oracle as O

ROOT = Path(__file__).resolve().parents[1]


def test_init_params_bit_identical_to_oracle():
    from paper_2505_19342_b200 import model
    for causal in (False, True):
        kw = dict(layers=2, hidden=32, heads=4, vocab_or_classes=10, max_tokens=20, causal=causal)
        ours = model.init_params(model.ModelConfig(**kw), seed=3)
        ref = O.init_params(O.Config(**kw), seed=3)
        np.testing.assert_array_equal(ours.pos.data, ref.pos)
        np.testing.assert_array_equal(ours.head.data, ref.head)
        for b, rb in zip(ours.blocks, ref.blocks):
            for f in ("wq", "wk", "wv", "wo", "w1", "b1", "w2", "b2"):
                np.testing.assert_array_equal(getattr(b, f).data, rb[f])
        if causal:
            np.testing.assert_array_equal(ours.embedding.data, ref.embedding)
        else:
            np.testing.assert_array_equal(ours.cls.data, ref.cls)


def test_synthetic_data_matches_oracle():
    from paper_2505_19342_b200 import data
    xs, ys = data.make_classify_data(768, 196, 3, seed=1, task_seed=0)
    oxs, oys = O.make_classify_data(768, 196, 3, seed=1, task_seed=0)
    for a, b in zip(xs, oxs):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(ys, oys)


def test_partition_and_plan_errors():
    from paper_2505_19342_b200 import cluster
    from paper_2505_19342_b200.errors import PlanError
    plan = cluster.partition_tokens(10, 4)
    assert plan.ranges == ((0, 2), (2, 4), (4, 7), (7, 10))
    np.testing.assert_array_equal(plan.owner_of(), [0, 0, 1, 1, 2, 2, 2, 3, 3, 3])
    assert cluster.partition_tokens(196, 8).shard_sizes() == [24] * 4 + [25] * 4
    with pytest.raises(PlanError):
        cluster.partition_tokens(3, 4)
    with pytest.raises(PlanError):
        cluster.ShardPlan(tokens=5, devices=2, ranges=((0, 2), (3, 5)))


def test_ledger_exact_bits_and_csv():
    """test_cluster.py:67-106 formula: sent = T_d*G*bits once; received by N-1 peers."""
    from paper_2505_19342_b200 import cluster
    from paper_2505_19342_b200.vq import index_bits
    led = cluster.CommsLedger()
    plan = cluster.partition_tokens(196, 4)
    bits = [s * 1 * index_bits(1024) for s in plan.shard_sizes()]
    for layer in range(12):
        led.record_exchange(layer, bits)
    assert led.total_bits_sent() == 23520          # golden CLI run: 120 bits/token
    assert led.bits_per_token(196) == 120
    csv = led.to_csv().splitlines()
    assert csv[0] == "layer,device,bits_sent,bits_received,messages"
    assert csv[1] == "0,0,490,1470,1"


def test_allgather_indices_protocol():
    from paper_2505_19342_b200 import cluster
    from paper_2505_19342_b200.errors import ProtocolError
    from paper_2505_19342_b200.vq import QuantizedTokens
    devs = [cluster.DeviceState(device_id=d, span=(d, d + 1), x_local=np.zeros((1, 2)),
                                replica=None, codebooks=[]) for d in range(3)]
    q = lambda d: QuantizedTokens(layer_id=0, token_count=1,  # noqa: E731
                                  indices=np.array([[d]], np.int32), bits_per_token=4)
    led = cluster.CommsLedger()
    with pytest.raises(ProtocolError):
        cluster.allgather_indices(devs, 0, led)
    for d in devs:
        d.staged = cluster.IndexMessage(sender=d.device_id, layer=0, payload=q(d.device_id))
    cluster.allgather_indices(devs, 0, led)
    assert sorted(devs[0].inbox) == [1, 2] and led.total_bits_sent() == 12
    assert all(d.staged is None for d in devs)


def test_checkpoint_roundtrip():
    from paper_2505_19342_b200 import model, vq
    cfg = model.ModelConfig(layers=2, hidden=16, heads=2, vocab_or_classes=5, max_tokens=9,
                            causal=False, codebook_size=4, groups=2)
    p = model.init_params(cfg, seed=1)
    rng = np.random.default_rng(0)
    for i, b in enumerate(p.blocks):
        b.codebook = vq.Codebook(layer_id=i, groups=2,
                                 centroids=[rng.normal(size=(4, 8)).astype(np.float32)] * 2)
    blob = model.save_checkpoint(p)
    q = model.load_checkpoint(blob)
    for (n, a), (m, b) in zip(p.named_tensors(), q.named_tensors()):
        assert n == m
        np.testing.assert_array_equal(a.data, b.data)
    assert model.save_checkpoint(q) == blob
    with pytest.raises(ValueError):
        model.load_checkpoint(b"XXXX" + blob[4:])
    with pytest.raises(ValueError):
        model.load_checkpoint(blob + b"\0")


def test_index_bits():
    from paper_2505_19342_b200.vq import index_bits
    assert [index_bits(k) for k in (1, 2, 3, 16, 1024)] == [0, 1, 2, 4, 10]


def _declared_symbols():
    text = (ROOT / "include" / "astra_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(astra_\w+)\(", text, re.M)))


def test_native_library_exports_every_declared_symbol():
    from paper_2505_19342_b200 import _native
    path = _native.lib_path()
    if not path.exists():
        from paper_2505_19342_b200 import build
        build.build()
    lib = ctypes.CDLL(str(path))
    declared = _declared_symbols()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.SIGNATURES), "ctypes table out of sync with the header"
    assert lib.astra_abi_version() == _native.ABI_VERSION


def test_softmax_perturbation_first_order():
    """attention.softmax_perturbation_first_order: finite-difference agreement, zero sum and
    validation as the reference's tests (test_attention.py:165-189)."""
    from paper_2505_19342_b200.attention import softmax_perturbation_first_order as f
    from paper_2505_19342_b200.errors import ShapeError
    rng = np.random.default_rng(0)
    logits = rng.normal(size=9)
    alpha = np.exp(logits - logits.max())
    alpha /= alpha.sum()
    e = rng.normal(size=9)
    h = 1e-6
    up = np.exp(logits + h * e - (logits + h * e).max())
    up /= up.sum()
    np.testing.assert_allclose(f(alpha, e), (up - alpha) / h, atol=1e-5)
    assert abs(f(np.array([0.5, 0.3, 0.2]), np.array([1.0, -2.0, 0.5])).sum()) < 1e-12
    with pytest.raises(ShapeError):
        f(np.array([0.5, 0.5]), np.zeros(3))
    with pytest.raises(ValueError):
        f(np.array([0.9, 0.3]), np.zeros(2))
