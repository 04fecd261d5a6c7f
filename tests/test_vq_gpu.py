"""VQ encode/decode on the GPU vs the fp64 oracle: indices must be bit-exact."""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import astra_oracle as O
from tests.golden.cases import VQ_CASES, vq_case_inputs

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("i", range(len(VQ_CASES)))
def test_quantize_golden(cuda, i):
    from paper_2505_19342_b200 import vq
    gold = np.load(G / "golden_vq.npz")
    k, d, g, m = VQ_CASES[i]
    if i == len(VQ_CASES) - 1:
        cents = [np.array([[1.0, 0.0], [-1.0, 0.0]], np.float32)]
        x = np.zeros((m, d), np.float32)
    else:
        cents, x = vq_case_inputs(i, k, d, g, m)
    cb = vq.Codebook(layer_id=0, groups=g, centroids=cents)
    q, xhat = vq.quantize(cb, x)
    np.testing.assert_array_equal(q.indices, gold[f"c{i}_idx"])
    np.testing.assert_array_equal(xhat, O.dequantize(cents, q.indices))
    assert q.bits_per_token == int(gold[f"c{i}_bits"][0])


@pytest.mark.parametrize("m,k,d,g,scale", [(6000, 1024, 768, 1, 1.0), (3000, 1024, 768, 16, 1.0),
                                           (2000, 1024, 768, 32, 0.3), (4000, 4096, 64, 1, 1.0),
                                           (3000, 256, 1024, 1, 5.0), (513, 8, 32, 1, 1.0),
                                           # wide codebooks: > 32 chunk records per row (G=1),
                                           # run mode with 1024-code parts (G=16)
                                           (3000, 4096, 1024, 1, 1.0), (2000, 4096, 1024, 16, 1.0)])
def test_quantize_random_bit_exact(cuda, m, k, d, g, scale):
    from paper_2505_19342_b200 import vq
    rng = np.random.default_rng(m + k + d + g)
    gd = d // g
    # clustered data: tokens near codes -> many near-ties, the hard case for the window
    cents = [(rng.normal(size=(k, gd)) * scale).astype(np.float32) for _ in range(g)]
    base = np.concatenate([c[rng.integers(0, k, size=m)] for c in cents], axis=1)
    x = (base + rng.normal(size=(m, d)) * 0.05 * scale).astype(np.float32)
    dc = vq.DeviceCodebook(torch.from_numpy(np.stack(cents)).cuda())
    stats = torch.zeros(4, dtype=torch.int32, device="cuda")
    idx = dc.encode(torch.from_numpy(x).cuda(), stats=stats).cpu().numpy()
    want = O.quantize(cents, x)
    assert (idx != want).sum() == 0, f"{(idx != want).sum()} mismatches; stats={stats.tolist()}"


def test_quantize_real_layer_inputs(cuda):
    """ViT-B width, K=1024: the reference's own layer inputs and codebooks."""
    from paper_2505_19342_b200 import vq
    meta = json.loads((G / "golden_infer_meta.json").read_text())["vitb2"]
    gold = np.load(G / "golden_infer.npz")
    cfg = O.Config(**meta["model"])
    params = O.init_params(cfg, seed=0)
    xs, _ = O.make_classify_data(768, 196, 8, seed=0, task_seed=0)
    O.initialize_codebooks(params, xs, "classify", seed=0)
    x_in = O.make_classify_data(768, 196, 1, seed=1, task_seed=0)[0][0]
    caps = O.capture_block_inputs(params, [x_in])
    want = gold["vitb2_n1_distributed_indices"].reshape(2, 196)
    for layer in range(2):
        cb = vq.Codebook(layer_id=layer, groups=1, centroids=params.codebooks[layer])
        q, _ = vq.quantize(cb, caps[layer])
        np.testing.assert_array_equal(q.indices[:, 0], want[layer])


def test_dequantize_rejects_corrupt(cuda):
    from paper_2505_19342_b200 import vq
    from paper_2505_19342_b200.errors import IndexCorruptionError
    cb = vq.Codebook(layer_id=0, groups=1, centroids=[np.eye(4, dtype=np.float32)])
    q = vq.QuantizedTokens(layer_id=0, token_count=2, indices=np.array([[0], [7]], np.int32),
                           bits_per_token=2)
    with pytest.raises(IndexCorruptionError):
        vq.dequantize(cb, q)
    dc = cb.on_device()
    with pytest.raises(IndexCorruptionError):
        dc.decode(torch.tensor([[1], [9]], dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("bits,n", [(10, 3136), (1, 77), (12, 1000), (5, 33), (0, 10)])
def test_pack_roundtrip(cuda, bits, n):
    from paper_2505_19342_b200 import kernels
    rng = np.random.default_rng(bits * 1000 + n)
    k = max(1, 1 << bits)
    idx = rng.integers(0, k, size=n).astype(np.int32)
    words = kernels.pack_indices(torch.from_numpy(idx).cuda(), bits)
    if bits:
        np.testing.assert_array_equal(words.cpu().numpy().view(np.uint32), O.pack_indices(idx, bits))
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    back = kernels.unpack_indices(words, n, bits, k, err=err)
    np.testing.assert_array_equal(back.cpu().numpy(), idx if bits else np.zeros(n, np.int32))
    assert int(err.item()) == 0
    if bits >= 2:   # a code >= K in the stream is flagged
        bad = kernels.unpack_indices(words, n, bits, int(idx.max()), err=err)
        assert int(err.item()) == 1
        del bad


@pytest.mark.parametrize("m,k,d,g", [(3000, 1024, 768, 16), (777, 256, 1024, 16), (500, 64, 512, 2),
                                     (300, 32, 768, 32)])
def test_decode_layernorm_equals_decode_then_layernorm(cuda, m, k, d, g):
    """astra_vq_decode_layernorm (decode fused into LN1) is bitwise the two-kernel path, in both
    the fast (bf16) and the parity (bf16 hi/lo) operand forms; bad codes raise the flag."""
    from paper_2505_19342_b200 import _native
    from paper_2505_19342_b200.vq import DeviceCodebook
    import ctypes
    rng = np.random.default_rng(m + d)
    gd = d // g
    cents = torch.from_numpy(rng.normal(size=(g, k, gd)).astype(np.float32)).to(cuda)
    cb = DeviceCodebook(cents)
    idx = torch.from_numpy(rng.integers(0, k, size=(m, g)).astype(np.int32)).to(cuda)
    gain = torch.from_numpy(rng.normal(size=d).astype(np.float32)).to(cuda)
    bias = torch.from_numpy(rng.normal(size=d).astype(np.float32)).to(cuda)
    s = torch.cuda.current_stream().cuda_stream
    err = torch.zeros(2, dtype=torch.int32, device=cuda)
    xhat = cb.decode(idx)
    want_hi = torch.empty(m, d, dtype=torch.bfloat16, device=cuda)
    want_lo = torch.empty_like(want_hi)
    _native.call("astra_layernorm", xhat.data_ptr(), m, d, d, gain.data_ptr(), bias.data_ptr(),
                 1e-5, None, 0, want_hi.data_ptr(), want_lo.data_ptr(), d, s)
    hi, lo = torch.empty_like(want_hi), torch.empty_like(want_lo)
    _native.call("astra_vq_decode_layernorm", ctypes.byref(cb.struct), idx.data_ptr(), m,
                 gain.data_ptr(), bias.data_ptr(), 1e-5, hi.data_ptr(), lo.data_ptr(), d,
                 err.data_ptr(), s)
    torch.cuda.synchronize()
    assert int(err[0]) == 0
    assert torch.equal(hi.view(torch.int16), want_hi.view(torch.int16))
    assert torch.equal(lo.view(torch.int16), want_lo.view(torch.int16))
    idx[m // 2, g - 1] = k   # out of range
    _native.call("astra_vq_decode_layernorm", ctypes.byref(cb.struct), idx.data_ptr(), m,
                 gain.data_ptr(), bias.data_ptr(), 1e-5, hi.data_ptr(), None, d, err.data_ptr(), s)
    torch.cuda.synchronize()
    assert int(err[0]) == 1


@pytest.mark.parametrize("g,m", [(16, 3000), (1, 2000)])
def test_quantize_overflow_scans_bit_exact(cuda, g, m):
    """Codebooks of near-duplicate codes: every token has ~16 codes inside the error window,
    so candidate lists overflow — run mode (G=16) sends the items to the split exact scans
    (more than the list capacity here, so the one-warp fallback runs too), records mode (G=1)
    scans the overflowing 64-code parts.  Indices stay bit-identical to the fp64 argmin."""
    from paper_2505_19342_b200 import vq
    rng = np.random.default_rng(7 + g)
    k, d = 1024, 1024
    gd = d // g
    cents = []
    for _ in range(g):
        base = rng.normal(size=(k // 16, gd))
        cents.append((np.repeat(base, 16, axis=0) + rng.normal(size=(k, gd)) * 1e-5).astype(np.float32))
    x = np.concatenate([c[rng.integers(0, k, size=m)] for c in cents], axis=1)
    x = (x + rng.normal(size=(m, d)) * 1e-3).astype(np.float32)
    dc = vq.DeviceCodebook(torch.from_numpy(np.stack(cents)).cuda())
    stats = torch.zeros(4, dtype=torch.int32, device="cuda")
    idx = dc.encode(torch.from_numpy(x).cuda(), stats=stats).cpu().numpy()
    want = O.quantize(cents, x)
    assert (idx != want).sum() == 0, f"{(idx != want).sum()} mismatches; stats={stats.tolist()}"
    assert stats[1].item() > 0, stats.tolist()   # exact scans ran


@pytest.mark.parametrize("m,k,g,d", [(3000, 1024, 16, 1024), (999, 256, 32, 1024), (500, 64, 48, 768)])
def test_decode_narrow_groups(cuda, m, k, g, d):
    """Per-float4 decode (groups narrower than 128): equals the CPU gather bytewise."""
    from paper_2505_19342_b200 import vq
    rng = np.random.default_rng(m + g)
    gd = d // g
    cents = rng.normal(size=(g, k, gd)).astype(np.float32)
    idx = rng.integers(0, k, size=(m, g)).astype(np.int32)
    dc = vq.DeviceCodebook(torch.from_numpy(cents).cuda())
    got = dc.decode(torch.from_numpy(idx).cuda()).cpu().numpy()
    want = np.concatenate([cents[j][idx[:, j]] for j in range(g)], axis=1)
    np.testing.assert_array_equal(got, want)
