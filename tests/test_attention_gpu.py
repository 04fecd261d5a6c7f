"""Mixed-precision attention kernels (tcgen05 bf16 and fp32 SIMT) vs a PyTorch fp32
reference of the same op: segments with local and remote (codebook-table) keys,
class-replica keys, causal masks."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _problem(seed, segs_spec, heads=12, dk=64, causal=False, dtype=torch.bfloat16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    D = heads * dk
    n_local = sum(nq for nq, _, _ in segs_spec) + 8
    qkv = (torch.randn(n_local, 3 * D, device="cuda", generator=g)).to(dtype)
    table = (torch.randn(300, 2 * D, device="cuda", generator=g)).to(dtype)
    rng = np.random.default_rng(seed)
    segs, key_src, key_pos = [], [], []
    q0 = 0
    for nq, nk, nrep in segs_spec:
        k0 = len(key_src)
        ncontent = nq - nrep
        for j in range(nk):
            if j < nk - nrep:
                if rng.random() < 0.5:
                    key_src.append(int(q0 + rng.integers(0, nq)))
                else:
                    key_src.append(-int(rng.integers(0, 300)) - 1)
                key_pos.append(j)
            else:
                key_src.append(q0 + nq - 1)
                key_pos.append(-1)
        segs.append([q0, nq, 5, ncontent, k0, nk])
        q0 += nq
    t = lambda a: torch.tensor(np.asarray(a, np.int32), device="cuda")  # noqa: E731
    return qkv, table, t(np.asarray(segs).reshape(-1)), t(key_src), t(key_pos), segs


def _reference(qkv, table, segs, key_src, key_pos, heads, dk, causal):
    D = heads * dk
    dt = torch.float64 if qkv.dtype == torch.float64 else torch.float32
    q_all, k_loc, v_loc = qkv[:, :D].to(dt), qkv[:, D:2 * D].to(dt), qkv[:, 2 * D:].to(dt)
    k_rem, v_rem = table[:, :D].to(dt), table[:, D:].to(dt)
    out = torch.zeros(qkv.shape[0], D, device="cuda", dtype=dt)
    ks, kp = key_src.cpu().numpy(), key_pos.cpu().numpy()
    for q0, nq, qpos0, ncontent, k0, nk in segs:
        src = ks[k0:k0 + nk]
        pos = torch.tensor(kp[k0:k0 + nk], device="cuda")
        loc = torch.tensor(src >= 0, device="cuda")
        li = torch.tensor(np.where(src >= 0, src, 0), device="cuda").long()
        ri = torch.tensor(np.where(src < 0, -(src + 1), 0), device="cuda").long()
        K = torch.where(loc[:, None], k_loc[li], k_rem[ri])
        V = torch.where(loc[:, None], v_loc[li], v_rem[ri])
        qpos = torch.tensor([qpos0 + i if i < ncontent else 2 ** 31 - 1 for i in range(nq)],
                            device="cuda")
        mask = (pos[None, :] <= qpos[:, None]) if causal else torch.ones(nq, nk, dtype=torch.bool,
                                                                          device="cuda")
        for h in range(heads):
            s = slice(h * dk, (h + 1) * dk)
            logits = (q_all[q0:q0 + nq, s] @ K[:, s].T) * (1.0 / math.sqrt(dk))
            logits = logits.masked_fill(~mask, float("-inf"))
            out[q0:q0 + nq, s] = torch.softmax(logits, dim=1) @ V[:, s]
    return out


def test_dropin_multihead_attention_golden(cuda):
    """attention.multihead_attention vs the reference's own outputs (test_attention.py:50: 1e-6)."""
    from pathlib import Path

    from paper_2505_19342_b200 import attention
    from tests.golden.cases import ATT_CASES, att_case_inputs
    gold = np.load(Path(__file__).resolve().parent / "golden" / "golden_attention.npz")
    for i, (r, c, d, h, p) in enumerate(ATT_CASES):
        q, k, v, mask = att_case_inputs(i, r, c, d, p)
        out = attention.multihead_attention(q, k, v, mask, h)
        np.testing.assert_allclose(out, gold[f"c{i}_out"], atol=1e-5)


def test_dropin_attention_errors(cuda):
    from paper_2505_19342_b200 import attention
    from paper_2505_19342_b200.errors import MaskError, ShapeError
    q = np.ones((4, 8), np.float32)
    with pytest.raises(ShapeError):
        attention.multihead_attention(q, q, q, np.ones((4, 4), bool), 3)
    m = np.ones((4, 4), bool)
    m[2] = False
    with pytest.raises(MaskError):
        attention.multihead_attention(q, q, q, m, 2)


SPECS = [[(197, 197, 1)], [(50, 197, 1), (49, 197, 1), (25, 197, 1)], [(130, 300, 0), (7, 7, 0)],
         [(256, 129, 1)], [(200, 600, 1), (64, 256, 0), (16, 16, 1)], [(1, 257, 1)]]


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("force_simt,variant", [(False, 0), (False, 1), (False, 2), (True, 0)])
def test_attention_kernels_vs_torch(cuda, spec, causal, force_simt, variant):
    from paper_2505_19342_b200 import _native
    heads, dk = 12, 64
    qkv, table, segs_t, ks, kp, segs = _problem(len(spec) + 7 * causal, spec, heads, dk, causal)
    D = heads * dk
    out = torch.zeros(qkv.shape[0], D, dtype=torch.bfloat16, device="cuda")
    lib = _native.load()
    lib.astra_attention_force_simt(int(force_simt))
    lib.astra_attention_variant(variant)
    try:
        es = qkv.element_size()
        _native.call("astra_attention", qkv.data_ptr(), 3 * D, qkv.data_ptr() + D * es,
                     qkv.data_ptr() + 2 * D * es, 3 * D, table.data_ptr(),
                     table.data_ptr() + D * es, 2 * D, ks.data_ptr(), kp.data_ptr(),
                     segs_t.data_ptr(), len(segs), max(s[1] for s in segs), heads, dk, int(causal),
                     1, float(np.float32(1 / math.sqrt(dk))), None, out.data_ptr(), None, D,
                     qkv.shape[0], qkv.shape[0], table.shape[0],
                     torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    finally:
        lib.astra_attention_force_simt(0)
        lib.astra_attention_variant(0)
    ref = _reference(qkv, table, segs, ks, kp, heads, dk, causal)
    rows = torch.cat([torch.arange(s[0], s[0] + s[1]) for s in segs]).cuda()
    err = (out.float()[rows] - ref[rows]).abs().max().item()
    tol = 2e-2 if not force_simt else 8e-3   # bf16 P (tcgen05) / bf16 output rounding (SIMT)
    assert err < tol, err


@pytest.mark.parametrize("variant", [0, 2])
@pytest.mark.parametrize("factor", [8.0, 60.0])
@pytest.mark.parametrize("causal", [False, True])
def test_attention_score_outliers(cuda, factor, causal, variant):
    """Keys whose scores sit far above the first keys of the row.  The single-pipeline kernel
    (variant 2) takes its exponent reference from keys 0..127 and must either absorb them
    (P up to 2^64) or redo keys 128.. with the exact row max; the default kernel uses the
    exact max throughout."""
    from paper_2505_19342_b200 import _native
    _native.load().astra_attention_variant(variant)
    heads, dk = 12, 64
    spec = [(197, 197, 1), (50, 300, 0)]
    qkv, table, segs_t, ks, kp, segs = _problem(11, spec, heads, dk, causal)
    D = heads * dk
    srcs = ks.cpu().numpy()
    for q0, nq, _, _, k0, nk in segs:
        for j in (100, nk - 40):
            r = int(srcs[k0 + j])
            if r < 0:
                table[-r - 1, :D] *= factor
            else:
                qkv[r, D:2 * D] *= factor
    out = torch.zeros(qkv.shape[0], D, dtype=torch.bfloat16, device="cuda")
    es = qkv.element_size()
    _native.call("astra_attention", qkv.data_ptr(), 3 * D, qkv.data_ptr() + D * es,
                 qkv.data_ptr() + 2 * D * es, 3 * D, table.data_ptr(),
                 table.data_ptr() + D * es, 2 * D, ks.data_ptr(), kp.data_ptr(),
                 segs_t.data_ptr(), len(segs), max(s[1] for s in segs), heads, dk, int(causal),
                 1, float(np.float32(1 / math.sqrt(dk))), None, out.data_ptr(), None, D,
                 qkv.shape[0], qkv.shape[0], table.shape[0],
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    _native.load().astra_attention_variant(0)
    ref = _reference(qkv, table, segs, ks, kp, heads, dk, causal)
    rows = torch.cat([torch.arange(s[0], s[0] + s[1]) for s in segs]).cuda()
    o = out.float()[rows]
    assert torch.isfinite(o).all()
    err = (o - ref[rows]).abs().max().item()
    assert err < 2e-2 * factor, err


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("force_simt", [False, True])
def test_attention_fp32_parity_kernels_vs_fp64(cuda, spec, causal, force_simt):
    """Parity-mode attention (fp32 operands): the split-bf16 tcgen05 kernel (attention_tc3) and
    the fp32 SIMT kernel against an fp64 evaluation of the same op; output as fp32 and as the
    bf16 hi/lo split the next GEMM consumes (hi + lo reconstructs it to 2^-16)."""
    from paper_2505_19342_b200 import _native
    heads, dk = 12, 64
    qkv, table, segs_t, ks, kp, segs = _problem(len(spec) + 7 * causal, spec, heads, dk, causal,
                                                dtype=torch.float32)
    qkv = qkv * 0.5
    table = table * 0.5
    D = heads * dk
    out = torch.zeros(qkv.shape[0], D, device="cuda")
    hi = torch.zeros(qkv.shape[0], D, dtype=torch.bfloat16, device="cuda")
    lo = torch.zeros_like(hi)
    lib = _native.load()
    lib.astra_attention_force_simt(int(force_simt))
    try:
        es = 4
        _native.call("astra_attention", qkv.data_ptr(), 3 * D, qkv.data_ptr() + D * es,
                     qkv.data_ptr() + 2 * D * es, 3 * D, table.data_ptr(),
                     table.data_ptr() + D * es, 2 * D, ks.data_ptr(), kp.data_ptr(),
                     segs_t.data_ptr(), len(segs), max(s[1] for s in segs), heads, dk, int(causal),
                     0, float(np.float32(1 / math.sqrt(dk))), out.data_ptr(), hi.data_ptr(),
                     lo.data_ptr(), D, qkv.shape[0], qkv.shape[0], table.shape[0],
                     torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    finally:
        lib.astra_attention_force_simt(0)
    ref = _reference(qkv.double(), table.double(), segs, ks, kp, heads, dk, causal)
    rows = torch.cat([torch.arange(s[0], s[0] + s[1]) for s in segs]).cuda()
    scale = ref[rows].abs().max().item()
    err = (out[rows].double() - ref[rows]).abs().max().item() / scale
    err_split = ((hi.double() + lo.double())[rows] - ref[rows]).abs().max().item() / scale
    # fp32-class: bf16x3 products (operand split error <= 2^-17 relative, lo*lo dropped) with
    # fp32 accumulation — the same class as the parity-mode GEMMs
    assert err < 2e-5, err
    assert err_split < 2e-5, err_split


@pytest.mark.parametrize("variant", [0, 2])
@pytest.mark.parametrize("fp32", [False, True])
def test_attention_causal_prefix_skip(cuda, variant, fp32):
    """causal = 2 (prefix keys, the runtime's causal layout): key chunks past a query tile's
    last position are skipped; results equal the masked reference."""
    from paper_2505_19342_b200 import _native
    heads, dk = 12, 64
    spec = [(130, 300, 0), (64, 700, 0), (7, 7, 0), (300, 520, 0)]
    qkv, table, segs_t, ks, kp, segs = _problem(99, spec, heads, dk, True,
                                                dtype=torch.float32 if fp32 else torch.bfloat16)
    D = heads * dk
    out = torch.zeros(qkv.shape[0], D, dtype=torch.float32 if fp32 else torch.bfloat16,
                      device="cuda")
    _native.load().astra_attention_variant(variant)
    es = qkv.element_size()
    try:
        _native.call("astra_attention", qkv.data_ptr(), 3 * D, qkv.data_ptr() + D * es,
                     qkv.data_ptr() + 2 * D * es, 3 * D, table.data_ptr(),
                     table.data_ptr() + D * es, 2 * D, ks.data_ptr(), kp.data_ptr(),
                     segs_t.data_ptr(), len(segs), max(s[1] for s in segs), heads, dk, 2,
                     0 if fp32 else 1, float(np.float32(1 / math.sqrt(dk))),
                     out.data_ptr() if fp32 else None, None if fp32 else out.data_ptr(), None, D,
                     qkv.shape[0], qkv.shape[0], table.shape[0],
                     torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    finally:
        _native.load().astra_attention_variant(0)
    ref = _reference(qkv, table, segs, ks, kp, heads, dk, True)
    rows = torch.cat([torch.arange(s[0], s[0] + s[1]) for s in segs]).cuda()
    err = (out.float()[rows] - ref[rows].float()).abs().max().item()
    assert err < (1e-4 if fp32 else 2e-2), err
