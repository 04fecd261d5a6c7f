"""CPU ORACLE — test infrastructure only.

A NumPy restatement of the reference's Astra inference path
(seqvq 0.1.0, /root/reference/pkg/src/seqvq).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline / reference legs
may import this module, and only as the checker or the timed CPU baseline —
never as part of the product path (the product raises if its CUDA library is
missing; it has no CPU fallback).

Every function cites the reference file:line it follows.  Numerics are kept
exactly as the reference computes them: fp32 storage, matmul accumulated in
fp64 then cast to fp32 (tensor.py:142-155), all elementwise math in fp32 under
NumPy 2 scalar promotion, VQ distances in fp64 (vq.py:126-131).

Pinning: tests/test_oracle_golden.py checks this module against golden
vectors produced by the reference itself (tests/golden/make_golden.py) —
indices/ledger bitwise, floats to the reference tests' own tolerances.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import erf

F32 = np.float32
LN_EPS = 1e-5                # model.py:28
MASK_FILL = -1e9             # tensor.py:16
_INV_SQRT2 = 0.7071067811865476  # tensor.py:17


# ----------------------------------------------------------------- rng.py
def _stable_hash(name) -> int:
    """rng.py:24-29"""
    if isinstance(name, (int, np.integer)):
        return int(name) & 0xFFFFFFFFFFFFFFFF
    return int.from_bytes(hashlib.sha256(str(name).encode("utf-8")).digest()[:8], "little")


def generator(seed: int, *names) -> np.random.Generator:
    """rng.py:32-37 — PCG64 over SeedSequence([seed, H(name)...])."""
    entropy = [int(seed) & 0xFFFFFFFFFFFFFFFF] + [_stable_hash(n) for n in names]
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))


# -------------------------------------------------------------- tensor.py
def matmul(a, b):
    """tensor.py:142-155: fp64 accumulate, cast back to storage dtype."""
    return (a.astype(np.float64) @ b.astype(np.float64)).astype(a.dtype)


def layer_norm(x, gain, bias, eps=LN_EPS):
    """tensor.py:318-345 (fp32 statistics, biased variance)."""
    mu = x.mean(axis=1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=1, keepdims=True)
    inv = 1.0 / np.sqrt(var + eps)
    xh = (xc * inv).astype(x.dtype)
    return (xh * gain[None, :] + bias[None, :]).astype(x.dtype)


def masked_softmax(logits, mask):
    """tensor.py:295-315: -1e9 fill, max-subtract, exp, exact zeros, normalise."""
    x = logits + np.asarray(MASK_FILL, dtype=logits.dtype) * (~mask)
    x = x - x.max(axis=1, keepdims=True)
    e = np.exp(x)
    e = np.where(mask, e, 0.0).astype(logits.dtype)
    return e / e.sum(axis=1, keepdims=True)


def gelu(x):
    """tensor.py:348-358: exact erf form."""
    cdf = 0.5 * (1.0 + erf(x * _INV_SQRT2))
    return (x * cdf).astype(x.dtype)


# ----------------------------------------------------------- attention.py
def multihead_attention(q, k, v, mask, heads):
    """attention.py:50-73 (per-head loop; scale applied after the matmul)."""
    r, d = q.shape
    dk = d // heads
    inv = 1.0 / math.sqrt(dk)
    outs = []
    for h in range(heads):
        s = slice(h * dk, (h + 1) * dk)
        logits = matmul(np.ascontiguousarray(q[:, s]), np.ascontiguousarray(k[:, s].T))
        logits = logits * np.asarray(inv, dtype=logits.dtype)
        w = masked_softmax(logits, mask)
        outs.append(matmul(w, np.ascontiguousarray(v[:, s])))
    return np.concatenate(outs, axis=1) if heads > 1 else outs[0]


def build_mask(tokens, ranges, causal):
    """attention.py:36-47: [T, 2T] routing mask (same shard -> full precision)."""
    owner = owner_of(ranges, tokens)
    same = owner[:, None] == owner[None, :]
    vis = np.tril(np.ones((tokens, tokens), bool)) if causal else np.ones((tokens, tokens), bool)
    return np.concatenate([vis & same, vis & ~same], axis=1)


# ------------------------------------------------------------------ vq.py
def index_bits(k: int) -> int:
    """vq.py:24-28"""
    return max(0, math.ceil(math.log2(k)))


def nearest(points, centroids):
    """vq.py:126-131: fp64 ||p||^2 - 2 p.c + ||c||^2, argmin (lowest index on ties)."""
    p = points.astype(np.float64)
    c = centroids.astype(np.float64)
    d2 = (p * p).sum(axis=1, keepdims=True) - 2.0 * (p @ c.T) + (c * c).sum(axis=1)[None, :]
    return np.argmin(d2, axis=1)


def quantize(centroids: list, x):
    """vq.py:207-222: per-group nearest index -> int32 [T, G]."""
    g_count = len(centroids)
    gd = centroids[0].shape[1]
    idx = np.empty((x.shape[0], g_count), dtype=np.int32)
    for g in range(g_count):
        idx[:, g] = nearest(x[:, g * gd:(g + 1) * gd], centroids[g])
    return idx


def dequantize(centroids: list, idx):
    """vq.py:225-233 (range check, groups concatenated in order)."""
    k = centroids[0].shape[0]
    if idx.size and (idx.min() < 0 or idx.max() >= k):
        raise IndexError("index outside codebook")
    return np.concatenate([centroids[g][idx[:, g]] for g in range(len(centroids))], axis=1)


def _lloyd(points, k, iterations, gen):
    """vq.py:134-166: Lloyd with farthest-point reseeding of empty clusters."""
    m = points.shape[0]
    pts = points.astype(np.float64)
    cents = pts[gen.choice(m, size=k, replace=False)].copy()
    history = []
    for _ in range(max(1, iterations)):
        assign = nearest(pts, cents)
        dist2 = ((pts - cents[assign]) ** 2).sum(axis=1)
        reseeded = False
        for idx in range(k):
            if not (assign == idx).any():
                far = int(np.argmax(dist2))
                cents[idx] = pts[far]
                assign[far] = idx
                dist2[far] = 0.0
                reseeded = True
        history.append(float(dist2.mean()))
        new = cents.copy()
        for idx in range(k):
            sel = assign == idx
            if sel.any():
                new[idx] = pts[sel].mean(axis=0)
        if not reseeded and np.array_equal(new, cents):
            break
        cents = new
    return cents, history


def kmeans_init(x, k, groups, iterations=25, seed=0, layer_id=0):
    """vq.py:169-204 (centroids only; EMA state is training-side)."""
    gd = x.shape[1] // groups
    dtype = x.dtype if x.dtype in (np.float32, np.float64) else np.float32
    out = []
    for g in range(groups):
        gen = generator(seed, "kmeans", layer_id, g)
        c, _ = _lloyd(x[:, g * gd:(g + 1) * gd], k, iterations, gen)
        out.append(c.astype(dtype))
    return out


# --------------------------------------------------------------- model.py
@dataclass(frozen=True)
class Config:
    """model.py:31-56"""
    layers: int
    hidden: int
    heads: int
    vocab_or_classes: int
    max_tokens: int
    causal: bool
    mlp_expansion: int = 4
    codebook_size: int = 16
    groups: int = 1


@dataclass
class Params:
    """model.py:59-123 (flattened: blocks are dicts of fp32 arrays)."""
    config: Config
    pos: np.ndarray
    blocks: list
    final_gain: np.ndarray
    final_bias: np.ndarray
    head: np.ndarray
    embedding: np.ndarray | None = None
    cls: np.ndarray | None = None
    codebooks: list | None = None   # per layer: list of G [K, D/G] fp32 tables


def init_params(cfg: Config, seed: int) -> Params:
    """model.py:126-160: N(0,1)*0.02 per named stream; pos *0.01; LN identity; zero biases."""
    d, m = cfg.hidden, cfg.hidden * cfg.mlp_expansion

    def w(name, shape, scl=0.02):
        return (generator(seed, "init", name).normal(size=shape) * scl).astype(F32)

    blocks = []
    for i in range(cfg.layers):
        blocks.append(dict(
            wq=w(f"b{i}.wq", (d, d)), wk=w(f"b{i}.wk", (d, d)), wv=w(f"b{i}.wv", (d, d)),
            wo=w(f"b{i}.wo", (d, d)), w1=w(f"b{i}.w1", (d, m)), b1=np.zeros(m, F32),
            w2=w(f"b{i}.w2", (m, d)), b2=np.zeros(d, F32),
            ln1_gain=np.ones(d, F32), ln1_bias=np.zeros(d, F32),
            ln2_gain=np.ones(d, F32), ln2_bias=np.zeros(d, F32)))
    return Params(
        config=cfg,
        embedding=w("embedding", (cfg.vocab_or_classes, d)) if cfg.causal else None,
        pos=w("pos", (cfg.max_tokens, d), 0.01),
        cls=w("cls", (1, d)) if not cfg.causal else None,
        blocks=blocks, final_gain=np.ones(d, F32), final_bias=np.zeros(d, F32),
        head=w("head", (d, cfg.vocab_or_classes)))


# --------------------------------------------------------------- train.py
_ANCHORS = np.array([[1.5, 1.5], [1.5, -1.5], [-1.5, 1.5], [-1.5, -1.5]])


def make_classify_data(dim, tokens, count, seed, spread=0.3, signal_fraction=0.25, task_seed=0):
    """train.py:66-90: rank-2 lifted cluster samples; returns (list of [T, dim] fp32, labels)."""
    gen = generator(seed, "classify-data")
    lift = generator(task_seed, "classify-lift").normal(size=(2, dim)) / math.sqrt(2.0)
    signal = max(1, round(tokens * signal_fraction))
    xs, labels = [], []
    for _ in range(count):
        label = int(gen.integers(0, len(_ANCHORS)))
        pts = gen.normal(size=(tokens, 2)) * spread
        where = gen.choice(tokens, size=signal, replace=False)
        pts[where] += _ANCHORS[label]
        xs.append((pts @ lift).astype(F32))
        labels.append(label)
    return xs, np.asarray(labels, dtype=np.int64)


def make_lm_data(vocab, tokens, count, seed, task_seed=0):
    """train.py:93-112: Markov-chain id sequences (vocab <= 64)."""
    gen = generator(seed, "lm-data")
    logits = 2.0 * generator(task_seed, "lm-chain").normal(size=(vocab, vocab))
    z = logits - logits.max(axis=1, keepdims=True)
    p = np.exp(z)
    p /= p.sum(axis=1, keepdims=True)
    seqs = []
    for _ in range(count):
        ids = np.empty(tokens + 1, dtype=np.int64)
        ids[0] = int(gen.integers(0, vocab))
        for t in range(tokens):
            ids[t + 1] = int(gen.choice(vocab, p=p[ids[t]]))
        seqs.append(ids)
    return seqs


# -------------------------------------------------------------- cluster.py
def partition_tokens(tokens: int, devices: int):
    """cluster.py:62-76: contiguous near-even shards, remainder to trailing devices."""
    if devices < 1 or tokens < devices:
        raise ValueError("bad plan")
    base, rem = divmod(tokens, devices)
    ranges, cur = [], 0
    for dev in range(devices):
        size = base + (1 if dev >= devices - rem else 0)
        ranges.append((cur, cur + size))
        cur += size
    return tuple(ranges)


def owner_of(ranges, tokens):
    """cluster.py:52-56"""
    owner = np.empty(tokens, dtype=np.int64)
    for dev, (s, e) in enumerate(ranges):
        owner[s:e] = dev
    return owner


@dataclass
class Ledger:
    """cluster.py:92-128 — bits sent/received and messages per (layer, device)."""
    rows: dict = field(default_factory=dict)

    def _row(self, layer, dev):
        return self.rows.setdefault((layer, dev), [0, 0, 0])

    def send(self, layer, dev, bits):
        r = self._row(layer, dev)
        r[0] += bits
        r[2] += 1

    def receive(self, layer, dev, bits):
        self._row(layer, dev)[1] += bits

    def to_csv(self) -> str:
        lines = ["layer,device,bits_sent,bits_received,messages"]
        for (layer, dev), v in sorted(self.rows.items()):
            lines.append(f"{layer},{dev},{v[0]},{v[1]},{v[2]}")
        return "\n".join(lines) + "\n"


def _device_layer(cfg, blk, ranges, tokens, dev, x_local, replica, remote, causal):
    """cluster.py:176-221: one device's attention + MLP from its mixed view.

    ``remote`` maps sender -> dequantized rows (already decoded)."""
    start, stop = ranges[dev]
    x_view = np.empty((tokens, cfg.hidden), dtype=x_local.dtype)
    x_view[start:stop] = x_local
    for sender in sorted(remote):
        s, e = ranges[sender]
        x_view[s:e] = remote[sender]
    has_rep = replica is not None
    stack = np.concatenate([x_view, replica], axis=0) if has_rep else x_view
    ln1 = layer_norm(stack, blk["ln1_gain"], blk["ln1_bias"])
    k = matmul(ln1, blk["wk"])
    v = matmul(ln1, blk["wv"])
    q = matmul(ln1, blk["wq"])
    local_rows = list(range(start, stop)) + ([tokens] if has_rep else [])
    n_keys = tokens + (1 if has_rep else 0)
    mask = np.zeros((len(local_rows), n_keys), dtype=bool)
    for i, row in enumerate(local_rows):
        if row < tokens:
            mask[i, :tokens] = (np.arange(tokens) <= row) if causal else True
        else:
            mask[i, :tokens] = True
        if has_rep:
            mask[i, tokens] = True
    attn = multihead_attention(q[local_rows], k, v, mask, cfg.heads)
    h = stack[local_rows] + matmul(attn, blk["wo"])
    ln2 = layer_norm(h, blk["ln2_gain"], blk["ln2_bias"])
    mlp = matmul(gelu(matmul(ln2, blk["w1"]) + blk["b1"][None, :]), blk["w2"]) + blk["b2"][None, :]
    h = h + mlp
    n = stop - start
    return h[:n], (h[n:] if has_rep else None), k, v


@dataclass
class Result:
    output: object
    ledger: Ledger
    indices: list = field(default_factory=list)   # per layer: per device int32 [T_d, G]


def run_inference(params: Params, ranges, x, mode="classify", steps=0, cls_mode="distributed",
                  class_replication=True) -> Result:
    """cluster.py:224-308: lockstep SP inference with index exchange and ledger.

    Also records every device's VQ indices per layer (test hook)."""
    cfg = params.config
    ndev = len(ranges)
    tokens = ranges[-1][1]
    ledger = Ledger()
    if mode == "generate":
        ids = np.asarray(x, dtype=np.int64)
        if steps == 0:
            return Result([], ledger)
        x0 = params.embedding[ids] + params.pos[:ids.shape[0]]                 # model.py:283-288
    else:
        x0 = (np.asarray(x, dtype=params.pos.dtype) + params.pos[:x.shape[0]])  # model.py:275-280
    owners = []
    if not cfg.causal and class_replication:
        owners = list(range(ndev)) if cls_mode == "distributed" else [0]      # model.py:163-169
    x_local = [x0[s:e].copy() for s, e in ranges]
    reps = [params.cls.copy() if d in owners else None for d in range(ndev)]
    bits = index_bits(params.codebooks[0][0].shape[0])   # the codebook's K (vq.py:74-76)
    res = Result(None, ledger)
    dec_k, dec_v = [], []
    for layer, blk in enumerate(params.blocks):
        books = params.codebooks[layer]
        idx = [quantize(books, x_local[d]) for d in range(ndev)]                # cluster.py:272-275
        res.indices.append(idx)
        if ndev > 1:                                                            # cluster.py:144-160
            for sender in range(ndev):
                payload = idx[sender].shape[0] * len(books) * bits
                ledger.send(layer, sender, payload)
                for d in range(ndev):
                    if d != sender:
                        ledger.receive(layer, d, payload)
        outs = []
        for d in range(ndev):
            remote = {s: dequantize(books, idx[s]) for s in range(ndev) if s != d}
            outs.append(_device_layer(cfg, blk, ranges, tokens, d, x_local[d], reps[d], remote,
                                      cfg.causal))
        for d in range(ndev):
            x_local[d], reps[d] = outs[d][0], outs[d][1]
        if mode == "generate":
            dec_k.append(outs[-1][2][:tokens])
            dec_v.append(outs[-1][3][:tokens])
    if mode == "classify":                                                      # cluster.py:290-295
        r = np.concatenate([rp for rp in reps if rp is not None])
        pooled = r.mean(axis=0, keepdims=True).astype(r.dtype)                  # tensor.py:200-208
        pooled = layer_norm(pooled, params.final_gain, params.final_bias)
        res.output = matmul(pooled, params.head)
        return res
    x_last = layer_norm(x_local[-1][-1:], params.final_gain, params.final_bias)  # cluster.py:299-308
    out = [int(np.argmax(matmul(x_last, params.head)[0]))]
    kc, vc = [k.copy() for k in dec_k], [v.copy() for v in dec_v]
    for i in range(1, steps):
        out.append(_decode_one(params, kc, vc, out[-1], tokens + i - 1))
    res.output = out
    return res


def _decode_one(params, kc, vc, token, position):
    """model.py:337-358: one greedy step on the decoding device (KV cache grows)."""
    cfg = params.config
    x = params.embedding[[token]] + params.pos[position:position + 1]
    for i, blk in enumerate(params.blocks):
        ln1 = layer_norm(x, blk["ln1_gain"], blk["ln1_bias"])
        q, kn, vn = matmul(ln1, blk["wq"]), matmul(ln1, blk["wk"]), matmul(ln1, blk["wv"])
        k_all = np.concatenate([kc[i], kn], axis=0)
        v_all = np.concatenate([vc[i], vn], axis=0)
        attn = multihead_attention(q, k_all, v_all, np.ones((1, k_all.shape[0]), bool), cfg.heads)
        x = x + matmul(attn, blk["wo"])
        ln2 = layer_norm(x, blk["ln2_gain"], blk["ln2_bias"])
        x = x + (matmul(gelu(matmul(ln2, blk["w1"]) + blk["b1"][None, :]), blk["w2"])
                 + blk["b2"][None, :])
        kc[i], vc[i] = k_all, v_all
    x = layer_norm(x, params.final_gain, params.final_bias)
    return int(np.argmax(matmul(x, params.head)[0]))


def capture_block_inputs(params: Params, xs, mode="classify"):
    """train.py:160-173: single-device, unquantized block inputs per layer (for k-means)."""
    cfg = params.config
    layers = [[] for _ in params.blocks]
    for x in xs:
        if mode == "classify":
            h = np.asarray(x, F32) + params.pos[:x.shape[0]]
            c = params.cls.copy()
        else:
            ids = np.asarray(x[:-1], dtype=np.int64)
            h = params.embedding[ids] + params.pos[:ids.shape[0]]
            c = None
        t = h.shape[0]
        for i, blk in enumerate(params.blocks):
            layers[i].append(h.copy())
            stack = np.concatenate([h, c], axis=0) if c is not None else h
            ln1 = layer_norm(stack, blk["ln1_gain"], blk["ln1_bias"])
            k, v, q = matmul(ln1, blk["wk"]), matmul(ln1, blk["wv"]), matmul(ln1, blk["wq"])
            n = stack.shape[0]
            mask = np.ones((n, n), bool)
            if cfg.causal:
                mask = np.tril(mask)
            attn = multihead_attention(q, k, v, mask, cfg.heads)
            hh = stack + matmul(attn, blk["wo"])
            ln2 = layer_norm(hh, blk["ln2_gain"], blk["ln2_bias"])
            hh = hh + (matmul(gelu(matmul(ln2, blk["w1"]) + blk["b1"][None, :]), blk["w2"])
                       + blk["b2"][None, :])
            h = hh[:t]
            c = hh[t:] if c is not None else None
    return [np.concatenate(xs_, axis=0) for xs_ in layers]


def initialize_codebooks(params: Params, xs, mode="classify", seed=0, iterations=25):
    """train.py:176-189 (centroids only)."""
    cfg = params.config
    caps = capture_block_inputs(params, xs, mode)
    params.codebooks = [kmeans_init(x, cfg.codebook_size, cfg.groups, iterations, seed, layer_id=i)
                        for i, x in enumerate(caps)]
    return params


def pack_indices(idx: np.ndarray, bits: int) -> np.ndarray:
    """Wire format of the exchange: LSB-first bitstream of ``bits``-bit
    codes, padded to whole u32 words.  (The reference only counts these bits,
    cluster.py:154-158; this is the CPU restatement of the packed payload.)"""
    flat = np.asarray(idx, dtype=np.uint64).reshape(-1)
    nwords = (flat.size * bits + 31) // 32
    words = np.zeros(nwords + 1, dtype=np.uint64)
    for i, v in enumerate(flat):
        bit = i * bits
        w, off = divmod(bit, 32)
        words[w] |= (int(v) << off) & 0xFFFFFFFF
        if off + bits > 32:
            words[w + 1] |= int(v) >> (32 - off)
    return words[:nwords].astype(np.uint32)
