"""Codebook fitting on the GPU (setup, not on the timed path).

Follows the reference's initialize_codebooks (train.py:160-189): capture every
layer's block input from an unquantized single-device forward over a few
synthetic sequences, then Lloyd's k-means per layer and group (vq.py:134-204:
random distinct initial points from the named stream ("kmeans", layer, g),
fp64 assignment with lowest-index ties, farthest-point reseeding of empty
clusters, stop when centroids are unchanged).  The forward capture runs through
AstraRuntime; Lloyd runs in fp64 on the device.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .errors import ShapeError
from .model import generator
from .vq import Codebook


def capture_block_inputs(params, xs, device=None, mode: str = "classify") -> list[torch.Tensor]:
    """Per-layer block inputs (content rows) of a single-device unquantized forward over a
    batch: classify inputs [n, T, D] fp32, or token-id sequences [n, T] for mode="lm"
    (train.py:160-173 runs classify / lm_logits with an on_layer capture)."""
    from .cluster import partition_tokens
    from .runtime import AstraRuntime
    if mode == "lm":
        ids = np.asarray(xs, dtype=np.int64)
        rt = AstraRuntime(params, partition_tokens(ids.shape[1], 1, class_replication=False),
                          batch=ids.shape[0], mode="lm", precision="parity", device=device,
                          encode_at_one_device=False, require_codebooks=False)
        rt.capture_inputs = []
        rt.set_ids(ids)
        rt.forward()
        torch.cuda.synchronize()
        return rt.capture_inputs
    xs = np.asarray(xs, dtype=np.float32)
    plan = partition_tokens(xs.shape[1], 1)
    rt = AstraRuntime(params, plan, batch=xs.shape[0], precision="parity", device=device,
                      encode_at_one_device=False, require_codebooks=False)
    rt.capture_inputs = []
    rt.classify_numpy(xs)
    return rt.capture_inputs


def _nearest64(pts: torch.Tensor, cents: torch.Tensor) -> torch.Tensor:
    """vq._nearest (vq.py:126-131) in fp64 on the GPU: (|p|^2 - 2 p.c) + |c|^2, first index
    on ties.  The dot products go through cuBLAS DGEMM, whose summation order differs from
    the host BLAS only at the 1e-16 level."""
    d2 = (pts * pts).sum(1, keepdim=True) - 2.0 * (pts @ cents.T) + (cents * cents).sum(1)[None, :]
    return d2.argmin(1)


def _segment_mean(pts: torch.Tensor, assign: torch.Tensor, k: int, mean: torch.Tensor,
                  sums: torch.Tensor | None = None) -> torch.Tensor:
    """Per-cluster fp64 mean in ascending sample order (astra_segment_mean_f64): the same
    rounding as NumPy's ``pts[assign == c].mean(axis=0)``; empty clusters keep ``mean``."""
    order = torch.sort(assign, stable=True).indices.to(torch.int32)
    counts = torch.bincount(assign, minlength=k)
    seg = torch.zeros(k + 1, dtype=torch.int32, device=pts.device)
    seg[1:] = torch.cumsum(counts, 0).to(torch.int32)
    _native.call("astra_segment_mean_f64", pts.data_ptr(), pts.stride(0), order.data_ptr(),
                 seg.data_ptr(), k, pts.shape[1], mean.data_ptr(),
                 None if sums is None else sums.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return counts


def _lloyd(pts: torch.Tensor, k: int, iterations: int, gen: np.random.Generator) -> torch.Tensor:
    """vq._lloyd (vq.py:134-166) on the GPU, deterministic: the same initial draw, fp64
    assignment, the reference's sequential farthest-point reseed (a reseed can empty a later
    cluster, which the loop then reseeds too), NumPy-order means, stop when unchanged."""
    m = pts.shape[0]
    cents = pts[torch.from_numpy(gen.choice(m, size=k, replace=False)).to(pts.device)].clone()
    for _ in range(max(1, iterations)):
        assign = _nearest64(pts, cents)
        counts = torch.bincount(assign, minlength=k)
        reseeded = bool((counts == 0).any())
        if reseeded:
            # rare: replay the reference's loop on the host, with its own dist2 expression
            p_h, c_h = pts.cpu().numpy(), cents.cpu().numpy()
            a_h = assign.cpu().numpy().copy()
            dist2 = ((p_h - c_h[a_h]) ** 2).sum(axis=1)
            for idx in range(k):
                if not (a_h == idx).any():
                    far = int(np.argmax(dist2))
                    c_h[idx] = p_h[far]
                    a_h[far] = idx
                    dist2[far] = 0.0
            cents = torch.from_numpy(c_h).to(pts.device)
            assign = torch.from_numpy(a_h).to(pts.device)
        new = cents.clone()
        _segment_mean(pts, assign, k, new)
        if not reseeded and torch.equal(new, cents):
            break
        cents = new
    return cents


def kmeans_init(x: torch.Tensor, codebook_size: int, groups: int, iterations: int = 25,
                seed: int = 0, layer_id: int = 0) -> Codebook:
    """vq.kmeans_init (vq.py:169-204) on device-resident [M, D] samples: per group, Lloyd
    from the named stream ("kmeans", layer, g), then the EMA state of the final assignment
    (counts, per-cluster fp64 sums in the reference's np.add.at order)."""
    if x.dim() != 2:
        raise ShapeError("kmeans_init expects [M, D] embeddings")
    m, d = x.shape
    if m < codebook_size:
        raise ValueError(f"need at least K={codebook_size} samples, got {m}")
    if d % groups != 0:
        raise ShapeError(f"width {d} is not divisible by {groups} groups")
    gd = d // groups
    x64 = x.double()
    tables, counts, sums = [], [], []
    for g in range(groups):
        pts = x64[:, g * gd:(g + 1) * gd].contiguous()
        c = _lloyd(pts, codebook_size, iterations, generator(seed, "kmeans", layer_id, g))
        assign = _nearest64(pts, c)
        gsum = torch.zeros(codebook_size, gd, dtype=torch.float64, device=x.device)
        cnt = _segment_mean(pts, assign, codebook_size, torch.empty_like(gsum), sums=gsum)
        tables.append(c.float().cpu().numpy())
        counts.append(cnt.double().cpu().numpy())
        sums.append(gsum.cpu().numpy())
    return Codebook(layer_id=layer_id, groups=groups, centroids=tables,
                    ema_counts=np.stack(counts), ema_sums=sums)


def fit_codebooks(params, xs: np.ndarray, codebook_size: int | None = None,
                  groups: int | None = None, seed: int = 0, iterations: int = 25,
                  device=None, mode: str = "classify") -> list[Codebook]:
    """initialize_codebooks (train.py:176-189) on the GPU: capture, then deterministic
    per-layer k-means; attaches the books to ``params`` (in place) and returns them."""
    cfg = params.config
    k = codebook_size or cfg.codebook_size
    g_count = groups or cfg.groups
    for b in params.blocks:
        b.codebook = None          # capture is the unquantized single-device forward
    caps = capture_block_inputs(params, xs, device=device, mode=mode)
    books = []
    for layer, x in enumerate(caps):
        cb = kmeans_init(x, k, g_count, iterations=iterations, seed=seed, layer_id=layer)
        params.blocks[layer].codebook = cb
        books.append(cb)
    return books


def initialize_codebooks(params, dataset, task: str, codebook_size: int, groups: int,
                         seed: int = 0, iterations: int = 25) -> None:
    """Drop-in for train.initialize_codebooks (train.py:176-189): ``dataset`` is the reference's
    ``(inputs, labels)`` pair for ``task="classify"`` or its list of token-id sequences for
    ``task="lm"`` (captured on ``ids[:-1]``, train.py:160-173); per-layer codebooks are fitted
    on the GPU (fit_codebooks) and attached in place.  The training-side residual statistics
    the reference also fits (fit_residual_stats, for NAVQ noise) are out of scope."""
    if task == "classify":
        xs, mode = np.asarray(dataset[0], dtype=np.float32), "classify"
    elif task == "lm":
        xs, mode = np.stack([np.asarray(s)[:-1] for s in dataset]), "lm"
    else:
        raise ValueError(f"unknown task {task!r}")
    fit_codebooks(params, xs, codebook_size, groups, seed=seed, iterations=iterations, mode=mode)


def load_codebook_tables(path, params=None) -> list[Codebook]:
    """Codebooks from a centroid archive ``{centroids: fp32 [L, G, K, D/G],
    centroids_sha256}`` — e.g. tests/golden/vitb16_codebooks.npz, the reference's own
    initialize_codebooks output (train.py:176-189) written by make_golden_vitb.py.  The
    SHA-256 of the centroid bytes is verified; with ``params`` the books are attached."""
    import hashlib
    with np.load(path) as z:
        cents = np.ascontiguousarray(z["centroids"], dtype=np.float32)
        want = str(z["centroids_sha256"]) if "centroids_sha256" in z else None
    if want is not None and hashlib.sha256(cents.tobytes()).hexdigest() != want:
        raise ValueError(f"{path}: centroid checksum mismatch")
    books = [Codebook(layer_id=i, groups=cents.shape[1], centroids=[c.copy() for c in cents[i]])
             for i in range(cents.shape[0])]
    if params is not None:
        if len(params.blocks) != len(books):
            raise ShapeError(f"{len(books)} codebooks for {len(params.blocks)} layers")
        for b, cb in zip(params.blocks, books):
            b.codebook = cb
    return books
