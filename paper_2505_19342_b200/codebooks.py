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

from .model import generator
from .vq import Codebook


def capture_block_inputs(params, xs: np.ndarray, device=None) -> list[torch.Tensor]:
    """Per-layer block inputs (content rows) of a single-device unquantized forward."""
    from .cluster import partition_tokens
    from .runtime import AstraRuntime
    xs = np.asarray(xs, dtype=np.float32)
    plan = partition_tokens(xs.shape[1], 1)
    rt = AstraRuntime(params, plan, batch=xs.shape[0], precision="parity", device=device,
                      encode_at_one_device=False, require_codebooks=False)
    rt.capture_inputs = []
    rt.classify_numpy(xs)
    return rt.capture_inputs


def _lloyd(pts: torch.Tensor, k: int, iterations: int, gen: np.random.Generator) -> torch.Tensor:
    m = pts.shape[0]
    cents = pts[torch.from_numpy(gen.choice(m, size=k, replace=False)).to(pts.device)].clone()
    pp = (pts * pts).sum(1, keepdim=True)
    ar = torch.arange(k, device=pts.device)
    for _ in range(max(1, iterations)):
        d2 = pp - 2.0 * (pts @ cents.T) + (cents * cents).sum(1)[None, :]
        assign = d2.argmin(1)
        dist2 = ((pts - cents[assign]) ** 2).sum(1)
        counts = torch.bincount(assign, minlength=k)
        empty = ar[counts == 0].tolist()
        reseeded = bool(empty)
        for idx in empty:
            far = int(dist2.argmax())
            cents[idx] = pts[far]
            assign[far] = idx
            dist2[far] = 0.0
        counts = torch.bincount(assign, minlength=k)
        sums = torch.zeros_like(cents).index_add_(0, assign, pts)
        new = torch.where(counts[:, None] > 0, sums / counts.clamp(min=1)[:, None].double(), cents)
        if not reseeded and torch.equal(new, cents):
            break
        cents = new
    return cents


def fit_codebooks(params, xs: np.ndarray, codebook_size: int | None = None,
                  groups: int | None = None, seed: int = 0, iterations: int = 25,
                  device=None) -> list[Codebook]:
    """Fit and attach per-layer codebooks to ``params`` (in place); returns them."""
    cfg = params.config
    k = codebook_size or cfg.codebook_size
    g_count = groups or cfg.groups
    caps = capture_block_inputs(params, xs, device=device)
    books = []
    for layer, x in enumerate(caps):
        x64 = x.double()
        gd = x64.shape[1] // g_count
        tables = []
        for g in range(g_count):
            c = _lloyd(x64[:, g * gd:(g + 1) * gd].contiguous(), k, iterations,
                       generator(seed, "kmeans", layer, g))
            tables.append(c.float().cpu().numpy())
        cb = Codebook(layer_id=layer, groups=g_count, centroids=tables)
        params.blocks[layer].codebook = cb
        books.append(cb)
    return books
