"""Synthetic inputs of the reference benchmarks (train.py:66-90), bit-identical:
rank-2 cluster samples lifted into D dimensions.  Host-side NumPy (setup, not timed)."""

from __future__ import annotations

import math

import numpy as np

from .model import generator

_ANCHORS = np.array([[1.5, 1.5], [1.5, -1.5], [-1.5, 1.5], [-1.5, -1.5]])


def make_classify_data(dim: int, tokens: int, count: int, seed: int, spread: float = 0.3,
                       signal_fraction: float = 0.25, task_seed: int = 0):
    """train.py:66-90: returns (list of [tokens, dim] fp32 arrays, int64 labels)."""
    gen = generator(seed, "classify-data")
    lift = generator(task_seed, "classify-lift").normal(size=(2, dim)) / math.sqrt(2.0)
    signal_count = max(1, round(tokens * signal_fraction))
    inputs, labels = [], []
    for _ in range(count):
        label = int(gen.integers(0, len(_ANCHORS)))
        pts = gen.normal(size=(tokens, 2)) * spread
        where = gen.choice(tokens, size=signal_count, replace=False)
        pts[where] += _ANCHORS[label]
        inputs.append((pts @ lift).astype(np.float32))
        labels.append(label)
    return inputs, np.asarray(labels, dtype=np.int64)


def make_classify_batch(dim: int, tokens: int, count: int, seed: int, task_seed: int = 0):
    """[count, tokens, dim] fp32 stack of make_classify_data (vectorised lift)."""
    xs, _ = make_classify_data(dim, tokens, count, seed, task_seed=task_seed)
    return np.stack(xs)
