"""Deterministic golden-case inputs shared by make_golden.py and the tests."""

import numpy as np


def vq_case_inputs(i, k, d, g, m):
    """Deterministic inputs of VQ case i (regenerated identically by the tests)."""
    rng = np.random.default_rng(20251017 + i)
    gd = d // g
    cents = [rng.normal(size=(k, gd)).astype(np.float32) for _ in range(g)]
    x = rng.normal(size=(m, d)).astype(np.float32)
    if i >= 3:  # duplicate a centroid and plant tokens on it: exact ties
        cents[0][5] = cents[0][2]
        x[:5] = np.concatenate(cents, axis=1)[2] + 0.0
    return cents, x


VQ_CASES = [(3, 4, 1, 40), (64, 8, 2, 40), (17, 9, 3, 40), (1024, 768, 1, 300),
            (256, 768, 16, 200), (4096, 64, 1, 150), (1024, 768, 32, 100), (2, 2, 1, 3)]


ATT_CASES = [(7, 7, 8, 1, 0.7), (7, 7, 8, 2, 0.7), (50, 197, 768, 12, 1.0), (30, 61, 64, 4, 0.5),
             (16, 16, 32, 4, -1)]


def att_case_inputs(i, r, c, d, p):
    rng = np.random.default_rng(4242 + i)
    q = rng.normal(size=(r, d)).astype(np.float32)
    k = rng.normal(size=(c, d)).astype(np.float32)
    v = rng.normal(size=(c, d)).astype(np.float32)
    if p < 0:
        mask = np.tril(np.ones((r, c), bool))
    else:
        mask = rng.random((r, c)) < p
        mask[:, 0] = True
    return q, k, v, mask
