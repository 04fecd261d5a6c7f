"""Host-side sequence-parallel layout (pure NumPy; shared by every rank and by tests).

For the devices of a ShardPlan that live on this GPU (all of them for "virtual devices",
one per rank under torch.distributed) this computes, once, every index array the
kernels consume:

* stack rows: per (device v, image b) the T_v content rows then the class replica
  (if v owns one, model.py:163-169) — the residual stream layout;
* embed maps: stack row -> input row (b*T + global position) and position row;
* attention segments [q0, nq, qpos0, ncontent, k0, nk] per (v, b) and the key map: a
  device's own keys are local stack rows; every other token t of the image is
  -(global content index + 1), resolved per layer to the codebook K/V table row of the
  received code (G = 1) or to a decoded K^/V^ row (G > 1) — the x_view of
  cluster.py:182-194;
* global content numbering (e, b, r) -> gofs[e] + b*T_e + r, which is also the order of
  the exchanged payloads (sender-major, cluster.py:152).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SPLayout:
    rows: int                    # stack rows on this GPU
    content_rows: np.ndarray     # stack row of each local content token, (v, b, r) order
    row_src: np.ndarray          # embed: input row (b*T + pos) or -1 for a replica
    row_pos: np.ndarray          # embed: position row
    segs: np.ndarray             # [S, 6] attention segments
    key_map: np.ndarray          # per segment key list (see module doc)
    key_pos: np.ndarray          # global token position per key (-1: replica key)
    rep_rows: np.ndarray         # stack rows of local class replicas, (v, b) order
    row_base: dict               # (v, b) -> first stack row
    gofs: np.ndarray             # global content offset per device (+ total at the end)


def sp_layout(tokens: int, ranges, batch: int, local: list[int], owners: list[int]) -> SPLayout:
    T, B = tokens, batch
    sizes = [e - s for s, e in ranges]
    starts = [s for s, _ in ranges]
    owner = np.empty(T, dtype=np.int64)
    for d, (s, e) in enumerate(ranges):
        owner[s:e] = d
    gofs = np.concatenate([[0], np.cumsum([B * s for s in sizes])]).astype(np.int64)
    rows = 0
    content, row_src, row_pos, segs, key_map, key_pos, rep_rows = [], [], [], [], [], [], []
    row_base = {}
    for v in local:
        rep = 1 if v in owners else 0
        for b in range(B):
            base = rows
            row_base[(v, b)] = base
            for r in range(sizes[v]):
                content.append(base + r)
                row_src.append(b * T + starts[v] + r)
                row_pos.append(starts[v] + r)
            if rep:
                row_src.append(-1)
                row_pos.append(0)
                rep_rows.append(base + sizes[v])
            k0 = len(key_map)
            for j in range(T):
                e = int(owner[j])
                if e == v:
                    key_map.append(base + j - starts[v])
                else:
                    key_map.append(-int(gofs[e] + b * sizes[e] + (j - starts[e]) + 1))
                key_pos.append(j)
            if rep:
                key_map.append(base + sizes[v])
                key_pos.append(-1)
            segs.append([base, sizes[v] + rep, starts[v], sizes[v], k0, T + rep])
            rows += sizes[v] + rep
    i32 = lambda a: np.asarray(a, dtype=np.int32)  # noqa: E731
    return SPLayout(rows=rows, content_rows=i32(content), row_src=i32(row_src),
                    row_pos=i32(row_pos), segs=i32(segs).reshape(-1, 6), key_map=i32(key_map),
                    key_pos=i32(key_pos), rep_rows=i32(rep_rows), row_base=row_base, gofs=gofs)


def resolve_keys(key_map: np.ndarray, codes_all: np.ndarray | None) -> np.ndarray:
    """Host restatement of astra_key_map: remote keys -> -(code + 1) (G = 1) or unchanged."""
    if codes_all is None:
        return key_map.copy()
    out = key_map.copy()
    rem = key_map < 0
    out[rem] = -(codes_all[-(key_map[rem] + 1)] + 1)
    return out
