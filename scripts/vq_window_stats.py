"""Diagnostic: how many VQ codes fall inside the bf16x3 error window, per layer, with and without
centring the group vectors on the codebook mean.  Usage: python scripts/vq_window_stats.py
[--config vitl --groups 16 --codebook 1024 --layers 0,6,12,23].  Prints one JSON line per layer."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_19342_b200 import codebooks  # noqa: E402

TAU = 2.0 ** -14


def window_stats(x, c):
    """x [M, gd], c [K, gd] fp64 -> dict of window candidate statistics."""
    d = (x * x).sum(1, keepdim=True) - 2 * x @ c.T + (c * c).sum(1)[None]
    best = d.min(1).values
    out = {}
    for name, mu in (("raw", torch.zeros_like(c[0])), ("centred", c.mean(0))):
        xn = (x - mu).norm(dim=1, keepdim=True)
        cn = (c - mu).norm(dim=1)[None]
        win = 2 * TAU * xn * cn            # per-code bound D_k (dominant term)
        bi = d.argmin(1, keepdim=True)
        dbest = torch.gather(win, 1, bi)
        cand = (d - win <= best[:, None] + dbest).sum(1).double()
        out[name] = {"cands_per_token": round(cand.mean().item(), 4),
                     "multi_rate": round((cand > 1).double().mean().item(), 5),
                     "max_cands": int(cand.max().item()), "over8": int((cand > 8).sum().item()),
                     "over4": int((cand > 4).sum().item()),
                     "xnorm": round(xn.mean().item(), 3), "cnorm": round(cn.mean().item(), 3)}
    dup = (torch.cdist(c, c) == 0).sum().item() - c.shape[0]
    out["duplicate_code_pairs"] = dup // 2
    s = d.sort(1).values
    out["gap12_median"] = round((s[:, 1] - s[:, 0]).median().item(), 5)
    out["best_d2_median"] = round(best.median().item() + 0.0, 3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="vitl")
    ap.add_argument("--groups", type=int, default=16)
    ap.add_argument("--codebook", type=int, default=1024)
    ap.add_argument("--layers", default="0,1,6,12,23")
    ap.add_argument("--images", type=int, default=8)
    a = ap.parse_args()
    w = bench.WORKLOADS[a.config]
    import dataclasses
    w = dataclasses.replace(w, G=a.groups, K=a.codebook)
    dev = torch.device("cuda", 0)
    params, xs, _ = bench._setup_params(w, device=dev)
    xs = np.asarray(xs)[:a.images]
    caps = codebooks.capture_block_inputs(params, xs, device=dev,
                                          mode="lm" if w.kind == "prefill" else "classify")
    for l in [int(v) for v in a.layers.split(",") if int(v) < w.L]:
        x = caps[l].double()
        cb = params.blocks[l].codebook
        gd = w.D // w.G
        per = []
        for g in range(w.G):
            c = torch.from_numpy(np.asarray(cb.centroids[g], np.float64)).to(dev)
            per.append(window_stats(x[:, g * gd:(g + 1) * gd], c))
        agg = {k: {kk: (float(np.max([p[k][kk] for p in per])) if kk == "max_cands" else
                        float(np.sum([p[k][kk] for p in per])) if kk.startswith("over") else
                        float(np.mean([p[k][kk] for p in per]))) for kk in per[0][k]}
               for k in ("raw", "centred")}
        agg["duplicate_code_pairs"] = int(sum(p["duplicate_code_pairs"] for p in per))
        agg["gap12_median"] = float(np.mean([p["gap12_median"] for p in per]))
        agg["best_d2_median"] = float(np.mean([p["best_d2_median"] for p in per]))
        print(json.dumps({"layer": l, "G": w.G, "K": w.K, **agg}), flush=True)


if __name__ == "__main__":
    main()
