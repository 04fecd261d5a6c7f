"""Standalone kernel microbenchmarks (BASELINE config #5): one JSON line per case.

  vq_encode   astra_vq_encode (split + bf16x3 distance GEMM + decision + fp64 re-rank) on random
              clustered rows, back-to-back launches; algorithmic 2*M*K*D FLOP against a third of
              the measured bf16 peak (three MMAs per MAC for exact indices)
  attention   the runtime's own astra_attention call (ViT-B/16 B=64, layer-0 arguments) for one
              rank of an N-way split (loopback exchange), back-to-back launches; algorithmic
              Q/K/V read + O write bytes against the measured HBM copy bandwidth

    python scripts/microbench.py [--reps 30] [--only vq|attention]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2505_19342_b200 import _native, cluster, data, model, vq  # noqa: E402
from paper_2505_19342_b200.runtime import AstraRuntime, LoopbackExchange  # noqa: E402

VQ_CASES = [  # name, tokens M, D, G, K
    ("vitb_g1_k1024", 64 * 196, 768, 1, 1024),
    ("vitl_g1_k1024", 32 * 576, 1024, 1, 1024),
    ("vitl_g1_k4096", 32 * 576, 1024, 1, 4096),
    ("vitl_g16_k1024", 32 * 576, 1024, 16, 1024),
    ("vitl_g32_k1024", 32 * 576, 1024, 32, 1024),
    ("gpt2m_g1_k1024", 2 * 4096, 1024, 1, 1024),
]


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1000.0


def vq_cases(reps, peaks, dev):
    rng = np.random.default_rng(0)
    for name, m, d, g, k in VQ_CASES:
        gd = d // g
        centers = rng.normal(size=(k, d)).astype(np.float32)
        cb = vq.DeviceCodebook(torch.from_numpy(
            np.ascontiguousarray(centers.reshape(k, g, gd).transpose(1, 0, 2))).to(dev))
        # tokens near the codes (the regime the error window is built for)
        x = torch.from_numpy((centers[rng.integers(0, k, m)] +
                              0.3 * rng.normal(size=(m, d))).astype(np.float32)).to(dev)
        out = torch.empty(m, g, dtype=torch.int32, device=dev)
        ws = torch.empty(max(cb.workspace_bytes(m), 1), dtype=torch.uint8, device=dev)
        t = timed(lambda: cb.encode(x, out=out, workspace=ws), reps)
        flops = 2.0 * m * k * d
        peak = peaks["bf16"] / 3.0
        print(json.dumps({"kernel": "vq_encode", "case": name, "tokens": m, "D": d, "G": g, "K": k,
                          "us": round(t * 1e6, 2), "tflops": round(flops / t / 1e12, 1),
                          "peak_tflops": round(peak, 1), "frac": round(flops / t / 1e12 / peak, 3),
                          "peak_source": f"{peaks['src']} bf16 burst / 3"}), flush=True)


def attention_cases(reps, peaks, dev):
    cfg = model.ModelConfig(layers=1, hidden=768, heads=12, vocab_or_classes=1000, max_tokens=197,
                            causal=False, codebook_size=1024, groups=1)
    params = model.init_params(cfg, seed=0)
    xs = data.make_classify_batch(768, 196, 64, seed=1)
    rng = np.random.default_rng(0)
    for i, b in enumerate(params.blocks):
        c = xs.reshape(-1, 768)[rng.choice(64 * 196, 1024, replace=False)]
        b.codebook = vq.Codebook(layer_id=i, groups=1, centroids=[c])
    lib = _native.load()
    for n in (1, 2, 4, 8):
        comm = LoopbackExchange(n - 1, n) if n > 1 else None
        rt = AstraRuntime(params, cluster.partition_tokens(196, n), batch=64, precision="fast",
                          comm=comm)
        rt.stage_input(xs)
        calls = []
        orig = _native.call

        def spy(name, *args):
            if name == "astra_attention":
                calls.append(args)
            return orig(name, *args)

        _native.call = spy
        try:
            rt.forward()
            torch.cuda.synchronize()
        finally:
            _native.call = orig
        args = calls[0]
        t = timed(lambda: lib.astra_attention(*args), reps)
        w = bench._kernel_work(rt)["attention"]
        gbs = w["bytes"] / t / 1e9
        print(json.dumps({"kernel": "attention", "case": f"vitb_b64_rank_of_{n}", "n": n,
                          "query_rows": int(rt.R), "us": round(t * 1e6, 2),
                          "gbs": round(gbs, 1), "tflops": round(w["flops"] / t / 1e12, 1),
                          "frac_hbm": round(gbs / peaks["hbm"], 3),
                          "peak_source": f"{peaks['src']} HBM copy"}), flush=True)
        del rt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--only", choices=["vq", "attention"], default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    peaks = bench._peaks()
    if a.only != "attention":
        vq_cases(a.reps, peaks, dev)
    if a.only != "vq":
        attention_cases(a.reps, peaks, dev)


if __name__ == "__main__":
    main()
