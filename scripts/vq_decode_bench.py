"""Standalone VQ decode microbenchmark (SURVEY 8d / BASELINE config #5): device time of

  astra_vq_decode            codes -> fp32 rows (vq.dequantize, vq.py:225-233)
  astra_vq_decode_layernorm  codes -> LN1(rows) as the K|V projection's bf16 operand (fast: hi;
                             parity: hi + lo), the decode fused into LN1

on the token counts of the bench workloads, CUDA events over `--reps` back-to-back launches
after warm-up.  Bytes per launch: HBM-visible = codes read + output written (the codebook,
G*K*gd*4 bytes, is L2-resident); gathered = the codebook rows read through L2.  GB/s is the
HBM-visible figure against MEASURED_PEAKS' HBM copy bandwidth.  One JSON line per case.

    python scripts/vq_decode_bench.py [--reps 50]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_19342_b200 import _native  # noqa: E402
from paper_2505_19342_b200.vq import DeviceCodebook  # noqa: E402

CASES = [  # (name, tokens M, D, G, K)
    ("vitl_g16_k1024", 32 * 576, 1024, 16, 1024),
    ("vitl_g16_k4096", 32 * 576, 1024, 16, 4096),
    ("vitl_g32_k256", 32 * 576, 1024, 32, 256),
    ("vitb_g16_k1024", 64 * 196, 768, 16, 1024),
    ("vitb_g1_k1024", 64 * 196, 768, 1, 1024),
    ("gpt2m_g16_k1024", 2 * 4096, 1024, 16, 1024),
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    peaks = bench._peaks()
    lib = _native.load()
    del lib
    rng = np.random.default_rng(0)
    st = torch.cuda.current_stream().cuda_stream
    for name, m, d, g, k in CASES:
        gd = d // g
        cb = DeviceCodebook(torch.from_numpy(rng.normal(size=(g, k, gd)).astype(np.float32)).to(dev))
        idx = torch.from_numpy(rng.integers(0, k, size=(m, g)).astype(np.int32)).to(dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        out = torch.empty(m, d, dtype=torch.float32, device=dev)
        hi = torch.empty(m, d, dtype=torch.bfloat16, device=dev)
        lo = torch.empty_like(hi)
        gain = torch.ones(d, device=dev)
        bias = torch.zeros(d, device=dev)
        ref = ctypes.byref(cb.struct)
        res = {"case": name, "tokens": m, "D": d, "G": g, "K": k,
               "codebook_MB": round(g * k * gd * 4 / 1e6, 2), "hbm_peak_gbs": peaks["hbm"]}
        variants = {
            "decode_f32": (lambda: _native.call("astra_vq_decode", ref, idx.data_ptr(), m,
                                                out.data_ptr(), d, err.data_ptr(), st), 4),
            "decode_ln_bf16": (lambda: _native.call("astra_vq_decode_layernorm", ref, idx.data_ptr(),
                                                    m, gain.data_ptr(), bias.data_ptr(), 1e-5,
                                                    hi.data_ptr(), None, d, err.data_ptr(), st), 2),
            "decode_ln_bf16x2": (lambda: _native.call("astra_vq_decode_layernorm", ref,
                                                      idx.data_ptr(), m, gain.data_ptr(),
                                                      bias.data_ptr(), 1e-5, hi.data_ptr(),
                                                      lo.data_ptr(), d, err.data_ptr(), st), 4),
        }
        if d not in (512, 768, 1024):
            variants = {"decode_f32": variants["decode_f32"]}
        for vname, (fn, out_bytes) in variants.items():
            t = timed(fn, a.reps)
            hbm = m * g * 4 + m * d * out_bytes
            gathered = m * d * 4
            res[vname] = {"us": round(t * 1e6, 2), "hbm_bytes": hbm,
                          "gbs": round(hbm / t / 1e9, 1),
                          "frac": round(hbm / t / 1e9 / peaks["hbm"], 3),
                          "gathered_gbs": round(gathered / t / 1e9, 1)}
        assert int(err.item()) == 0
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
