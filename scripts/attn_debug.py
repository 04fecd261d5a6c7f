"""Isolate attention kernel mismatches: run several single-spec problems, print max error."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tests.test_attention_gpu import _problem, _reference  # noqa: E402
from paper_2505_19342_b200 import _native  # noqa: E402

lib = _native.load()
heads, dk = 12, 64
D = heads * dk
for spec in [[(130, 300, 0)], [(128, 300, 0)], [(64, 300, 0)], [(64, 256, 0)], [(64, 257, 0)],
             [(7, 7, 0)], [(130, 300, 0), (7, 7, 0)], [(130, 200, 0)], [(200, 600, 1)]]:
    for causal in (False,):
        qkv, table, segs_t, ks, kp, segs = _problem(3, spec, heads, dk, causal)
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
        ref = _reference(qkv, table, segs, ks, kp, heads, dk, causal)
        errs = []
        for s in segs:
            e = (out.float()[s[0]:s[0] + s[1]] - ref[s[0]:s[0] + s[1]]).abs()
            errs.append(round(e.max().item(), 4))
            # per q-tile / per head detail for the first segment
        e0 = (out.float()[segs[0][0]:segs[0][0] + segs[0][1]] - ref[segs[0][0]:segs[0][0] + segs[0][1]]).abs()
        bad_rows = (e0.max(1).values > 0.02).nonzero().flatten().tolist()
        bad_heads = sorted({c // dk for c in (e0.max(0).values > 0.02).nonzero().flatten().tolist()})
        print(spec, causal, errs, "bad rows", bad_rows[:5], len(bad_rows), "bad heads", bad_heads)
