import sys, math, numpy as np, torch
sys.path.insert(0, '.')
from tests.test_attention_gpu import _problem, _reference
from paper_2505_19342_b200 import _native
heads, dk = 12, 64
for causal in (False,):
  for factor in (8.0, 20.0, 60.0):
    spec = [(197, 197, 1), (50, 300, 0)]
    qkv, table, segs_t, ks, kp, segs = _problem(11, spec, heads, dk, causal)
    D = heads * dk
    srcs = ks.cpu().numpy()
    for q0, nq, _, _, k0, nk in segs:
        for j in (100, nk - 40):
            r = int(srcs[k0 + j])
            if r < 0: table[-r - 1, :D] *= factor
            else: qkv[r, D:2 * D] *= factor
    ref = _reference(qkv, table, segs, ks, kp, heads, dk, causal)
    lib = _native.load()
    for v in (0, 2):
        lib.astra_attention_variant(v)
        out = torch.zeros(qkv.shape[0], D, dtype=torch.bfloat16, device="cuda")
        es = qkv.element_size()
        _native.call("astra_attention", qkv.data_ptr(), 3 * D, qkv.data_ptr() + D * es, qkv.data_ptr() + 2 * D * es, 3 * D, table.data_ptr(), table.data_ptr() + D * es, 2 * D, ks.data_ptr(), kp.data_ptr(), segs_t.data_ptr(), len(segs), max(s[1] for s in segs), heads, dk, int(causal), 1, float(np.float32(1 / math.sqrt(dk))), None, out.data_ptr(), None, D, qkv.shape[0], qkv.shape[0], table.shape[0], torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        rows = torch.cat([torch.arange(s[0], s[0] + s[1]) for s in segs]).cuda()
        o = out.float()[rows]
        bad = ~torch.isfinite(o)
        br = bad.any(1).nonzero().flatten().tolist()
        bh = sorted(set((bad.nonzero()[:,1] // 64).tolist()))
        err = (o - ref[rows]).abs().nan_to_num(0).max().item()
        print(f"causal={causal} factor={factor} variant={v}: nonfinite rows {len(br)} {br[:8]} heads {bh} err {err:.3g} ref finite {torch.isfinite(ref[rows]).all().item()}")
    lib.astra_attention_variant(0)
