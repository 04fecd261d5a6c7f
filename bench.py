"""Benchmark: Astra Mixed-Precision-Attention inference on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--config vitb|vitl|gpt2s|gpt2m] [--groups G] [--codebook K]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one rank per GPU, NCCL)

Default workload (BASELINE.json configs[1]): ViT-B/16 shape (L=12, D=768, H=12, MLP 3072, no
patch embedding — inputs are [196, 768] token embeddings like the reference), batch 64,
token sequence split across N GPUs (N=1 default), VQ codebook K=1024, G=1, distributed
class tokens.  Weights: the reference's seeded init_params(seed=0); codebooks: the
reference's OWN initialize_codebooks output (tests/golden/vitb16_codebooks.npz, written by
seqvq in tests/golden/make_golden_vitb.py); inputs: make_classify_data(seed=1).  A step =
one full forward of the 64-image batch.  Both precision modes are measured; the line's
`parity` blocks compare each with the reference's own logits / VQ indices for the same 64
images at the same N (tests/golden/golden_vitb.npz).

Other BASELINE configs (one JSON line per invocation):
  --config vitl   ViT-L/16@384 (L=24, D=1024, H=16, T=576, B=32), --groups / --codebook sweep
                  (config #4; scripts/sweep_vitl.sh runs G in {1,16,32} x K in {256,1024,4096})
  --config gpt2s  GPT-2-small shape causal prefill, T=1024, B=8 sequences (config #3)
  --config gpt2m  GPT-2-medium shape causal prefill, T=4096, B=2 sequences (config #5)
Their codebooks are fitted on the GPU with the reference recipe (train.py:176-189:
unquantized capture, deterministic Lloyd k-means identical to vq._lloyd) and handed
unchanged to the CPU oracle, which runs the same samples as the CPU baseline and checker.

Prints ONE JSON line (rank 0).  `value` is the metric with inputs resident in HBM (CUDA graph
replay, device-timed, max over ranks); `e2e` is the same metric through the public runtime
API with the host->device input copy and device->host result read inside every step;
`roofline` is the dominant kernel vs MEASURED_PEAKS.json; `cpu_baseline` is the CPU oracle
port of the reference path timed on this host (rank 0, N=1 only).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


@dataclass(frozen=True)
class Workload:
    kind: str          # "classify" (images/s) or "prefill" (tokens/s)
    name: str
    L: int
    D: int
    H: int
    T: int
    B: int
    K: int
    G: int
    classes: int
    max_tokens: int


WORKLOADS = {
    "vitb": Workload("classify", "ViT-B/16", 12, 768, 12, 196, 64, 1024, 1, 1000, 197),
    "vitl": Workload("classify", "ViT-L/16@384", 24, 1024, 16, 576, 32, 1024, 1, 1000, 577),
    "gpt2s": Workload("prefill", "GPT-2-small", 12, 768, 12, 1024, 8, 1024, 1, 50257, 1024),
    "gpt2m": Workload("prefill", "GPT-2-medium", 24, 1024, 16, 4096, 2, 1024, 1, 50257, 4096),
}
VITB_METRIC = "ViT-B/16 Astra images/sec (B=64, token sequence split across N B200)"


def _metric(w):
    if w.kind == "prefill":
        return (f"{w.name} Astra causal prefill tokens/sec (T={w.T}, B={w.B}, G={w.G}, K={w.K}, "
                f"token sequence split across N B200)"), "tokens/s"
    if w == WORKLOADS["vitb"]:
        return VITB_METRIC, "images/s"
    return (f"{w.name} Astra images/sec (B={w.B}, T={w.T}, G={w.G}, K={w.K}, token sequence "
            f"split across N B200)"), "images/s"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d["bf16_tflops_sustained"],
                    src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1590.0, src="fallback (B200_PROFILING.md)")


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.05)
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if "Not" not in v
                          and v.strip() not in ("", "[N/A]")})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- setup
GOLDEN = ROOT / "tests" / "golden"
CODEBOOKS = GOLDEN / "vitb16_codebooks.npz"


def _ids(w, count, seed):
    """GPT-2-shape synthetic token ids (make_lm_data caps vocab at 64)."""
    from paper_2505_19342_b200.model import generator
    return generator(seed, "gpt2-ids").integers(0, w.classes, size=(count, w.T)).astype(np.int64)


def _setup_params(w, device=None):
    """Seeded weights (init_params(seed=0), bit-identical to the reference's), codebooks and the
    synthetic inputs.  ViT-B/16 K=1024 G=1 uses the REFERENCE's own k-means output
    (tests/golden/vitb16_codebooks.npz, SHA-256 checked); other shapes fit theirs on the GPU
    with the reference recipe (codebooks.fit_codebooks).  Returns (params, inputs, source)."""
    from paper_2505_19342_b200 import codebooks, data, model
    cfg = model.ModelConfig(layers=w.L, hidden=w.D, heads=w.H, vocab_or_classes=w.classes,
                            max_tokens=w.max_tokens, causal=w.kind == "prefill",
                            codebook_size=w.K, groups=w.G)
    params = model.init_params(cfg, seed=0)
    if w == WORKLOADS["vitb"]:
        codebooks.load_codebook_tables(CODEBOOKS, params)
        src = "the reference's own initialize_codebooks output (tests/golden/vitb16_codebooks.npz)"
    elif w.kind == "prefill":
        codebooks.fit_codebooks(params, _ids(w, max(2, -(-w.K // w.T) + 1), seed=0), seed=0,
                                device=device, mode="lm")
        src = "reference recipe fitted on the GPU (deterministic Lloyd, 2+ sequences)"
    else:
        codebooks.fit_codebooks(params, data.make_classify_batch(w.D, w.T, 8, seed=0, task_seed=0),
                                seed=0, device=device)
        src = "reference recipe fitted on the GPU (deterministic Lloyd, 8 images)"
    if w.kind == "prefill":
        xs = _ids(w, w.B, seed=1)
    else:
        xs = data.make_classify_batch(w.D, w.T, w.B, seed=1, task_seed=0)
    return params, xs, src


def _broadcast_codebooks(params, dist, dev):
    """Under torchrun every rank must run rank 0's codebooks (the runtime broadcasts all
    parameters at upload too; this keeps the host copies equal for the checker)."""
    import torch
    for b in params.blocks:
        for g, c in enumerate(b.codebook.centroids):
            t = torch.from_numpy(np.ascontiguousarray(c, np.float32)).to(dev)
            dist.broadcast(t, src=0)
            b.codebook.centroids[g] = t.cpu().numpy()


def _golden(n):
    """Reference logits / per-layer indices of the 64 ViT-B images at N = n (or None)."""
    p = GOLDEN / "golden_vitb.npz"
    if not p.exists():
        return None
    z = np.load(p)
    if f"n{n}_logits" not in z:
        return None
    return z[f"n{n}_logits"], z[f"n{n}_indices"]


def _compare(got, want_logits, codes, want_idx, T, tol, what):
    """Parity summary: top-1 agreement, max |logit error| (overall and over the images with no
    flipped VQ code), per-layer VQ index agreement (SURVEY 8a')."""
    per_layer, flipped = [], np.zeros(len(got), bool)
    for l in range(codes.shape[1] // T):
        eq = codes[:, l * T:(l + 1) * T] == want_idx[:, l * T:(l + 1) * T]
        per_layer.append(float(eq.mean()))
        flipped |= ~eq.all(axis=1)
    err = float(np.abs(got - want_logits).max())
    clean = ~flipped
    err_clean = float(np.abs(got[clean] - want_logits[clean]).max()) if clean.any() else None
    return {"reference": what,
            "top1_agreement": float((got.argmax(1) == want_logits.argmax(1)).mean()),
            "max_abs_logit_err": err, "logit_tolerance": tol, "within_tolerance": err <= tol,
            "images_with_a_flipped_code": int(flipped.sum()),
            "max_abs_logit_err_images_without_flips": err_clean,
            "min_layer_index_agreement": min(per_layer) if per_layer else None,
            "indices_bitwise": all(a == 1.0 for a in per_layer),
            "per_layer_index_agreement": [round(a, 6) for a in per_layer]}


def _traced_forward(rt, xs):
    """One eager forward recording every layer's VQ codes; returns (outputs, codes [B, L*T])."""
    rt.trace = []
    if rt.mode == "generate":
        rt.set_ids(xs)
    else:
        rt.stage_input(xs)
    rt.forward()
    codes = np.stack([rt.codes_by_image(t)[:, :, 0] for t in rt.trace], axis=1)
    rt.trace = None
    out = rt.first_out.cpu().numpy().copy() if rt.mode == "generate" else rt.logits.cpu().numpy().copy()
    return out, codes.reshape(codes.shape[0], -1)


def _oracle_params(params):
    from oracle import astra_oracle as O
    cfg = params.config
    oc = O.Config(layers=cfg.layers, hidden=cfg.hidden, heads=cfg.heads,
                  vocab_or_classes=cfg.vocab_or_classes, max_tokens=cfg.max_tokens,
                  causal=cfg.causal, codebook_size=cfg.codebook_size, groups=cfg.groups)
    blocks = [{f: np.asarray(getattr(b, f).data) for f in b.TENSOR_FIELDS} for b in params.blocks]
    op = O.Params(config=oc, pos=params.pos.data, blocks=blocks, final_gain=params.final_gain.data,
                  final_bias=params.final_bias.data, head=params.head.data,
                  embedding=params.embedding.data if params.embedding is not None else None,
                  cls=params.cls.data if params.cls is not None else None)
    op.codebooks = [[np.asarray(c) for c in b.codebook.centroids] for b in params.blocks]
    return op


def _oracle_one(op, w, ranges, x):
    """The reference path (oracle port of cluster.run_inference) on one sample; returns
    (output, per-layer codes in global token order)."""
    from oracle import astra_oracle as O
    if w.kind == "prefill":
        r = O.run_inference(op, ranges, x, mode="generate", steps=1)
        out = np.asarray(r.output[:1])
    else:
        r = O.run_inference(op, ranges, x)
        out = np.asarray(r.output).reshape(-1)
    codes = np.concatenate([np.concatenate([i[:, 0] for i in layer]) for layer in r.indices])
    return out, codes


def _cpu_leg(op, w, xs, n_dev, budget_s, max_samples):
    """Time the CPU oracle (reference algorithm port) per sample on a bounded sample; keep its
    outputs for the parity check."""
    from oracle import astra_oracle as O
    ranges = O.partition_tokens(w.T, n_dev)
    outs, codes = [], []
    t0 = time.perf_counter()
    while len(outs) < max_samples and (not outs or time.perf_counter() - t0 < budget_s):
        o, c = _oracle_one(op, w, ranges, xs[len(outs) % len(xs)])
        outs.append(o)
        codes.append(c)
    dt = time.perf_counter() - t0
    return len(outs) / dt, len(outs), dt, np.stack(outs), np.stack(codes)


# ------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The reference's CPU path (the oracle port of seqvq run_inference, pinned bitwise to the
    reference by tests/test_oracle_golden.py and tests/test_headline_cpu.py) on this host, same
    weights / codebooks / samples.  (seqvq itself is not pip-installed here: DESIGN.md §7.)"""
    if rank != 0:
        return
    w = _workload(args)
    from oracle import astra_oracle as O
    if w != WORKLOADS["vitb"]:
        import torch
        if not torch.cuda.is_available():
            print(json.dumps({"impl": "reference", "unavailable": "this workload's codebooks are "
                              "fitted on the GPU; run the ViT-B default"}))
            return
    params, xs, _ = _setup_params(w)
    op = _oracle_params(params)
    ranges = O.partition_tokens(w.T, args.gpus)
    for i in range(args.warmup):
        _oracle_one(op, w, ranges, xs[i % len(xs)])
    t0 = time.perf_counter()
    for i in range(args.steps):
        _oracle_one(op, w, ranges, xs[(args.warmup + i) % len(xs)])
    dt = time.perf_counter() - t0
    per = w.T if w.kind == "prefill" else 1
    metric, unit = _metric(w)
    val = args.steps * per / dt
    cores = os.cpu_count()
    sample = (f"{args.steps} sample(s) of the B={w.B} workload, one per step (the reference API "
              f"has no batch dimension, cluster.py:224), N={args.gpus} simulated devices, "
              f"numpy/OpenBLAS on {cores} host threads")
    line = {"metric": metric, "value": val, "unit": unit, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64",
            "data": _data(w), "config": _config(args, w, "reference"), "impl": "reference",
            "cpu_baseline": {"value": val, "unit": unit, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _data(w):
    if w == WORKLOADS["vitb"]:
        return ("synthetic: make_classify_data(768, 196, 64, seed=1); init_params(seed=0) weights; "
                "the reference's own k-means codebooks (tests/golden/vitb16_codebooks.npz, "
                "sha256-checked)")
    inp = (f"token ids rng.generator(1, 'gpt2-ids') [{w.B}, {w.T}]" if w.kind == "prefill"
           else f"make_classify_data({w.D}, {w.T}, {w.B}, seed=1)")
    return (f"synthetic: {inp}; init_params(seed=0) weights; k-means codebooks fitted with the "
            f"reference recipe on the GPU (same tables given to the CPU oracle)")


def _config(args, w, precision):
    kind = ("causal prefill + first greedy token" if w.kind == "prefill"
            else "classification, distributed class tokens")
    return {"workload": f"{w.name} Astra MPA inference ({kind}): L={w.L}, D={w.D}, H={w.H}, "
                        f"T={w.T}, B={w.B}, codebook K={w.K}, G={w.G}, sequence split over "
                        f"{args.gpus} GPU(s)",
            "global_batch": w.B, "seq_len": w.T, "parallelism": f"sp{args.gpus}",
            "precision": precision,
            "l2": "no flush: the per-step working set (weights + activations) exceeds the 126 MB "
                  "L2; e2e re-stages inputs every step"}


# --------------------------------------------------------------- our arm
def _kernel_work(rt):
    """Algorithmic FLOPs / bytes per launch of each op family."""
    R, Dm, M, G = rt.R, rt.D, rt.n_content, rt.G
    ebf = 2 if rt.fast else 4
    pairs = 0
    for sg in rt.segs.view(-1, 6).cpu().numpy():
        q0, nq, qpos0, ncontent, k0, nk = (int(v) for v in sg)
        if rt.cfg.causal:   # query at global position p sees keys 0..p
            pairs += sum(qpos0 + i + 1 for i in range(ncontent)) + (nq - ncontent) * nk
        else:
            pairs += nq * nk
    att_flops = 4 * rt.H * pairs * rt.dk
    att_bytes = R * 3 * Dm * ebf + R * Dm * 2
    Fm = 4 * Dm
    return {
        "vq_encode": dict(flops=2 * M * rt.K * Dm, bytes=M * Dm * 4 + rt.K * Dm * 4 + M * G * rt.bits / 8),
        "gemm_qkv": dict(flops=2 * R * 3 * Dm * Dm, bytes=(R * Dm + 3 * Dm * Dm + R * 3 * Dm) * 2),
        "gemm_wo": dict(flops=2 * R * Dm * Dm, bytes=(R * Dm + Dm * Dm) * 2 + R * Dm * 8),
        "gemm_w1": dict(flops=2 * R * Fm * Dm, bytes=(R * Dm + Fm * Dm + R * Fm) * 2),
        "gemm_w2": dict(flops=2 * R * Fm * Dm, bytes=(R * Fm + Fm * Dm) * 2 + R * Dm * 8),
        "attention": dict(flops=att_flops, bytes=att_bytes),
        # LN1 also writes the bf16 hi/lo split of the raw rows and their norms (VQ operand)
        "ln1": dict(flops=0, bytes=R * Dm * (4 + 2 + (4 if rt.presplit else 0)) + (R * 4 if rt.presplit else 0)),
        "ln2": dict(flops=0, bytes=R * Dm * (4 + 2)),
        # N > 1, G > 1: received codes -> gathered codebook rows -> LN1 bf16 operand (fused), and
        # the K|V projection of every received row
        "decode_ln": dict(flops=0, bytes=rt.n_content_all * (G * 4 + Dm * 4 + Dm * ebf)),
        "gemm_kv": dict(flops=2 * rt.n_content_all * 2 * Dm * Dm,
                        bytes=(rt.n_content_all * Dm + 2 * Dm * Dm + rt.n_content_all * 2 * Dm) * 2),
    }


def _ncu_traffic(op):
    """DRAM bytes (read + write) per launch of `op` from the newest committed ncu --set full
    capture (profiles/traffic_rNN.json); None if that op was not captured."""
    files = sorted((ROOT / "profiles").glob("traffic_r*.json"))
    if not files:
        return None
    ops = json.loads(files[-1].read_text())["ops"]
    e = ops.get(op) or ops.get(op + "_gemm")
    return None if e is None else e["dram_bytes"]


def _profile(rt, steps=3):
    """Per-op device time of an eager forward with the VQ side stream folded back into the
    main stream, so every op is timed in isolation (the graphed step overlaps them)."""
    import torch
    rt.overlap_vq = False
    rt.profile = {}
    for _ in range(steps):
        rt.forward()
    torch.cuda.synchronize()
    out = {}
    for name, evs in rt.profile.items():
        ms = [st.elapsed_time(en) for st, en in evs]
        out[name] = dict(total_ms=sum(ms) / steps, launches=len(ms) // steps,
                         avg_ms=sum(ms) / len(ms))
    rt.profile = None
    rt.overlap_vq = True
    return out


def _kernels_and_roofline(rt, peaks, vitb):
    """Per-op timing + roofline.  Each op is event-timed alone in an eager pass (not inside a
    long step), so the BURST peaks apply; 3-pass (bf16x3, fp32-class) kernels are measured
    against a third of the bf16 peak (3 MMAs per algorithmic MAC)."""
    prof = _profile(rt, steps=3)
    work = _kernel_work(rt)
    step_ms_eager = sum(v["total_ms"] for v in prof.values())
    kernels = {}
    for name, p in prof.items():
        w = work.get(name)
        entry = {"ms_per_step": round(p["total_ms"], 4), "launches_per_step": p["launches"],
                 "avg_launch_us": round(1000 * p["avg_ms"], 2),
                 "share": round(p["total_ms"] / step_ms_eager, 4)}
        if w:
            sec = p["avg_ms"] / 1000
            three = name == "vq_encode" or (not rt.fast and name not in ("ln1", "ln2"))
            tpeak = peaks["bf16"] / (3.0 if three else 1.0)
            t_tensor = w["flops"] / (tpeak * 1e12) if w["flops"] else 0.0
            t_hbm = w["bytes"] / (peaks["hbm"] * 1e9)
            bound = "tensor" if t_tensor >= t_hbm else "hbm"
            entry.update(bound=bound, frac=round(max(t_tensor, t_hbm) / sec, 3),
                         achieved_gbs=round(w["bytes"] / sec / 1e9, 1))
            if w["flops"]:
                entry.update(achieved_tflops=round(w["flops"] / sec / 1e12, 1),
                             peak_tflops=round(tpeak, 1))
        kernels[name] = entry
    dom = max((n for n in kernels if n in work), key=lambda n: kernels[n]["share"])
    dk, w = kernels[dom], work[dom]
    traffic = _ncu_traffic(dom) if (rt.fast and vitb) else None
    if dk["bound"] == "tensor":
        roof = {"kernel": dom, "bound": "tensor", "achieved": dk["achieved_tflops"],
                "peak": dk["peak_tflops"], "unit": "TFLOP/s", "frac": dk["frac"], "traffic": traffic,
                "peak_source": f"{peaks['src']} bf16 burst"
                               + (" / 3 (bf16x3)" if dk["peak_tflops"] < peaks["bf16"] / 2 else "")
                               + " (op event-timed alone)",
                "per_launch": f"{w['flops'] / 1e9:.2f} GFLOP algorithmic"}
    else:
        roof = {"kernel": dom, "bound": "hbm", "achieved": dk["achieved_gbs"], "peak": peaks["hbm"],
                "unit": "GB/s", "frac": dk["frac"], "traffic": traffic,
                "peak_source": f"{peaks['src']} HBM copy",
                "per_launch": f"{w['bytes'] / 1e6:.1f} MB algorithmic"}
    return kernels, roof


def _measure(prec, w, params, xs, plan, comm, dev, dev_index, args, world, rank, barrier,
             max_over_ranks, peaks):
    import torch
    from paper_2505_19342_b200 import _native
    from paper_2505_19342_b200.runtime import AstraRuntime
    prefill = w.kind == "prefill"
    rt = AstraRuntime(params, plan, batch=w.B, precision=prec, comm=comm, device=dev,
                      mode="generate" if prefill else "classify")
    if prefill:
        rt.set_ids(xs)
    else:
        rt.stage_input(xs)
    torch.cuda.synchronize()
    try:
        rt.capture(warmup=1)
        graphed = True
    except Exception:  # capture unsupported (e.g. collective inside capture): eager launches
        torch.cuda.synchronize()
        rt.graph = None
        graphed = False
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = Clocks(dev_index)
    with clocks:   # sampler starts before the warm-up so every sample is taken under load
        for _ in range(args.warmup):
            rt.run()
        torch.cuda.synchronize()
        barrier()
        s.record()
        for _ in range(args.steps):
            rt.run()
        e.record()
        torch.cuda.synchronize()
        barrier()
    ms = max_over_ranks(s.elapsed_time(e)) / args.steps
    rt.check_errors()
    per_step = w.B * (w.T if prefill else 1)
    out = dict(ms=ms, value=per_step / (ms / 1000.0), graphed=graphed, clocks=clocks.summary())

    # launches per step (eager pass with the launch counter on)
    _native.count_launches(True)
    rt.forward()
    out["launches"] = sum(_native.count_launches(False).values())
    torch.cuda.synchronize()

    # VQ exactness counters (one eager pass with them on)
    rt.vq_stats.zero_()
    rt.collect_vq_stats = True
    rt.forward()
    rt.collect_vq_stats = False
    torch.cuda.synchronize()
    vs = rt.vq_stats.cpu().numpy().astype(float)
    tokens_encoded = rt.n_content * w.L
    out["vq_exactness"] = {
        "tokens_encoded_per_step": tokens_encoded,
        "tokens_reranked_fp64": vs[0] + vs[1], "tokens_with_overflowed_chunk": vs[1],
        "rerank_rate": round((vs[0] + vs[1]) / max(tokens_encoded, 1), 5),
        "window_candidates_per_token": round(vs[2] / max(tokens_encoded, 1), 4)}
    out["kernels"], out["roofline"] = _kernels_and_roofline(rt, peaks, w == WORKLOADS["vitb"])

    # one traced forward (every rank: it holds the collectives) for the parity checks
    got, codes = _traced_forward(rt, xs)
    out["traced"] = (got, codes)
    out["parity"] = None
    g = _golden(args.gpus) if w == WORKLOADS["vitb"] else None
    if g is not None and rank == 0:
        out["parity"] = _compare(got, g[0], codes, g[1], w.T, 3e-2 if rt.fast else 1e-4,
                                 f"seqvq run_inference at N={args.gpus} on the same weights, "
                                 f"codebooks and {len(got)} images (tests/golden/golden_vitb.npz)")
    torch.cuda.synchronize()
    barrier()

    # e2e through the public runtime API: pinned host batches in, results read on the host
    # after every step (classify_stream / prefill_stream: H2D of batch i+1 overlaps batch i)
    if prefill:
        host_in = torch.from_numpy(np.ascontiguousarray(xs, dtype=np.int32)).pin_memory()
        res_shape, res_dt, serve = (w.B,), torch.int32, rt.prefill_stream
    else:
        start, stop = plan.ranges[rank] if world > 1 else (0, w.T)
        host_in = torch.from_numpy(np.ascontiguousarray(xs[:, start:stop])).pin_memory()
        res_shape, res_dt, serve = (w.B, rt.classes), torch.float32, rt.classify_stream
    outs = [torch.empty(res_shape, dtype=res_dt).pin_memory() for _ in range(2)]
    serve([host_in] * 3, out=outs * 2)
    torch.cuda.synchronize()
    barrier()
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es.record()
    serve([host_in] * args.steps, out=[outs[i % 2] for i in range(args.steps)])
    ee.record()
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(es.elapsed_time(ee)) / args.steps
    out["e2e"] = {"value": per_step / (e2e_ms / 1000.0), "unit": _metric(w)[1],
                  "h2d_bytes_per_step": host_in.numel() * host_in.element_size(),
                  "d2h_bytes_per_step": outs[0].numel() * outs[0].element_size(),
                  "ms_per_step": e2e_ms}
    del rt
    torch.cuda.empty_cache()
    return out


def _workload(args):
    w = WORKLOADS[args.config]
    if args.groups or args.codebook or args.batch:
        w = Workload(w.kind, w.name, w.L, w.D, w.H, w.T, args.batch or w.B, args.codebook or w.K,
                     args.groups or w.G, w.classes, w.max_tokens)
    return w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fast", choices=["fast", "parity"])
    ap.add_argument("--config", default="vitb", choices=sorted(WORKLOADS))
    ap.add_argument("--groups", type=int, default=0)
    ap.add_argument("--codebook", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--only-main", action="store_true", help="skip the second precision mode")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.gpus != world:
        args.gpus = world
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    w = _workload(args)
    metric, unit = _metric(w)

    import torch
    import torch.distributed as dist
    from paper_2505_19342_b200.cluster import partition_tokens
    from paper_2505_19342_b200.runtime import TorchDistExchange

    # ASTRA_BENCH_ONE_GPU=1: every rank on cuda:0 with the gloo exchange (functional check of
    # the multi-rank path on a one-GPU box; NCCL refuses two ranks on one device)
    one_gpu = os.environ.get("ASTRA_BENCH_ONE_GPU") == "1"
    dev_index = 0 if one_gpu else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    comm = None
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        comm = TorchDistExchange()
    peaks = _peaks()
    params, xs, cb_src = _setup_params(w, device=dev)
    if world > 1 and w != WORKLOADS["vitb"]:
        _broadcast_codebooks(params, dist, "cpu" if one_gpu else dev)
    plan = partition_tokens(w.T, args.gpus, class_replication=w.kind != "prefill")

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if one_gpu else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    main_prec = args.precision
    precs = [main_prec] + ([] if args.only_main else [p for p in ("fast", "parity") if p != main_prec])
    res = {p: _measure(p, w, params, xs, plan, comm, dev, dev_index, args, world, rank, barrier,
                       max_over_ranks, peaks) for p in precs}
    m = res[main_prec]

    # CPU baseline (rank 0, N=1): the oracle port on this host, same weights / codebooks /
    # samples; for workloads without reference goldens its outputs are also the parity check
    cpu = None
    if rank == 0 and args.gpus == 1 and not args.no_cpu_baseline:
        op = _oracle_params(params)
        budget = 12.0 if w == WORKLOADS["vitb"] else 20.0
        rate, n, dt, o_out, o_codes = _cpu_leg(op, w, xs, 1, budget, 16 if w.kind == "classify" else 2)
        per = w.T if w.kind == "prefill" else 1
        cpu = {"value": rate * per, "unit": unit, "cores": os.cpu_count(), "kind": "port",
               "sample": f"{n} sample(s) of the same workload through oracle.run_inference "
                         f"(N=1), {dt:.1f} s; numpy/OpenBLAS with all host threads"}
        if w != WORKLOADS["vitb"]:
            for p in precs:
                got, codes = res[p]["traced"]
                fast = p == "fast"
                if w.kind == "prefill":
                    res[p]["parity"] = {
                        "reference": f"oracle run_inference (generate, steps=1) on {n} of the "
                                     f"{w.B} sequences, same weights and codebooks",
                        "first_token_agreement": float((got[:n] == o_out[:, 0]).mean()),
                        "min_layer_index_agreement": float(min(
                            (codes[:n, l * w.T:(l + 1) * w.T] == o_codes[:, l * w.T:(l + 1) * w.T]).mean()
                            for l in range(w.L)))}
                else:
                    res[p]["parity"] = _compare(got[:n], o_out, codes[:n], o_codes, w.T,
                                                3e-2 if fast else 1e-4,
                                                f"oracle run_inference on {n} of the {w.B} images, "
                                                f"same weights and codebooks")

    if rank == 0:
        line = {
            "metric": metric, "value": m["value"], "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["ms"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if main_prec == "fast" else "bf16x3",
            "data": _data(w), "config": _config(args, w, main_prec),
            "codebooks": cb_src,
            "per_layer_ms": m["ms"] / w.L,
            "cuda_graph": m["graphed"],
            "parity": m["parity"],
            "roofline": m["roofline"],
            "kernels": m["kernels"],
            "vq_encode_gbs": m["kernels"].get("vq_encode", {}).get("achieved_gbs"),
            "vq_exactness": m["vq_exactness"],
            "cpu_baseline": cpu,
            "e2e": m["e2e"],
            "gpu_launches": m["launches"] * args.steps,
            "gpu_launches_per_step": m["launches"],
            "clocks": m["clocks"],
        }
        for p in precs[1:]:
            o = res[p]
            line[f"{p}_mode"] = {"value": o["value"], "ms_per_step": o["ms"],
                                 "per_layer_ms": o["ms"] / w.L,
                                 "dtype": "bf16" if p == "fast" else "bf16x3 (fp32-class)",
                                 "cuda_graph": o["graphed"], "e2e": o["e2e"],
                                 "parity": o["parity"], "roofline": o["roofline"],
                                 "kernels": o["kernels"], "gpu_launches_per_step": o["launches"],
                                 "clocks": o["clocks"]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
