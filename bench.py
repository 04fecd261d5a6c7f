"""Benchmark: ViT-B/16 Astra Mixed-Precision-Attention inference on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one rank per GPU, NCCL)

Workload (BASELINE.json configs[1]): ViT-B/16 shape (L=12, D=768, H=12, MLP 3072, no
patch embedding — inputs are [196, 768] token embeddings like the reference), batch 64,
token sequence split across N GPUs (N=1 default), VQ codebook K=1024, G=1, distributed
class tokens.  Weights: the reference's seeded init_params(seed=0); codebooks: the
reference's OWN initialize_codebooks output (tests/golden/vitb16_codebooks.npz, written by
seqvq in tests/golden/make_golden_vitb.py); inputs: make_classify_data(seed=1).  A step =
one full forward of the 64-image batch.  Both precision modes are measured; the line's
`parity` blocks compare each with the reference's own logits / VQ indices for the same 64
images at the same N (tests/golden/golden_vitb.npz).

Prints ONE JSON line (rank 0).  `value` is images/s with inputs resident in HBM (CUDA
graph replay, device-timed, max over ranks); `e2e` is the same metric through the public
runtime API with the host->device input copy and device->host logits read inside every
step; `roofline` is the dominant kernel vs MEASURED_PEAKS.json; `cpu_baseline` is the CPU
oracle port of the reference path timed on this host (rank 0, N=1 only).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ViT-B/16 Astra images/sec (B=64, token sequence split across N B200)"
UNIT = "images/s"
L, D, H, T, B, K = 12, 768, 12, 196, 64, 1024


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


def _setup_params():
    """Seeded weights (init_params(seed=0), bit-identical to the reference's), the REFERENCE's
    own k-means codebooks (initialize_codebooks(..., K=1024, G=1, seed=0) run by seqvq in
    tests/golden/make_golden_vitb.py; SHA-256 checked on load) and the synthetic batch
    make_classify_data(seed=1).  Both arms run exactly these inputs."""
    from paper_2505_19342_b200 import codebooks, data, model
    cfg = model.ModelConfig(layers=L, hidden=D, heads=H, vocab_or_classes=1000, max_tokens=197,
                            causal=False, codebook_size=K, groups=1)
    params = model.init_params(cfg, seed=0)
    codebooks.load_codebook_tables(CODEBOOKS, params)
    xs = data.make_classify_batch(D, T, B, seed=1, task_seed=0)
    return params, xs


def _golden(n):
    """Reference logits / per-layer indices of the same 64 images at N = n (or None)."""
    p = GOLDEN / "golden_vitb.npz"
    if not p.exists():
        return None
    z = np.load(p)
    if f"n{n}_logits" not in z:
        return None
    return z[f"n{n}_logits"], z[f"n{n}_indices"]


def _parity_block(rt, xs, n, tol):
    """Run one traced eager forward and compare with the reference's own outputs for the same
    weights, codebooks and images (golden_vitb.npz): top-1 agreement over the batch, max |logit
    error|, VQ index agreement per layer (SURVEY 8a')."""
    g = _golden(n)
    if g is None:
        return None
    want_logits, want_idx = g
    rt.trace = []
    rt.stage_input(xs)
    rt.forward()
    got = rt.logits.cpu().numpy()
    per_layer = []
    flipped = np.zeros(len(got), bool)
    for l, t in enumerate(rt.trace):
        codes = rt.codes_by_image(t)[:, :, 0]
        eq = codes == want_idx[:, l * T:(l + 1) * T]
        per_layer.append(float(eq.mean()))
        flipped |= ~eq.all(axis=1)
    rt.trace = None
    err = float(np.abs(got - want_logits).max())
    clean = ~flipped
    err_clean = float(np.abs(got[clean] - want_logits[clean]).max()) if clean.any() else None
    top1 = float((got.argmax(1) == want_logits.argmax(1)).mean())
    return {"reference": f"seqvq run_inference at N={n} on the same weights, codebooks and "
                         f"{len(got)} images (tests/golden/golden_vitb.npz)",
            "top1_agreement": top1, "max_abs_logit_err": err, "logit_tolerance": tol,
            "within_tolerance": err <= tol,
            "images_with_a_flipped_code": int(flipped.sum()),
            "max_abs_logit_err_images_without_flips": err_clean,
            "min_layer_index_agreement": min(per_layer) if per_layer else None,
            "indices_bitwise": all(a == 1.0 for a in per_layer),
            "per_layer_index_agreement": [round(a, 6) for a in per_layer]}


def _oracle_params(params):
    from oracle import astra_oracle as O
    cfg = params.config
    oc = O.Config(layers=cfg.layers, hidden=cfg.hidden, heads=cfg.heads,
                  vocab_or_classes=cfg.vocab_or_classes, max_tokens=cfg.max_tokens,
                  causal=cfg.causal, codebook_size=cfg.codebook_size, groups=cfg.groups)
    blocks = [{f: np.asarray(getattr(b, f).data) for f in b.TENSOR_FIELDS} for b in params.blocks]
    op = O.Params(config=oc, pos=params.pos.data, blocks=blocks, final_gain=params.final_gain.data,
                  final_bias=params.final_bias.data, head=params.head.data,
                  cls=params.cls.data if params.cls is not None else None)
    op.codebooks = [[np.asarray(c) for c in b.codebook.centroids] for b in params.blocks]
    return op


def _time_oracle(op, xs, n_dev, budget_s=12.0, max_images=16, min_images=1):
    """Time the CPU oracle (reference algorithm port) per image; bounded sample."""
    from oracle import astra_oracle as O
    ranges = O.partition_tokens(T, n_dev)
    done, t0 = 0, time.perf_counter()
    while done < max_images and (done < min_images or time.perf_counter() - t0 < budget_s):
        O.run_inference(op, ranges, xs[done % len(xs)])
        done += 1
    dt = time.perf_counter() - t0
    return done / dt, done, dt


# ------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The reference's CPU path (the oracle port of seqvq run_inference, pinned bitwise to the
    reference by tests/test_oracle_golden.py) on this host, same weights / codebooks / images."""
    if rank != 0:
        return
    from oracle import astra_oracle as O
    params, xs = _setup_params()   # host-side: seeded weights, committed codebooks, inputs
    op = _oracle_params(params)
    ranges = O.partition_tokens(T, args.gpus)
    for i in range(args.warmup):
        O.run_inference(op, ranges, xs[i % B])
    t0 = time.perf_counter()
    for i in range(args.steps):
        O.run_inference(op, ranges, xs[(args.warmup + i) % B])
    dt = time.perf_counter() - t0
    val = args.steps / dt
    cores = os.cpu_count()
    sample = (f"{args.steps} image(s) of the B={B} workload, one image per step (the reference "
              f"API has no batch dimension, cluster.py:224), N={args.gpus} simulated devices, "
              f"numpy/OpenBLAS on {cores} host threads")
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64",
            "data": DATA, "config": _config(args, "reference"), "impl": "reference",
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


DATA = ("synthetic: make_classify_data(768, 196, 64, seed=1); init_params(seed=0) weights; the "
        "reference's own k-means codebooks (tests/golden/vitb16_codebooks.npz, sha256-checked)")


def _config(args, precision):
    return {"workload": f"ViT-B/16 Astra MPA inference: L={L}, D={D}, H={H}, T={T}, B={B}, "
                        f"codebook K={K}, G=1, distributed class tokens, sequence split over "
                        f"{args.gpus} GPU(s)",
            "global_batch": B, "seq_len": T, "parallelism": f"sp{args.gpus}",
            "precision": precision,
            "l2": "no flush: the per-step working set (weights 170 MB bf16 / 340 MB split + "
                  "activations > 400 MB) exceeds the 126 MB L2; e2e re-stages inputs every step"}


# --------------------------------------------------------------- our arm
def _kernel_work(rt):
    """Algorithmic FLOPs / bytes per launch of each op family."""
    R, Dm, M, G = rt.R, rt.D, rt.n_content, rt.G
    ebf = 2 if rt.fast else 4
    att_flops = 0
    segs = rt.segs.view(-1, 6).cpu().numpy()
    for sg in segs:
        att_flops += 4 * rt.H * int(sg[1]) * int(sg[5]) * rt.dk
    att_bytes = R * 3 * Dm * ebf + R * Dm * 2
    return {
        "vq_encode": dict(flops=2 * M * rt.K * Dm, bytes=M * Dm * 4 + rt.K * Dm * 4 + M * G * rt.bits / 8),
        "gemm_qkv": dict(flops=2 * R * 3 * Dm * Dm, bytes=(R * Dm + 3 * Dm * Dm + R * 3 * Dm) * 2),
        "gemm_wo": dict(flops=2 * R * Dm * Dm, bytes=(R * Dm + Dm * Dm) * 2 + R * Dm * 8),
        "gemm_w1": dict(flops=2 * R * 4 * Dm * Dm, bytes=(R * Dm + 4 * Dm * Dm + 4 * R * Dm) * 2),
        "gemm_w2": dict(flops=2 * R * 4 * Dm * Dm, bytes=(4 * R * Dm + 4 * Dm * Dm) * 2 + R * Dm * 8),
        "attention": dict(flops=att_flops, bytes=att_bytes),
        # LN1 also writes the bf16 hi/lo split of the raw rows and their norms (VQ operand)
        "ln1": dict(flops=0, bytes=R * Dm * (4 + 2 + (4 if rt.presplit else 0)) + (R * 4 if rt.presplit else 0)),
        "ln2": dict(flops=0, bytes=R * Dm * (4 + 2)),
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


def _kernels_and_roofline(rt, peaks):
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
            three = name == "vq_encode" or (not rt.fast and name != "ln1" and name != "ln2")
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
    traffic = _ncu_traffic(dom) if rt.fast else None
    if dk["bound"] == "tensor":
        roof = {"kernel": dom, "bound": "tensor", "achieved": dk["achieved_tflops"],
                "peak": dk["peak_tflops"], "unit": "TFLOP/s", "frac": dk["frac"], "traffic": traffic,
                "peak_source": f"{peaks['src']} bf16 burst" + (" / 3 (bf16x3)" if dk["peak_tflops"] < peaks["bf16"] / 2 else "")
                               + " (op event-timed alone)",
                "per_launch": f"{w['flops'] / 1e9:.2f} GFLOP algorithmic"}
    else:
        roof = {"kernel": dom, "bound": "hbm", "achieved": dk["achieved_gbs"], "peak": peaks["hbm"],
                "unit": "GB/s", "frac": dk["frac"], "traffic": traffic,
                "peak_source": f"{peaks['src']} HBM copy",
                "per_launch": f"{w['bytes'] / 1e6:.1f} MB algorithmic"}
    return kernels, roof


def _measure(prec, params, xs, plan, comm, dev, dev_index, args, world, rank, barrier,
             max_over_ranks, peaks):
    import torch
    from paper_2505_19342_b200 import _native
    from paper_2505_19342_b200.runtime import AstraRuntime
    rt = AstraRuntime(params, plan, batch=B, precision=prec, comm=comm, device=dev)
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
    out = dict(ms=ms, value=B / (ms / 1000.0), graphed=graphed, clocks=clocks.summary())

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
    tokens_encoded = rt.n_content * L
    out["vq_exactness"] = {
        "tokens_encoded_per_step": tokens_encoded,
        "tokens_reranked_fp64": vs[0] + vs[1], "tokens_with_overflowed_chunk": vs[1],
        "rerank_rate": round((vs[0] + vs[1]) / max(tokens_encoded, 1), 5),
        "window_candidates_per_token": round(vs[2] / max(tokens_encoded, 1), 4)}
    out["kernels"], out["roofline"] = _kernels_and_roofline(rt, peaks)

    # parity against the reference's own outputs (same weights, codebooks, images, N)
    out["parity"] = _parity_block(rt, xs, args.gpus, 3e-2 if rt.fast else 1e-4) if rank == 0 \
        else None
    if world > 1 and rank != 0:   # every rank runs the traced forward (it holds a collective)
        rt.trace = []
        rt.stage_input(xs)
        rt.forward()
        rt.trace = None
    torch.cuda.synchronize()
    barrier()

    # e2e through the public runtime API: pinned host batches in, logits read on the host
    # after every step (AstraRuntime.classify_stream: H2D of batch i+1 overlaps batch i)
    start, stop = plan.ranges[rank] if world > 1 else (0, T)
    local_x = torch.from_numpy(np.ascontiguousarray(xs[:, start:stop])).pin_memory()
    outs = [torch.empty(B, rt.classes, dtype=torch.float32).pin_memory() for _ in range(2)]
    rt.classify_stream([local_x] * 3, out=outs * 2)
    torch.cuda.synchronize()
    barrier()
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es.record()
    rt.classify_stream([local_x] * args.steps, out=[outs[i % 2] for i in range(args.steps)])
    ee.record()
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(es.elapsed_time(ee)) / args.steps
    out["e2e"] = {"value": B / (e2e_ms / 1000.0), "unit": UNIT,
                  "h2d_bytes_per_step": local_x.numel() * 4,
                  "d2h_bytes_per_step": B * rt.classes * 4, "ms_per_step": e2e_ms}
    out["classes"] = rt.classes
    del rt
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fast", choices=["fast", "parity"])
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
    params, xs = _setup_params()
    plan = partition_tokens(T, args.gpus)

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
    res = {p: _measure(p, params, xs, plan, comm, dev, dev_index, args, world, rank, barrier,
                       max_over_ranks, peaks) for p in precs}
    m = res[main_prec]

    # CPU baseline: oracle port on this host, rank 0, N=1 only, same weights/codebooks/images
    cpu = None
    if rank == 0 and args.gpus == 1 and not args.no_cpu_baseline:
        op = _oracle_params(params)
        rate, n_img, dt = _time_oracle(op, xs, 1)
        cpu = {"value": rate, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": f"{n_img} image(s) of the same workload through oracle.run_inference "
                         f"(N=1), {dt:.1f} s; numpy/OpenBLAS with all host threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["ms"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if main_prec == "fast" else "bf16x3",
            "data": DATA, "config": _config(args, main_prec),
            "per_layer_ms": m["ms"] / L,
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
                                 "per_layer_ms": o["ms"] / L,
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
