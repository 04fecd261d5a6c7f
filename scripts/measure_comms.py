"""Measured variant of the reference's speedup table (comms.py:193-262) for ViT-B/16, B=64:

  compute_s  per-rank device time of the Astra forward at N (scripts/bench_ranks.py JSON lines,
             the rank's own shard with a loopback exchange) — "single" = the N=1 forward;
  comm_s     12 packed-index all-gathers of the runtime's exact wire payload on a LinkModel:
             * under torchrun with > 1 GPU, fitted to all_gather_into_tensor timings of the
               payload sizes over NCCL (NVLink/NVSwitch), device-timed, max over ranks;
             * otherwise (one GPU per box here) an ASSUMED NVLink-5 link, labelled as such.

    python scripts/measure_comms.py --ranks profiles/r02_ranks.jsonl --out profiles/r02_comms_vitb.csv
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 scripts/measure_comms.py --ranks ...
Writes the reference's CSV columns plus a `link` comment header line.
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_19342_b200 import comms as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ranks", required=True, help="bench_ranks.py JSON lines (config vitb)")
ap.add_argument("--out", required=True)
ap.add_argument("--assumed-alpha-us", type=float, default=5.0)
ap.add_argument("--assumed-beta-gbs", type=float, default=900.0)
args = ap.parse_args()

T, B, D, L, K, G = 196, 64, 768, 12, 1024, 1
comp = {}
for line in Path(args.ranks).read_text().splitlines():
    r = json.loads(line)
    if r.get("config") != "vitb":
        continue
    n, sec = int(r["n"]), float(r["ms_per_step"]) / 1e3
    comp[("astra", n, T)] = sec
    if n == 1:
        comp[("single", 1, T)] = sec
devices = sorted({k[1] for k in comp if k[0] == "astra"})

world = int(os.environ.get("WORLD_SIZE", "1"))
if world > 1:
    import torch
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    sizes = sorted({C.astra_wire_bytes(T, world, G, K, B)} | {1 << s for s in range(10, 25, 2)})
    samples = C.measure_allgather(sizes, reps=50, warmup=5, device="cuda")
    link = C.fit_link(samples, f"nccl all_gather_into_tensor, {world} GPUs, measured")
    dist.destroy_process_group()
    if rank != 0:
        sys.exit(0)
else:
    samples = []
    link = C.LinkModel(args.assumed_alpha_us * 1e-6, args.assumed_beta_gbs * 1e9,
                       "ASSUMED NVLink-5 (one GPU per box: no NCCL transfer measurable here)")

cfg = C.CommsConfig(layers=L, hidden=D, tokens=T, devices=1, bandwidth_bps=int(link.beta_Bps * 8),
                    codebook_size=K, groups=G)
rows = C.speedup_table_measured(cfg, [C.MethodSpec("astra")], devices,
                                [T], link=link, compute_s=comp, batch=B)
text = (f"# link: alpha {link.alpha_s * 1e6:.3f} us, beta {link.beta_Bps / 1e9:.1f} GB/s ({link.source}); "
        f"compute_s = measured per-rank device time ({args.ranks}); speedup vs the measured N=1 "
        f"forward; samples {json.dumps(samples)}\n") + C.bench_csv(rows)
Path(args.out).write_text(text)
print(text)
