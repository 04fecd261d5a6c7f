"""Summarise ncu captures for profiles/: per kernel duration, DRAM traffic, tensor-pipe
and SM utilisation, top stall reasons (from `--set full` reports) or per-kernel time shares
(from a `--metrics gpu__time_duration.sum --csv` launch list).

    python scripts/ncu_summary.py report.ncu-rep [...] > profiles/xxx.md
    python scripts/ncu_summary.py --launches launches.csv [--last N] > profiles/yyy.md
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_insts",
}


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    res = []
    for v in rows[2:]:
        d = dict(zip(h, v))
        e = {"kernel": d.get("Kernel Name", "")[:90]}
        for k, name in KEYS.items():
            if k in d and d[k] not in ("", "n/a"):
                x = float(d[k].replace(",", ""))
                e[name] = round(x, 3)
        st = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                    "_per_issue_active.ratio") and d.get(k) not in (None, "", "n/a"):
                st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len(
                    "_per_issue_active.ratio")]))
        st.sort(reverse=True)
        e["top_stalls"] = [f"{n}:{x:.2f}" for x, n in st[:4]]
        res.append(e)
    return res


def launches(path, last=None):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                data.append(d)
    if last:
        data = data[-last:]
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = v / 1000 if u in ("nsecond", "ns") else (v * 1000 if u in ("msecond", "ms") else v)
        name = d["Kernel Name"].split("(")[0][:80]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    out = []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k, "launches": n, "total_us": round(t, 1),
                    "avg_us": round(t / n, 2), "share": round(t / tot, 4)})
    return out, tot


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else None
        rows, tot = launches(sys.argv[2], last)
        print(f"| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|")
        for r in rows:
            print(f"| {r['kernel']} | {r['launches']} | {r['total_us']} | {r['avg_us']} | "
                  f"{100 * r['share']:.1f}% |")
        print(f"\ntotal {tot:.1f} us over {sum(r['launches'] for r in rows)} launches")
    else:
        allr = []
        for p in sys.argv[1:]:
            allr += report(p)
        print(json.dumps(allr, indent=1))
