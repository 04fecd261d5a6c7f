"""Print the headline numbers of a bench.py JSON line (file argument)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001
        print(path, "bench failed", e)
        try:
            print(open(path.replace(".json", ".err")).read()[-3000:])
        except OSError:
            pass
        continue
    par = d.get("parity") or {}
    print(path, "value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms",
          round(d["ms_per_step"], 3), "top1", par.get("top1_agreement"), "maxerr",
          par.get("max_abs_logit_err"), "min_idx_agree", par.get("min_layer_index_agreement"))
    print("  vq", d.get("vq_exactness"))
    for k, v in d["kernels"].items():
        print(f"  {k:12s} {v['avg_launch_us']:8.2f} us  share {v['share']:.3f}  {v.get('frac', '')}")
    pm = d.get("parity_mode")
    if pm:
        print("  parity_mode ms", pm["ms_per_step"], (pm.get("parity") or {}).get("max_abs_logit_err"))
