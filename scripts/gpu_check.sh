#!/bin/bash
# Full GPU test suite + bench lines for the default config and ViT-L G=16.  Usage: bash scripts/gpu_check.sh TAG
TAG=${1:-rXX}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -15 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b_vitb_$TAG.json 2> gpurun_out/b_vitb_$TAG.err
timeout 600 python bench.py --no-cpu-baseline --config vitl --groups 16 --steps 10 > gpurun_out/b_vitl_$TAG.json 2> gpurun_out/b_vitl_$TAG.err
for f in gpurun_out/b_vitb_$TAG.json gpurun_out/b_vitl_$TAG.json; do
python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], "value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms", round(d["ms_per_step"], 3), "parity", {k: d.get("parity", {}).get(k) for k in ("top1_agreement", "max_abs_logit_err", "min_layer_index_agreement")})
    print("  vq", d.get("vq_exactness"))
    for k, v in d["kernels"].items():
        print(f"  {k:12s} {v['avg_launch_us']:8.2f} us  share {v['share']:.3f}  {v.get('frac', '')}")
    pm = d.get("parity_mode")
    if pm: print("  parity_mode ms", pm["ms_per_step"], pm.get("parity"))
except Exception as e:
    print("bench failed", e); print(open(sys.argv[1].replace('.json', '.err')).read()[-3000:])
PY
done
