#!/bin/bash
# quick GPU iteration: selected tests + bench line.  Usage: bash scripts/gpu_quick.sh "<pytest -k expr>" [bench args]
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_pytest.log
tail -5 gpurun_out/quick_pytest.log
shift
timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/quick_bench.json").read().strip().splitlines()[-1])
    print("value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms", round(d["ms_per_step"], 3))
    for k, v in d["kernels"].items():
        print(f"  {k:12s} {v['avg_launch_us']:8.2f} us  share {v['share']:.3f}  {v.get('frac', '')}")
except Exception as e:
    print("bench failed", e); print(open("gpurun_out/quick_bench.err").read()[-3000:])
PY
