#!/bin/bash
# A/B of an env switch on the default bench (fast mode only): bash scripts/gpu_ab.sh TAG VAR [extra bench args]
TAG=${1:-ab}; VAR=${2:-ASTRA_PDL}; shift 2
mkdir -p gpurun_out
for v in ${VALUES:-1 0 1 0}; do
  env $VAR=$v timeout 300 python bench.py --no-cpu-baseline --only-main --steps 100 "$@" > gpurun_out/ab_${TAG}_$v.json 2>> gpurun_out/ab_${TAG}.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_${TAG}_$v.json').read().strip().splitlines()[-1]); print('$VAR=$v', round(d['ms_per_step'],4), 'ms', round(d['value']), d.get('parity',{}).get('max_abs_logit_err'), d['clocks'])"
done
