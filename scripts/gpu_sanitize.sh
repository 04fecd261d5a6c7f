#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_small.py.
# Usage: bash scripts/gpu_sanitize.sh TAG
TAG=${1:-san}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_small.py \
     > gpurun_out/${TAG}_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_$tool.txt
  tail -2 gpurun_out/${TAG}_$tool.txt
done
