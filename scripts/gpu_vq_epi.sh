#!/bin/bash
# VQ encode check: bit-exact VQ + runtime parity tests, microbench, (optional) GEMM isolation
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_vq_gpu.py tests/test_runtime_gpu.py tests/test_headline_gpu.py -x -q 2>&1 | tail -3
timeout 300 python scripts/microbench.py --reps 30 2>&1 | grep vq_encode | cut -c1-120
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:'vq_final|vq_rerank' -c 12 --csv python scripts/microbench.py --reps 3 2>/dev/null \
  | grep -i "gpu__time" | awk -F'","' '{print $NF, substr($5,1,40)}'
[ "$1" = iso ] && bash scripts/vq_gemm_isolate.sh
exit 0
