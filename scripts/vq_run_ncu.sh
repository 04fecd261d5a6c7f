#!/bin/bash
# ncu --set full (source-level) of the run-mode VQ GEMM: the G=16 (skip 0) or G=32 (skip 6) case
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:VqRunEpilogue -s ${1:-6} -c 1 -o gpurun_out/vq_run_${2:-g32} \
  python scripts/microbench.py --reps 3 --only vq > gpurun_out/vq_run_${2:-g32}.log 2>&1
tail -2 gpurun_out/vq_run_${2:-g32}.log
