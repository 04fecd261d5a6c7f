#!/bin/bash
# ncu --set full of the G=1 VQ re-rank and finalize launches of layer 0 (bench workload)
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:'vq_rerank|vq_finalize' -c 2 -o gpurun_out/rerank_${1:-r02j} python scripts/profile_forward.py --iters 1 > gpurun_out/rerank_${1:-r02j}.log 2>&1
tail -2 gpurun_out/rerank_${1:-r02j}.log
