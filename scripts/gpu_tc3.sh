#!/bin/bash
# Parity-mode attention (attention_tc3_kernel) evidence: one `--set full` capture with source
# of the layer-0 launch of the ViT-B/16 B=64 parity forward.  Usage: bash scripts/gpu_tc3.sh TAG
TAG=${1:-tc3}
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:'attention_tc3' -c 1 -o gpurun_out/tc3_$TAG python scripts/profile_forward.py --parity --iters 1 \
   > gpurun_out/tc3_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/tc3_$TAG.log
