#!/bin/bash
# ncu evidence for the forward: launch list (device time per kernel, 2 forwards) and one
# `--set full` capture of every hot kernel of layer 0.  Usage: bash scripts/gpu_profile.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$TAG.csv python scripts/profile_forward.py --iters 2 > gpurun_out/launch_$TAG.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:'tc_gemm|attention_tc|vq_finalize|layernorm' -c 9 \
   -o gpurun_out/full_$TAG python scripts/profile_forward.py --iters 1 > gpurun_out/full_$TAG.log 2>&1
ls -la gpurun_out
