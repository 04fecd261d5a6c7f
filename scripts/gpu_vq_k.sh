#!/bin/bash
# VQ tests, then launch lists of one ViT-L forward at K=4096 for G = 1, 16, 32.  Usage: bash scripts/gpu_vq_k.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "vq or runtime or headline" > gpurun_out/pytest_vqk_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_vqk_$TAG.log
tail -2 gpurun_out/pytest_vqk_$TAG.log
for g in 1 16 32; do
  timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_vitl_g${g}_k4096_$TAG.csv python scripts/profile_forward.py --config vitl --groups $g --codebook 4096 --iters 1 > /dev/null 2>&1
  python scripts/ncu_summary.py --launches gpurun_out/launch_vitl_g${g}_k4096_$TAG.csv | head -14
done
