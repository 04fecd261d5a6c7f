#!/bin/bash
# ViT-L G x K sweep + decode microbenchmark.  Usage: bash scripts/gpu_sweep.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 300 python scripts/vq_decode_bench.py > gpurun_out/decode_$TAG.jsonl 2> gpurun_out/decode_$TAG.err
STEPS=10 timeout 3000 bash scripts/sweep_vitl.sh
cp gpurun_out/sweep_vitl.jsonl gpurun_out/sweep_vitl_$TAG.jsonl
wc -l gpurun_out/sweep_vitl_$TAG.jsonl
