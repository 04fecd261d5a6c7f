#!/bin/bash
# VQ iteration: VQ + runtime tests, then the ViT-L G=16 bench line (no CPU leg).  Usage: bash scripts/gpu_vq.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "vq or runtime or headline" > gpurun_out/pytest_vq_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_vq_$TAG.log
tail -3 gpurun_out/pytest_vq_$TAG.log
timeout 600 python bench.py --no-cpu-baseline --only-main --config vitl --groups 16 --steps 10 > gpurun_out/b_vitl_$TAG.json 2> gpurun_out/b_vitl_$TAG.err
timeout 600 python bench.py --no-cpu-baseline --only-main --steps 30 > gpurun_out/b_vitb_$TAG.json 2> gpurun_out/b_vitb_$TAG.err
for f in gpurun_out/b_vitl_$TAG.json gpurun_out/b_vitb_$TAG.json; do python scripts/show_bench.py $f; done
