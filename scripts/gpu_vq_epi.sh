#!/bin/bash
# VQ records-epilogue check: bit-exact VQ tests, microbench, per-launch GEMM times (ncu)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_vq_gpu.py -x -q 2>&1 | tail -3
timeout 300 python scripts/microbench.py --reps 30 2>&1 | grep vq_encode
bash scripts/vq_gemm_isolate.sh
