#!/bin/bash
# Quick check: attention / runtime / headline GPU tests, then the default bench (fast only).
# Usage: bash scripts/gpu_quick2.sh TAG [pytest -k expr]
TAG=${1:-x}; K=${2:-"attention or runtime or headline"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_q_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q_$TAG.log
tail -3 gpurun_out/pytest_q_$TAG.log
timeout 300 python bench.py --no-cpu-baseline --only-main --steps 100 > gpurun_out/b_q_$TAG.json 2> gpurun_out/b_q_$TAG.err
python scripts/show_bench.py gpurun_out/b_q_$TAG.json
