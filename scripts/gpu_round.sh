#!/bin/bash
# One GPU session: parity tests, bench line, ncu launch list + full captures of the hot kernels.
# Usage: bash scripts/gpu_round.sh TAG
TAG=${1:-rXX}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep 'Model name' >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$TAG.csv python scripts/profile_forward.py --iters 2 > gpurun_out/launch_$TAG.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:'tc_gemm|attention_tcp|vq_finalize|layernorm' -c 9 \
   -o gpurun_out/full_$TAG python scripts/profile_forward.py --iters 1 > gpurun_out/full_$TAG.log 2>&1
ls gpurun_out | tail -20
timeout 600 python scripts/bench_ranks.py --config vitb --n 1 2 4 8 > gpurun_out/ranks_$TAG.jsonl 2> gpurun_out/ranks_$TAG.err
timeout 900 python bench.py --config gpt2s --steps 20 > gpurun_out/b_gpt2s_$TAG.json 2> gpurun_out/b_gpt2s_$TAG.err
timeout 1200 python bench.py --config gpt2m --steps 10 > gpurun_out/b_gpt2m_$TAG.json 2> gpurun_out/b_gpt2m_$TAG.err
