#!/bin/bash
# Round artefacts: ViT-L G x K sweep (config #4), GPT-2 small/medium prefill lines (configs #3/#5),
# VQ decode microbenchmark, per-rank loopback times + measured-comm table.  Usage: bash scripts/gpu_artifacts.sh TAG
TAG=${1:-rXX}
mkdir -p gpurun_out
timeout 600 python scripts/bench_ranks.py --config vitb --n 1 2 4 8 > gpurun_out/ranks_$TAG.jsonl 2> gpurun_out/ranks_$TAG.err
python scripts/measure_comms.py --ranks gpurun_out/ranks_$TAG.jsonl --out gpurun_out/comms_vitb_$TAG.csv > /dev/null 2>&1
timeout 300 python scripts/vq_decode_bench.py > gpurun_out/decode_$TAG.jsonl 2> gpurun_out/decode_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:'vq_decode|layernorm' -c 12 --csv --log-file gpurun_out/decode_ncu_$TAG.csv python scripts/vq_decode_bench.py --reps 2 > /dev/null 2>&1
timeout 900 python bench.py --config gpt2s --steps 20 > gpurun_out/b_gpt2s_$TAG.json 2> gpurun_out/b_gpt2s_$TAG.err
timeout 1200 python bench.py --config gpt2m --steps 10 > gpurun_out/b_gpt2m_$TAG.json 2> gpurun_out/b_gpt2m_$TAG.err
STEPS=10 timeout 3600 bash scripts/sweep_vitl.sh
cp gpurun_out/sweep_vitl.jsonl gpurun_out/sweep_vitl_$TAG.jsonl
ls -la gpurun_out | tail -20
