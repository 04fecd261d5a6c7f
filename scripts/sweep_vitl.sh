#!/bin/bash
# BASELINE config #4: ViT-L/16@384 (T=576, B=32) over VQ groups G x codebook size K, one bench
# line per point -> gpurun_out/sweep_vitl.jsonl (copy to profiles/ to commit).
mkdir -p gpurun_out
out=gpurun_out/sweep_vitl.jsonl
: > $out
for g in 1 16 32; do
  for k in 256 1024 4096; do
    timeout 900 python bench.py --config vitl --groups $g --codebook $k --steps ${STEPS:-20} \
        --warmup 3 ${EXTRA:-} >> $out 2>> gpurun_out/sweep_vitl.err || echo "{\"failed\": \"G=$g K=$k\"}" >> $out
  done
done
wc -l $out
