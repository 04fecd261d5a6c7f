#!/bin/bash
# launch list of one rank of an 8-way ViT-B split (loopback exchange), 2 forwards
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_rank8.csv python scripts/profile_forward.py --rank-of ${1:-8} --iters 2 > gpurun_out/launch_rank8.log 2>&1
python scripts/ncu_summary.py --launches gpurun_out/launches_rank8.csv
