#!/bin/bash
# Attention diagnostics: PV / softmax probes and the tcp kernel timeline.  Usage: bash scripts/gpu_attn_diag.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
(cd scripts/probes && timeout 120 ./pv_probe) > gpurun_out/pv_probe_$TAG.txt 2>&1
(cd scripts/probes && timeout 120 ./softmax_probe) > gpurun_out/softmax_probe_$TAG.txt 2>&1
timeout 300 python scripts/attn_trace.py 1 > gpurun_out/attn_trace_$TAG.txt 2>&1
tail -5 gpurun_out/pv_probe_$TAG.txt gpurun_out/softmax_probe_$TAG.txt
