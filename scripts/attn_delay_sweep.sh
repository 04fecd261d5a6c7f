#!/bin/bash
# Attention experiment: start pipeline 1 of the two-pipeline kernel late (ns), back-to-back timing
for d in ${VALUES:-0 500 1000 1500 2000 3000}; do
  ASTRA_ATTN_PIPE_DELAY=$d timeout 300 python scripts/microbench.py --reps 50 --only attention 2>&1 | grep '"attention"' | grep -E 'rank_of_(1|2)"' | sed "s/^/delay=$d /" | cut -c1-160
done
