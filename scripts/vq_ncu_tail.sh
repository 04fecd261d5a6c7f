timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:'vq_final|vq_rerank|VqEpi' -c 12 --csv python scripts/microbench.py --reps 3 2>/dev/null \
  | grep -i "gpu__time" | awk -F'","' '{print $NF, substr($5,1,40)}'
