for m in 0 1 2 4; do
  ASTRA_VQ_GEMM_DEBUG=$m timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:VqEpilogue -s 10 -c 5 --csv python scripts/microbench.py --reps 5 2>/dev/null | grep -i "gpu__time" | awk -F'","' -v m=$m '{print "mode", m, $NF}' | head -5
done
