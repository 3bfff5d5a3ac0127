#!/bin/bash
# Pair-GEMM per-launch duration + tensor-pipe activity at locked base clocks under
# PLORA_DEBUG_FLAGS variants given as arguments (default: 0 8 2 1).
FLAGS=${@:-0 8 2 1}
for f in $FLAGS; do
  PLORA_DEBUG_FLAGS=$f ncu --clock-control base --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    -k regex:plora_gemm_pair --csv python tools/gemm_once.py 2>/dev/null | grep -E "gpu__time|tensor" | \
    awk -F'","' -v f=$f '{gsub(/"/,"",$NF); printf "%s %s %s\n", f, $(NF-2), $NF}'
done
