#!/bin/bash
# Pair-GEMM per-launch duration at locked base clocks under PLORA_DEBUG_FLAGS variants
# (0 normal, 4 TMEM drain only, 1 no epilogue, 2 no operand traffic).
for f in 0 4 1 2; do
  PLORA_DEBUG_FLAGS=$f ncu --clock-control base --metrics gpu__time_duration.sum -k regex:plora_gemm_pair --csv \
    python tools/gemm_once.py 2>/dev/null | grep gpu__time | awk -F'","' -v f=$f '{gsub(/"/,"",$NF); print f, $NF}'
done
