#!/bin/bash
# A/B of the GEMM kernels at locked base clocks: per-launch gpu__time_duration for
# build/libplora_base.so vs the in-tree libplora.so.  Usage: tools/ncu_ab.sh [script]
S=${1:-tools/gemm_once.py}
for tag in base new; do
  if [ $tag = base ]; then export PLORA_LIB=build/libplora_base.so; else unset PLORA_LIB; fi
  ncu --clock-control base --metrics gpu__time_duration.sum -k regex:plora_gemm --csv python $S 2>/dev/null \
    | grep gpu__time_duration | awk -F'","' -v t=$tag '{print t, $5, $NF}' | sed 's/"//g'
done
