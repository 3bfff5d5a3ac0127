#!/bin/bash
# On the GPU box: alternate bench.py over several libplora builds, N rounds.
# Usage: tools/lib_sweep.sh N lib1.so lib2.so ...  (the in-tree library: "tree")
N=$1; shift
for i in $(seq $N); do
  for L in "$@"; do
    if [ "$L" = tree ]; then unset PLORA_LIB; else export PLORA_LIB=$L; fi
    timeout 400 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
  done
done
unset PLORA_LIB
