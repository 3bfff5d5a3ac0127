#!/bin/bash
# On the GPU box: alternate bench.py of build/ab_base (A) and this tree (B), N rounds.
N=${1:-2}
shift
for i in $(seq $N); do
  (cd build/ab_base && timeout 400 python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('A', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])")
  timeout 400 python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
done
