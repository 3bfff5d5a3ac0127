#!/bin/bash
# On the GPU box: alternate bench.py over several environment settings, N rounds.
# Usage: tools/env_sweep.sh N "VAR=a" "VAR=b" ...
N=$1; shift
for i in $(seq $N); do
  for E in "$@"; do
    env $E timeout 400 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$E', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])
except Exception as e:
    print('$E', 'failed')"
  done
done
