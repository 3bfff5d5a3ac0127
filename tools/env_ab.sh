#!/bin/bash
# On the GPU box: alternate bench.py of this tree under two env settings, N rounds.
# Usage: tools/env_ab.sh N "VAR=a" "VAR=b" [bench args]
N=$1; A=$2; B=$3; shift 3
for i in $(seq $N); do
  for tag in A B; do
    if [ $tag = A ]; then E=$A; else E=$B; fi
    env $E timeout 400 python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '$E', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
  done
done
