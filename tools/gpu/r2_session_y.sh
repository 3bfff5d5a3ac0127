cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_swiglu_segred.py -x -q 2>&1 | tail -3
for i in 1 2; do
  timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('fused', round(d['value']), d['clocks']['sm_mhz'], d['kernels'].get('swiglu_segred'))"
  (cd build/ab_base && timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('base ', round(d['value']), d['clocks']['sm_mhz'])")
done
