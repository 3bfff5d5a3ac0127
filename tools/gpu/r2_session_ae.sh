cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_adamw.py tests/test_gpu_graph.py -x -q 2>&1 | tail -2
for i in 1 2; do
  timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/ae_new_$i.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ae_new_$i.json').read()); print('new ', round(d['value']), d['clocks']['sm_mhz'], d['kernels']['adamw'])"
  (cd build/ab_base && timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null > ../../gpurun_out/ae_base_$i.json)
  python -c "
import json; d=json.loads(open('gpurun_out/ae_base_$i.json').read()); print('base', round(d['value']), d['clocks']['sm_mhz'], d['kernels']['adamw'])"
done
