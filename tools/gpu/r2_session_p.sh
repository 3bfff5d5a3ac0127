cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dual.py -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo bench_rc=$?
tail -3 gpurun_out/r2p_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2p_bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','gpu_launches')}, d['clocks'], d['kernels'], d['lora_shapes'])
"
for i in 1 2; do
  timeout 400 python bench.py --no-cpu-baseline --steps 5 --no-fuse-dual 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('sep  ', round(d['value']), d['clocks']['sm_mhz'])"
  timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('fused', round(d['value']), d['clocks']['sm_mhz'], d['kernels'].get('dual'))"
done
