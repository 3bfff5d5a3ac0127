cd $GRAFT_REPO_ROOT
timeout 300 python tools/bench_lora.py > gpurun_out/r2n_bench_lora.log 2>&1; tail -5 gpurun_out/r2n_bench_lora.log | head -4
PLORA_LIB=build/libplora_skall.so timeout 300 python tools/bench_lora.py > gpurun_out/r2n_bench_lora_skall.log 2>&1; tail -5 gpurun_out/r2n_bench_lora_skall.log | head -4
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err; echo bench_rc=$?
tail -3 gpurun_out/r2n_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2n_bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','gpu_launches')}, d['e2e']['value'], d['roofline'], d['clocks'], d['kernels'], d['kernel_stats'], d['lora_shapes'])
"
for i in 1 2 3; do
  (cd build/ab_base && timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('A', round(d['value']), d['clocks']['sm_mhz'])")
  timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B', round(d['value']), d['clocks']['sm_mhz'], d['kernels']['shrink'], d['kernels']['segred'])"
  PLORA_LIB=build/libplora_skall.so timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C', round(d['value']), d['clocks']['sm_mhz'], d['kernels']['shrink'], d['kernels']['segred'])"
done
