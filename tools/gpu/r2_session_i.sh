set -x
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_pytest.log 2>&1; echo rc=$?
tail -4 gpurun_out/r2i_pytest.log
timeout 900 python tools/split_projection.py --gpus 8 --steps 5 --warmup 2 --kernels > gpurun_out/r2i_split8_kernels.log 2>&1; echo rc=$?
grep '"job"' gpurun_out/r2i_split8_kernels.log | head -2 | cut -c1-400
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2i_bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','gpu_launches')}, d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['kernels'])
"
timeout 1200 python tools/split_projection.py --gpus 1,2,4,8 --steps 5 --warmup 2 --graph > gpurun_out/r2i_split_graph.log 2>&1; echo rc=$?
grep -v '"projection"' gpurun_out/r2i_split_graph.log | tail -5
