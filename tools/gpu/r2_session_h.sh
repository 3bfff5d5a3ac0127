set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_streamk.py -x -q > gpurun_out/r2h_streamk.log 2>&1; echo rc=$?
tail -30 gpurun_out/r2h_streamk.log
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_lorapack.py tests/test_gpu_model.py tests/test_gpu_graph.py -x -q > gpurun_out/r2h_linear.log 2>&1; echo rc=$?
tail -30 gpurun_out/r2h_linear.log
timeout 900 python tools/split_projection.py --gpus 8 --steps 5 --warmup 2 --kernels > gpurun_out/r2h_split8_kernels.log 2>&1; echo rc=$?
grep '"job"' gpurun_out/r2h_split8_kernels.log | head -3 | cut -c1-600
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2h_bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','gpu_launches')}, d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['kernels'])
"
tail -3 gpurun_out/r2h_bench.err
