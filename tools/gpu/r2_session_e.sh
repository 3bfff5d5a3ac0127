set -x
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2e_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/r2e_pytest.log
timeout 600 python -m pytest tests/test_gpu_model_c3.py -x -q -s 2>&1 | grep -E "adapter|passed|failed"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2e_bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','step_mode','gpu_launches')}, d['e2e']['value'], d['eager']['value'], d['roofline']['frac'], d['clocks'])
"
tail -3 gpurun_out/r2e_bench.err
timeout 1200 python tools/split_projection.py --gpus 1,8 --steps 5 --warmup 2 --graph --kernels > gpurun_out/r2e_split_graph.log 2>&1; echo split_rc=$?
grep -v '"projection"' gpurun_out/r2e_split_graph.log | tail -12
