cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v_build.log 2>&1; echo build_rc=$?
timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/v_pytest.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/v_bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','gpu_launches','step_mode')}, d['e2e']['value'], d['roofline']['frac'], d['clocks'], d.get('cpu_baseline',{}).get('value'), d.get('dropin_api',{}).get('value'), list(d['roofline'].keys()))
"
timeout 900 python bench.py --impl reference > gpurun_out/v_ref.json 2>/dev/null; echo ref_rc=$?; tail -c 250 gpurun_out/v_ref.json
