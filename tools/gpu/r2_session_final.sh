cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin_pytest.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/fin_bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','gpu_launches')}, d['e2e']['value'], d['roofline']['frac'], d['clocks'], d.get('cpu_baseline',{}).get('value'), d.get('dropin_api',{}).get('value'))
"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_ref.json 2>/dev/null; tail -c 300 gpurun_out/fin_ref.json
PLORA_PROFILE_RANGE=1 PLORA_RECORDS_OUT=gpurun_out/fin_records.json timeout 1500 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/fin_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu_bench.log 2>&1; echo ncu_rc=$?
python tools/dram_by_shape.py gpurun_out/fin_launches.csv gpurun_out/fin_records.json gpurun_out/fin_dram_by_shape.json gpurun_out/fin_gemm_traffic.json | head -8
python tools/summarize_launches.py gpurun_out/fin_launches.csv gpurun_out/fin_launch_summary.json > /dev/null
PLORA_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"plora_gemm_pair_kernel<0, 2, 2>|plora_gemm_pair_kernel<false, 2, 2>" -c 1 -o gpurun_out/fin_swiglu_gemm -f python bench.py --steps 1 --warmup 3 \
  --no-cpu-baseline > /dev/null 2>&1; echo ncu_full_rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"dual_kernel" -s 2 -c 1 \
     -o gpurun_out/fin_dual python tools/dbg/dual_one.py 14336 > /dev/null 2>&1; echo ncu_dual_rc=$?
timeout 1500 python tools/split_projection.py --gpus 1,2,4,8 --steps 5 --warmup 2 --graph > gpurun_out/fin_split.log 2>&1; echo split_rc=$?
grep -v '"projection"' gpurun_out/fin_split.log | tail -4
