set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_tp.py tests/test_gpu_tp_dist.py tests/test_gpu_packed_linear_op.py tests/test_bench_launch.py -x -q > gpurun_out/r2b_pytest_tp.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/r2b_pytest_tp.log
timeout 600 python -c "
import bench, json
print(json.dumps(bench.dropin_api_sample('llama-3.1-8b')))
print(json.dumps(bench.dropin_api_sample('llama-3.1-8b')))
" > gpurun_out/r2b_dropin.log 2>&1; echo dropin_rc=$?; cat gpurun_out/r2b_dropin.log | tail -3
timeout 1200 python tools/split_projection.py --steps 5 --warmup 2 > gpurun_out/r2b_split.log 2>&1; echo split_rc=$?
head -6 gpurun_out/r2b_split.log
PLORA_PROFILE_RANGE=1 PLORA_RECORDS_OUT=gpurun_out/r2b_records.json timeout 1500 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/r2b_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_ncu_bench.log 2>&1; echo ncu_rc=$?
python tools/dram_by_shape.py gpurun_out/r2b_launches.csv gpurun_out/r2b_records.json gpurun_out/r2b_dram_by_shape.json gpurun_out/r2b_gemm_traffic.json
