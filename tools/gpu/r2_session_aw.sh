cd $GRAFT_REPO_ROOT
PLORA_PROFILE_RANGE=1 PLORA_RECORDS_OUT=gpurun_out/aw_records.json timeout 1500 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/aw_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/aw_ncu_bench.log 2>&1; echo ncu_rc=$?
python tools/dram_by_shape.py gpurun_out/aw_launches.csv gpurun_out/aw_records.json gpurun_out/aw_dram_by_shape.json gpurun_out/aw_gemm_traffic.json | head -8
python tools/summarize_launches.py gpurun_out/aw_launches.csv gpurun_out/aw_launch_summary.json | head -14
timeout 1500 python tools/split_projection.py --gpus 1,2,4,8 --steps 5 --warmup 2 --graph > gpurun_out/aw_split.log 2>&1; echo split_rc=$?
grep -v '"projection"' gpurun_out/aw_split.log | tail -4
