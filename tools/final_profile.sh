#!/bin/bash
# End-of-session evidence on one B200: default bench line, one-step launch list (duration + DRAM
# bytes, timed step only via PLORA_PROFILE_RANGE), and an ncu --set full capture of the first
# pair-GEMM launch of the timed step.  Usage: tools/final_profile.sh <tag>
TAG=${1:-final}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -c 600 gpurun_out/${TAG}_bench.json
PLORA_PROFILE_RANGE=1 timeout 1500 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_launch_summary.json | head -12
PLORA_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:plora_gemm_pair -c 1 -o gpurun_out/${TAG}_pair_full -f python bench.py --steps 1 --warmup 3 \
  --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/${TAG}_pair_full.ncu-rep
