cd $GRAFT_REPO_ROOT
timeout 1800 python tools/c4_shard_bench.py --tp 8 --steps 3 --warmup 2 > gpurun_out/ai_c4.log 2>&1; echo rc=$?; tail -3 gpurun_out/ai_c4.log
