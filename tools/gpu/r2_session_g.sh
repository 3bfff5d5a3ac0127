set -x
cd $GRAFT_REPO_ROOT
timeout 1200 python tools/split_projection.py --gpus 8 --steps 5 --warmup 2 --kernels > gpurun_out/r2g_split8_kernels.log 2>&1; echo rc=$?
timeout 1200 python tools/split_projection.py --gpus 1,2,4,8 --steps 5 --warmup 2 --graph > gpurun_out/r2g_split_graph.log 2>&1; echo rc=$?
grep -v '"projection"' gpurun_out/r2g_split_graph.log | tail -12
