set -x
cd $GRAFT_REPO_ROOT
timeout 900 python tools/split_projection.py --gpus 8 --steps 5 --warmup 2 --kernels > gpurun_out/r2c_split8.log 2>&1; echo rc=$?
grep '"kernels"' gpurun_out/r2c_split8.log | head -2
timeout 900 python -m pytest tests/test_gpu_model_c3.py -x -q -s > gpurun_out/r2c_model_c3.log 2>&1; echo rc=$?
tail -5 gpurun_out/r2c_model_c3.log
