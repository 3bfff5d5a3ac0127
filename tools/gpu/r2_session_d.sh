set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_linear.py -k "c3_widths" -x -q > gpurun_out/r2d_c3w.log 2>&1; echo rc=$?
tail -15 gpurun_out/r2d_c3w.log
timeout 900 python -m pytest tests/test_gpu_model_c3.py -x -q -s > gpurun_out/r2d_model_c3.log 2>&1; echo rc=$?
grep -E "block|C3 shapes" gpurun_out/r2d_model_c3.log | head -20
