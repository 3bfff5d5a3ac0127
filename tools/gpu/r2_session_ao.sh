cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_swiglu_segred.py tests/test_gpu_dual.py -x -q 2>&1 | tail -1
timeout 1200 python tools/overfit_check.py --steps 40 > gpurun_out/ao_overfit.log 2>&1; echo rc=$?; tail -20 gpurun_out/ao_overfit.log
