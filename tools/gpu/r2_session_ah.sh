cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_dual.py tests/test_gpu_adamw.py tests/test_gpu_graph.py tests/test_gpu_model.py -x -q > gpurun_out/ah_pytest.log 2>&1; echo rc=$?; tail -3 gpurun_out/ah_pytest.log
