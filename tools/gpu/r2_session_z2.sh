cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_swiglu_segred.py tests/test_gpu_elementwise.py tests/test_gpu_linear.py tests/test_gpu_model.py -x -q 2>&1 | tail -25
timeout 400 python bench.py --no-cpu-baseline --steps 2 --warmup 3 2>&1 | tail -12
