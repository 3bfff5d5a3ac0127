cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_pair_streamk.py -x -q 2>&1 | tail -15
