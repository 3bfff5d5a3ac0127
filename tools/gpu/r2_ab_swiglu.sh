cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in A B; do echo "== $v"; PLORA_LIB=build/ab/libplora_$v.so timeout 300 python tools/bench_swiglu.py; done; done
PLORA_LIB=build/ab/libplora_B.so timeout 600 python -m pytest tests/test_gpu_linear.py tests/test_gpu_gemm.py -x -q 2>&1 | tail -3
