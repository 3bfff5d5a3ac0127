cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 2 -c 1 -o gpurun_out/ap_swiglu_gemm python tools/bench_swiglu.py > gpurun_out/ap.log 2>&1; echo rc=$?
