cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for v in default evf swd3; do
  if [ $v = default ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
  echo "== $v $(PLORA_LIB=$L timeout 300 python tools/bench_swiglu.py 2>&1 | head -1)"
done; done 2>&1 | tee gpurun_out/r2o2.log
