cd $GRAFT_REPO_ROOT
for v in default swb4 swb6 swb12 swb16 swbm16; do
  if [ $v = default ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
  t=$(PLORA_LIB=$L timeout 300 python tools/bench_swiglu.py 2>&1 | head -1)
  PLORA_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:pair_kernel -s 2 -c 1 python tools/bench_swiglu.py > gpurun_out/am_$v.log 2>&1
  echo "== $v $t | $(grep -E 'dram__bytes_read|dram__bytes_write|gpu__time' gpurun_out/am_$v.log | awk '{print $NF}' | tr '\n' ' ')"
done
