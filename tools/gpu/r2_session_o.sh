cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in default evf swd1 swd3; do
  if [ $v = default ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
  echo "== $v"; PLORA_LIB=$L timeout 300 python tools/bench_swiglu.py 2>&1 | head -3
done; done
for v in default evf; do
  if [ $v = default ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
  PLORA_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pair_kernel -c 3 python tools/bench_swiglu.py > gpurun_out/r2o_ncu_$v.log 2>&1
  grep -E "pair_kernel|duration|dram__bytes|hit_rate" gpurun_out/r2o_ncu_$v.log | head -16
done
