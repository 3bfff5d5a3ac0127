cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"dual" -s 4 -c 2 \
     -o gpurun_out/ncu_dual_4096 python tools/dbg/dual_one.py 4096 > gpurun_out/ncu_dual.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_dual.log
