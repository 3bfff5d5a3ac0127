cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"plora_gemm_kernel" -s 4 -c 2 \
     -o gpurun_out/ncu_split8_sk python tools/dbg/lora_one.py split8 4096 sk > gpurun_out/ncu_split8.log 2>&1; echo ncu_rc=$?
tail -2 gpurun_out/ncu_split8.log
