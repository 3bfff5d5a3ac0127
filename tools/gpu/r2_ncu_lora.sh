cd $GRAFT_REPO_ROOT
for cfg in "split8 4096 sk" "c3 4096 sk" "c3 4096 whole"; do
  set -- $cfg
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:plora_gemm_kernel -s 4 -c 2 \
     -o gpurun_out/ncu_lora_$1_$2_$3 python tools/dbg/lora_one.py $1 $2 $3 > gpurun_out/ncu_lora_$1_$2_$3.log 2>&1
  echo "$cfg rc=$?"
done
