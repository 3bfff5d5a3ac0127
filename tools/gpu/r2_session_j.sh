cd $GRAFT_REPO_ROOT
for mode in "" "--whole-lora"; do
timeout 900 python tools/split_projection.py --gpus 1,8 --steps 3 --warmup 2 --kernels $mode > gpurun_out/r2j_split_kernels$mode.log 2>&1; echo rc=$?
done
