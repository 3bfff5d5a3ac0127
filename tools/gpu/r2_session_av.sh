cd $GRAFT_REPO_ROOT
for v in joint oldplan; do
  if [ $v = joint ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
  PLORA_LIB=$L timeout 900 python tools/split_projection.py --gpus 8 --steps 3 --warmup 2 --graph --kernels 2>&1 | grep '"job"' | sed "s/^/$v /" > gpurun_out/av_$v.log
done
