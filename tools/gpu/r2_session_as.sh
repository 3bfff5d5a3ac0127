cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/as_pytest.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/as_pytest.log
for i in 1 2; do
  for v in default nopsk; do
    if [ $v = default ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
    PLORA_LIB=$L timeout 900 python tools/split_projection.py --gpus 4,8 --steps 5 --warmup 2 --graph 2>&1 | grep '"gpus"' | sed "s/^/$v /" | cut -c1-160
  done
done
