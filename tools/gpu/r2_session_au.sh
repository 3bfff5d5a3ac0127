cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dual.py tests/test_abi.py -x -q > gpurun_out/au_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/au_pytest.log
for i in 1 2; do
  for v in joint oldplan; do
    if [ $v = joint ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
    PLORA_LIB=$L timeout 900 python tools/split_projection.py --gpus 8 --steps 5 --warmup 2 --graph 2>&1 | grep '"gpus"' | head -1 | sed "s/^/$v /" | cut -c1-170
  done
done
for i in 1 2; do
  for v in joint oldplan; do
    if [ $v = joint ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
    PLORA_LIB=$L timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), d['clocks']['sm_mhz'], d['kernels']['dual'])"
  done
done
PLORA_LIB=paper_2508_02932_b200/libplora.so timeout 900 python tools/split_projection.py --gpus 8 --steps 3 --warmup 2 --graph --kernels 2>&1 | grep '"job"' | head -3 | cut -c1-400
