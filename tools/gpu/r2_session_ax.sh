cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dual.py tests/test_gpu_graph.py -x -q > gpurun_out/ax_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/ax_pytest.log
for i in 1 2; do
  for v in fixpdl nofixpdl; do
    if [ $v = fixpdl ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
    PLORA_LIB=$L timeout 900 python tools/split_projection.py --gpus 8 --steps 3 --warmup 2 --graph --kernels 2>&1 | grep '"job"' | python -c "
import sys, json
tot=0; st=0
for l in sys.stdin:
    d=json.loads(l); tot+=d['kernels']['dual']['ms']; st+=d['ms_per_step']
print('$v', 'sum over 8 ranks: dual ms', round(tot,2), 'step ms', round(st,2))"
  done
done
for i in 1 2; do
  for v in fixpdl nofixpdl; do
    if [ $v = fixpdl ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
    PLORA_LIB=$L timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), d['clocks']['sm_mhz'], d['kernels']['dual']['ms_total'])"
  done
done
