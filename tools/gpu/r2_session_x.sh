cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2x_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2x_pytest.log
for i in 1 2; do
  PLORA_LIB=build/libplora_nopdl.so timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nopdl', round(d['value']), d['clocks']['sm_mhz'])"
  timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pdl  ', round(d['value']), d['clocks']['sm_mhz'])"
done
for L in build/libplora_nopdl.so paper_2508_02932_b200/libplora.so; do
  PLORA_LIB=$L timeout 900 python tools/split_projection.py --gpus 8 --steps 5 --warmup 2 --graph 2>&1 | grep '"gpus"' | head -1
done
