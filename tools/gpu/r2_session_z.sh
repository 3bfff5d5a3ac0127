cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_swiglu_segred.py tests/test_gpu_elementwise.py tests/test_gpu_linear.py tests/test_gpu_model.py -x -q 2>&1 | tail -3
PLORA_LIB=build/libplora_reg200.so timeout 900 python -m pytest tests/test_gpu_linear.py -x -q 2>&1 | tail -1
for i in 1 2; do
  for v in default reg200 reg200s1; do
    if [ $v = default ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
    PLORA_LIB=$L timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['clocks']['sm_mhz'], d['kernels'].get('swiglu_segred',{}).get('ms_total'), d['gemm_shapes']['gateup+swiglu N14336K4096k'])"
  done
  (cd build/ab_base && timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('base', round(d['value']), d['clocks']['sm_mhz'])")
done
