cd $GRAFT_REPO_ROOT
for i in 1 2; do
  for v in default reg200; do
    if [ $v = default ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
    PLORA_LIB=$L timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/z3_$v.json 2> gpurun_out/z3_$v.err
    python -c "
import json,sys; d=json.loads(open('gpurun_out/z3_$v.json').read()); print('$v', round(d['value']), d['clocks']['sm_mhz'], d['kernels'].get('swiglu_segred',{}).get('ms_total'), d['gemm_shapes']['gateup+swiglu N14336K4096k'])" || tail -5 gpurun_out/z3_$v.err
  done
  (cd build/ab_base && timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('base', round(d['value']), d['clocks']['sm_mhz'])")
done
