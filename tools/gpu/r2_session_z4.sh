cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
  timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/z4_new_$i.json 2> gpurun_out/z4_new_$i.err
  python -c "
import json; d=json.loads(open('gpurun_out/z4_new_$i.json').read()); print('new ', round(d['value']), d['clocks']['sm_mhz'], d['kernels'].get('swiglu_segred',{}).get('ms_total'), d['gemm_shapes']['gateup+swiglu N14336K4096k']['tflops'])"
  (cd build/ab_base && timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null > ../../gpurun_out/z4_base_$i.json)
  python -c "
import json; d=json.loads(open('gpurun_out/z4_base_$i.json').read()); print('base', round(d['value']), d['clocks']['sm_mhz'], d['gemm_shapes']['gateup+swiglu N14336K4096k']['tflops'])"
done
