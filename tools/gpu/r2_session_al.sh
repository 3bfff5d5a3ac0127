cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in default swd1 swd3; do
  if [ $v = default ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
  echo "== $v $(PLORA_LIB=$L timeout 300 python tools/bench_swiglu.py 2>&1 | head -1)"
done; done
for i in 1 2; do for v in default swd3; do
  if [ $v = default ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
  PLORA_LIB=$L timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/al_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/al_$v.json').read()); print('$v', round(d['value']), d['clocks']['sm_mhz'], d['gemm_shapes']['gateup+swiglu N14336K4096k']['tflops'])"
done; done
