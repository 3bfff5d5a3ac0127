cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_adamw.py tests/test_gpu_model.py tests/test_gpu_model_c3.py tests/test_gpu_tp.py tests/test_gpu_dual.py -x -q 2>&1 | tail -2
for i in 1 2; do
  timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/af_new_$i.json 2>/dev/null
  (cd build/ab_base && timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null > ../../gpurun_out/af_base_$i.json)
done
python -c "
import json
for f in ['af_new_1','af_base_1','af_new_2','af_base_2']:
    d=json.loads(open('gpurun_out/%s.json'%f).read()); print(f, round(d['value']), d['clocks']['sm_mhz'], d['kernels'].get('dual',{}).get('ms_total'), d['kernels'].get('shrink',{}).get('launches'), d['kernels'].get('segred',{}).get('launches'))
"
