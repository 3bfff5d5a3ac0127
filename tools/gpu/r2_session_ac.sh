cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dual.py tests/test_gpu_model.py tests/test_gpu_model_c3.py -x -q 2>&1 | tail -3
for i in 1 2; do
  timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/ac_new_$i.json 2>gpurun_out/ac_new_$i.err
  python -c "
import json; d=json.loads(open('gpurun_out/ac_new_$i.json').read()); print('multi', round(d['value']), d['clocks']['sm_mhz'], d['kernels'].get('dual'), {k:v for k,v in d['lora_shapes'].items() if k.startswith('dual')})" || tail -3 gpurun_out/ac_new_$i.err
  (cd build/ab_base && timeout 400 python bench.py --no-cpu-baseline --steps 5 2>/dev/null > ../../gpurun_out/ac_base_$i.json)
  python -c "
import json; d=json.loads(open('gpurun_out/ac_base_$i.json').read()); print('base ', round(d['value']), d['clocks']['sm_mhz'])"
done
timeout 1500 python tools/split_projection.py --gpus 8 --steps 5 --warmup 2 --graph 2>&1 | grep '"gpus"' | head -1
