cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_dual.py tests/test_gpu_adamw.py tests/test_gpu_graph.py -x -q 2>&1 | tail -2
for i in 1 2; do
  timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/ag_plain_$i.json 2>/dev/null
  timeout 400 python bench.py --no-cpu-baseline --steps 5 --overlap-k5 > gpurun_out/ag_ovl_$i.json 2>/dev/null
done
python -c "
import json
for f in ['ag_plain_1','ag_ovl_1','ag_plain_2','ag_ovl_2']:
    try:
        d=json.loads(open('gpurun_out/%s.json'%f).read()); print(f, round(d['value']), d['clocks']['sm_mhz'], d['step_mode'])
    except Exception as e: print(f, 'ERR', e)
"
for o in "" "--overlap-k5"; do timeout 900 python tools/split_projection.py --gpus 8 --steps 5 --warmup 2 --graph $o 2>&1 | grep '"gpus"' | head -1; done
