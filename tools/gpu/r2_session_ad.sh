cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --config qwen2.5-3b --no-cpu-baseline --steps 5 > gpurun_out/ad_c2.json 2> gpurun_out/ad_c2.err; echo c2_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/ad_c2.json').read()); print('C2', round(d['value']), d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['roofline']['step_frac_of_burst_peak'])" || tail -3 gpurun_out/ad_c2.err
timeout 1500 python tools/split_projection.py --gpus 8 --steps 5 --warmup 2 --graph --kernels > gpurun_out/ad_split8_kernels.log 2>&1; echo rc=$?
python - <<'PY'
import json
for line in open('gpurun_out/ad_split8_kernels.log'):
    if line.startswith('{"job"'):
        d = json.loads(line); k = d['kernels']
        print(d['job'], d['T'], d['ms_per_step'], {x: k[x]['ms'] for x in ('gemm','shrink','segred','dual','swiglu_segred','adamw') if x in k})
    elif line.startswith('{"gpus"'):
        print(line.strip())
PY
