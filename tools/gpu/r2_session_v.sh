cd $GRAFT_REPO_ROOT
timeout 1500 python tools/split_projection.py --gpus 1,8 --steps 5 --warmup 2 --graph --kernels > gpurun_out/r2v_split8_kernels.log 2>&1; echo rc=$?
tail -2 gpurun_out/r2v_split8_kernels.log | cut -c1-300
python - <<'PY'
import json
for line in open('gpurun_out/r2v_split8_kernels.log'):
    if line.startswith('{"job"'):
        d = json.loads(line); k = d['kernels']
        print(d['job'], d['T'], d['ms_per_step'], {x: k[x]['ms'] for x in ('gemm','shrink','segred','dual','adamw') if x in k}, {x: k[x]['ms'] for x in k if x.startswith('dual[')})
    elif line.startswith('{"gpus"'):
        print(line.strip())
PY
