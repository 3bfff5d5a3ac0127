cd $GRAFT_REPO_ROOT
i=0
for o in "--eager" "--eager --no-fuse-dual" "--eager --no-fuse-swiglu-bwd" ""; do
  i=$((i+1))
  timeout 900 python tools/c4_shard_bench.py --tp 8 --steps 3 --warmup 2 --depths 64 $o > gpurun_out/ak_c4_$i.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ak_c4_$i.log').read().strip().splitlines()[-1]); print('$o', d['ms_per_step_rank'], d['per_gpu_tokens_per_s_if_comm_hidden'], d['per_gpu_base_gemm_tflops'])" || tail -2 gpurun_out/ak_c4_$i.log
done
