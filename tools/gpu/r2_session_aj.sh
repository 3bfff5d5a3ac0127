cd $GRAFT_REPO_ROOT
for o in "" "--no-fuse-dual" "--no-fuse-swiglu-bwd" "--eager"; do
  timeout 900 python tools/c4_shard_bench.py --tp 8 --steps 3 --warmup 2 --depths 64 $o > gpurun_out/aj_c4.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/aj_c4.log').read().strip().splitlines()[-1]); print('$o', d['ms_per_step_rank'], d['per_gpu_tokens_per_s_if_comm_hidden'], d['per_gpu_base_gemm_tflops'], d['measured'])" || tail -3 gpurun_out/aj_c4.log
done
