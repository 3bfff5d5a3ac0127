cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_streamk.py tests/test_gpu_linear.py tests/test_gpu_graph.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err; echo bench_rc=$?
tail -3 gpurun_out/r2m_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2m_bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','gpu_launches')}, d['e2e']['value'], d['roofline'], d['clocks'], d['kernels'], d['kernel_stats'], d['lora_shapes'])
"
bash tools/ab_run.sh 3 > gpurun_out/r2m_ab.log 2>&1; cat gpurun_out/r2m_ab.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"plora_gemm_kernel|segred" -s 4 -c 2 \
     -o gpurun_out/ncu_shrink_c3_4096 python tools/dbg/lora_one.py c3 4096 whole > gpurun_out/ncu_shrink.log 2>&1; echo ncu_rc=$?
