set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/r2a_bench.json
timeout 600 python bench.py --gpus 2 --config qwen2.5-3b --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2a_bench2.json 2> gpurun_out/r2a_bench2.err; echo bench2_rc=$?
tail -c 1500 gpurun_out/r2a_bench2.json; tail -5 gpurun_out/r2a_bench2.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r2a_ref.json 2>&1; echo ref_rc=$?
tail -c 1200 gpurun_out/r2a_ref.json
