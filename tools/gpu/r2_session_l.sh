cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2l_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/r2l_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/r2l_smoke.log
bash tools/ab_run.sh 2 > gpurun_out/r2l_ab.log 2>&1; cat gpurun_out/r2l_ab.log
timeout 300 python tools/bench_lora.py > gpurun_out/r2l_bench_lora.log 2>&1; tail -5 gpurun_out/r2l_bench_lora.log
