set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_pytest.log 2>&1; echo pytest_rc=$?
tail -6 gpurun_out/r2f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo smoke_rc=$?; tail -3 gpurun_out/r2f_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo bench_rc=$?
tail -c 4000 gpurun_out/r2f_bench.json; tail -3 gpurun_out/r2f_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_ref.json 2> gpurun_out/r2f_ref.err; echo ref_rc=$?
tail -c 1500 gpurun_out/r2f_ref.json
