cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dual.py -x -q 2>&1 | tail -3
PLORA_LIB=build/libplora_dualn64.so timeout 900 python -m pytest tests/test_gpu_dual.py -x -q 2>&1 | tail -2
for v in default dualn64; do
  if [ $v = default ]; then L=paper_2508_02932_b200/libplora.so; else L=build/libplora_$v.so; fi
  echo "== $v"; PLORA_LIB=$L timeout 300 python tools/bench_lora.py 2>&1 | grep -v lora_kernels
done
