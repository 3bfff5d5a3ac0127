cd $GRAFT_REPO_ROOT
for i in 1 2; do
  python tools/gemm_waves.py nb2
  PLORA_LIB=build/libplora_nb1.so python tools/gemm_waves.py nb1
done 2>&1 | tee gpurun_out/at_gemm_waves.log
