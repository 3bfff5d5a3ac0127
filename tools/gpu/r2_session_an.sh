cd $GRAFT_REPO_ROOT
for i in 1 2; do for o in "--no-overlap-k5" "--overlap-k5"; do
  timeout 900 python tools/split_projection.py --gpus 4,8 --steps 5 --warmup 2 --graph $o 2>&1 | grep '"gpus"' | sed "s/^/$o /"
done; done
