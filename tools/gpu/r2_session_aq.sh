cd $GRAFT_REPO_ROOT
timeout 300 python tools/dbg/launch_cost.py 2>&1 | tail -8
