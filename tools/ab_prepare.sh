#!/bin/bash
# Prepare an A/B baseline: check out <ref> (default HEAD) into build/ab_base and build
# its libplora.so there, so one gpurun call can time both trees on the same box
# (tools/ab_run.sh).  build/ travels with the gpurun snapshot.
set -e
REF=${1:-HEAD}
cd "$(dirname "$0")/.."
rm -rf build/ab_base
git worktree prune
git worktree add -f --detach build/ab_base "$REF" >/dev/null
(cd build/ab_base && python __graft_entry__.py build >/dev/null)
echo "baseline $REF ready in build/ab_base"
