#!/bin/bash
# The level-scheduled traversal (walkl) against the persistent walks at small P.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_walk4.py -m gpu -q -x -p no:cacheprovider -k "${PYTEST_K:-walkl}" > gpurun_out/pytest_walkl.log 2>&1
echo "pytest rc=$?"; tail -8 gpurun_out/pytest_walkl.log
for s in ${SITES:-1250 2500 5000 10000 20000}; do
  for v in 0 1; do
    echo "C2 sites=$s PG_WALKL=$v: $(PG_WALKL=$v timeout 300 python scripts/profile_walk.py --config C2 --sites $s --evals 4 2>&1 | tail -1 | sed 's/geometry.*kernel/kernel/')"
  done
done
