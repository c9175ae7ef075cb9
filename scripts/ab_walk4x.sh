#!/bin/bash
# A/B of the category-parallel walk4x against walk4 (PG_WALK4X=0) + parity tests.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_walk4.py tests/test_gpu_fullsize.py tests/test_clock.py \
  tests/test_cpp_facade.py -m gpu -q -x -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_ab.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_ab.log
for cfg in ${CFGS:-C3 C2}; do
  for v in 0 1; do
    PG_WALK4X=$v timeout 600 python scripts/profile_walk.py --config $cfg --sites ${SITES:-0} --evals 4 > gpurun_out/ab_${cfg}_x$v.log 2>&1
    echo "$cfg PG_WALK4X=$v"; tail -2 gpurun_out/ab_${cfg}_x$v.log
  done
done
