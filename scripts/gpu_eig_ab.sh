#!/bin/bash
# A/B of the factored (eigen) walk4s variant on C3 (PG_WALK4S_EIG), with the
# 4-state parity suite first.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "${PYTEST_K:-walk4 or fullsize}" > gpurun_out/pytest_w4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_w4.log
tail -3 gpurun_out/pytest_w4.log
fi
VARIANTS="${VARIANTS:-eig=PG_WALK4S_EIG=1 noeig=PG_WALK4S_EIG=0 eigb=PG_WALK4S_EIG=1 noeigb=PG_WALK4S_EIG=0}" CONFIGS=${CONFIGS:-C3} bash scripts/ab_env.sh
for f in gpurun_out/ab_*_C3.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['clocks']['sm_mhz'])"; done
