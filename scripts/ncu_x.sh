#!/bin/bash
# ncu --set full of one walk launch (2nd evaluation) for env-selected variants
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
CMD="python scripts/profile_walk.py --config ${CFG:-C3} --sites ${SITES:-100000} --evals 2"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:walk -s 1 -c 1 -o gpurun_out/${TAG} -f $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/plain_${TAG}.log; tail -3 gpurun_out/ncu_${TAG}.log
