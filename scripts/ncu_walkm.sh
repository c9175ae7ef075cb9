#!/bin/bash
# ncu captures of the DMMA walk kernel on C4 and C5 samples
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
TAG=${TAG:-m1}
for cfg in C4 C5; do
  CMD="python scripts/profile_walk.py --config $cfg --sites ${SITES:-20000} --evals 2"
  $CMD > gpurun_out/plain_${TAG}_$cfg.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:walk -s 1 -c 1 -o gpurun_out/walkm_${TAG}_$cfg -f $CMD > gpurun_out/ncu_${TAG}_$cfg.log 2>&1
  echo "$cfg rc=$?"; tail -2 gpurun_out/plain_${TAG}_$cfg.log
done
