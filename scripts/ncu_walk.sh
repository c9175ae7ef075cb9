#!/bin/bash
# ncu capture of one walk_kernel launch (the 2nd evaluation's) + the launch list.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
CFG=${CFG:-C3}; SITES=${SITES:-100000}; TAG=${TAG:-r01}
CMD="python scripts/profile_walk.py --config $CFG --sites $SITES --evals 2"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:walk -s 1 -c 1 -o gpurun_out/walk_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/plain_$TAG.log; tail -5 gpurun_out/ncu_full_$TAG.log
