#!/bin/bash
# ncu evidence for the bench workloads: one --set full capture of the walk
# kernel per config at its FULL bench size (2nd evaluation), plus the launch
# list of the default bench command.  Run each command plain first (ncu rule).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
TAG=${TAG:-final}
for cfg in ${CONFIGS:-C3 C2 C4 C5}; do
  CMD="python scripts/profile_walk.py --config $cfg --sites 0 --evals 2"
  $CMD > gpurun_out/pf_${TAG}_$cfg.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:walk -s 1 -c 1 -o gpurun_out/walk_${TAG}_$cfg -f $CMD > gpurun_out/ncu_${TAG}_$cfg.log 2>&1
  echo "$cfg rc=$?"; tail -1 gpurun_out/pf_${TAG}_$cfg.log
done
BCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --also \"\""
$BCMD > gpurun_out/bench_plain_${TAG}.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_${TAG}.csv $BCMD > gpurun_out/ncu_launch_bench_${TAG}.log 2>&1
echo "launch list rc=$?"
