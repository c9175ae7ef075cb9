#!/bin/bash
# Round evidence on one GPU: full-size ncu captures of the walk kernels in
# $PROFILE_CONFIGS (each command run plain first), the launch list of the
# default bench command, then the bench line of every config and the CPU
# reference arm.  Outputs under gpurun_out/ with tag $TAG.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
TAG=${TAG:-ev}
CONFIGS="${PROFILE_CONFIGS:-C4 C5}" TAG=$TAG bash scripts/profile_all.sh
for c in ${BENCH_CONFIGS:-C2 C3 C4 C5}; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
  echo "bench $c rc=$?"; tail -c 400 gpurun_out/bench_${TAG}_$c.json
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_${TAG}_ref_C3.json 2> gpurun_out/bench_${TAG}_ref_C3.err
echo "ref rc=$?"
