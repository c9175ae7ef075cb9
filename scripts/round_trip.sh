#!/bin/bash
# tests + bench (+ optional ncu of the walk kernel) in one GPU call
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
BENCH_CONFIGS="${BENCH_CONFIGS:-C3}" bash scripts/gpu_check.sh
if [ -n "$NCU" ]; then TAG=${TAG:-rx} CFG=${CFG:-C3} SITES=${SITES:-100000} bash scripts/ncu_walk.sh; fi
