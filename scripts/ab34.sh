#!/bin/bash
# A/B of library builds on the 4-state configs (see scripts/ab.sh)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
CONFIGS="${CONFIGS:-C2 C3}" bash scripts/ab.sh
