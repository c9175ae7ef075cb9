#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
for ms in 0 100 1000; do
  python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --clock-ms $ms 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('clock-ms', $ms, 'ms/step', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), 'walk', round(d['roofline']['walk_ms'],2), d['clocks'])"
done
