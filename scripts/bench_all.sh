#!/bin/bash
# short bench of every config (device-leg summary line per config)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
for c in ${CONFIGS:-C2 C3 C4 C5}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup 2 --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
  echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']; print('$c', round(d['ms_per_step'],2), 'ms', '%.3e'%d['value'], r['bound'], 'frac', round(r['frac'],3), d['config']['geometry']['kernel'])" 2>&1 | tail -1
done
