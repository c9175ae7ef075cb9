#!/bin/bash
# A/B of engine environment switches on one box: for each "NAME=ENV..." entry
# of $VARIANTS run the short bench of $CONFIGS with that environment.
#   VARIANTS="f=PG_WALK4F=1 nof=PG_WALK4F=0" CONFIGS=C3 scripts/ab_env.sh
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
for v in ${VARIANTS}; do
  name=${v%%=*}; envs=${v#*=}
  for c in ${CONFIGS:-C3}; do
    env ${envs//,/ } timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab_${name}_$c.json 2>gpurun_out/ab_${name}_$c.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_${name}_$c.json')); r=d['roofline']; p=d.get('parity') or {}
print('$name $c', round(d['ms_per_step'],2), 'ms walk', round(r['walk_ms'],2), 'frac', round(r['frac'],3), d['geometry']['kernel'], 'parity', p.get('within_1e-9'), p.get('grad_max_rel_to_condition'))" 2>&1 | tail -1
  done
done
