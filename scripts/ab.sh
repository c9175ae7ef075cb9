#!/bin/bash
# A/B of alternative library builds: for each _ab/<name>.so run the short
# bench of $CONFIGS with that library swapped in (restores the original).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
SO=paper_1905_12146_b200/_build/libphylograd_b200.so
cp $SO /tmp/orig.so
for v in cur ${VARIANTS:-$(ls _ab | sed 's/\.so$//')}; do
  if [ "$v" = cur ]; then cp /tmp/orig.so $SO; else cp _ab/$v.so $SO; fi
  for c in ${CONFIGS:-C4 C5}; do
    timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_$c.json 2>gpurun_out/ab_${v}_$c.err
    python -c "import json; d=json.load(open('gpurun_out/ab_${v}_$c.json')); r=d['roofline']; print('$v $c', round(d['ms_per_step'],2), 'ms frac', round(r['frac'],3))" 2>&1 | tail -1
  done
done
cp /tmp/orig.so $SO
