#!/bin/bash
# Round-2 GPU round trip: smoke, the whole GPU suite, bench C3 (+ reference
# arm), small-P C2 walk timings (the 8-GPU shard proxy).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/smoke.log; tail -12 gpurun_out/pytest_gpu.log
for cfg in ${BENCH_CONFIGS-C3}; do
  timeout 900 python bench.py --config $cfg --steps ${BENCH_STEPS:-10} --warmup 3 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "bench $cfg rc=$?"
  cat gpurun_out/bench_$cfg.json
done
if [ -n "$REF" ]; then
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
  grep -c libphylograd /proc/self/maps >/dev/null
fi
for s in ${SMALLP}; do
  python scripts/profile_walk.py --config C2 --sites $s --evals 3 2>&1 | tail -1
done
