#!/bin/bash
# Round-2 evidence on one GPU: smoke, the whole GPU suite, bench lines for
# every config (+ the CPU reference arm), full-size ncu captures of the walk
# kernels, the launch list of the default bench command, and a probe for the
# reference's third-party headers.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
TAG=${TAG:-r22}
(ls -d /usr/include/eigen3 /usr/local/include/eigen3 /usr/include/boost/math 2>&1; \
 find / -maxdepth 4 -name "Eigen" -type d 2>/dev/null | head -3) > gpurun_out/probe_eigen_boost_$TAG.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log; tail -6 gpurun_out/pytest_gpu_$TAG.log
for c in ${BENCH_CONFIGS:-C3 C2 C4 C5}; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
  echo "bench $c rc=$?"; tail -c 300 gpurun_out/bench_${TAG}_$c.json
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_${TAG}_ref_C3.json 2> gpurun_out/bench_${TAG}_ref_C3.err
echo "ref rc=$?"
[ -n "$NO_NCU" ] || CONFIGS="${PROFILE_CONFIGS:-C3 C2 C4 C5}" TAG=$TAG bash scripts/profile_all.sh
