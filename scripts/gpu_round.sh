#!/bin/bash
# One GPU session: tests, smoke, bench.  Everything under gpurun_out/.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
for ex in ${EXECUTORS:-1}; do
for wl in ${WORKLOADS:-rn50_b8}; do
  for dt in ${DTYPES:-f32}; do
    timeout 600 python bench.py --workload $wl --dtype $dt --executor $ex ${BENCH_ARGS} > gpurun_out/bench_${wl}_${dt}_x${ex}.json 2> gpurun_out/bench_${wl}_${dt}_x${ex}.err
  done
done
done
cp profiles/tuned_*.json gpurun_out/ 2>/dev/null || true
