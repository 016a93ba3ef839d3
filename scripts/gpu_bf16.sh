#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for wl in bert rn50_b8; do
  timeout 900 python bench.py --workload $wl --dtype bf16 --no-cpu-baseline --retune > gpurun_out/bench_${wl}_bf16.json 2> gpurun_out/bench_${wl}_bf16.err
done
cp profiles/tuned_*bf16*.json gpurun_out/ 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
