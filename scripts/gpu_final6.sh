#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --workload bert --dtype bf16 --no-cpu-baseline --retune > gpurun_out/bench_bert_bf16.json 2> gpurun_out/bench_bert_bf16.err
timeout 900 python bench.py --workload rn50_b8 --dtype bf16 --no-cpu-baseline --retune > gpurun_out/bench_rn50_b8_bf16.json 2> gpurun_out/bench_rn50_b8_bf16.err
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
cp profiles/tuned_*bf16*.json gpurun_out/ 2>/dev/null
