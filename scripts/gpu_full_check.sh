#!/bin/bash
# full GPU suite + smoke + default bench line (+ ncu launch list of the default step)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi_before.txt
timeout 1200 python bench.py > gpurun_out/default.json 2> gpurun_out/default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/reference.json 2> gpurun_out/reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity --secondary "" > gpurun_out/ncu_launch.log 2>&1
echo done
