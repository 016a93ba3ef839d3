#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/final2
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "tcgen05 or conv_epilogue or pair or nhwc or kslices or tuned" > gpurun_out/final2/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final2/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final2/smoke.log
timeout 1200 python bench.py > gpurun_out/final2/default.json 2> gpurun_out/final2/default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final2/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity --secondary "" > gpurun_out/final2/ncu_launch.log 2>&1
echo done
