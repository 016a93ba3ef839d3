#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for wl in bert mbv1_b32 rn50_b8 rn50_b1; do
  timeout 900 python bench.py --workload $wl --dtype f16 --no-cpu-baseline > gpurun_out/bench_${wl}_f16.json 2> gpurun_out/bench_${wl}_f16.err
done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_tcp -s 2 -c 1 -o gpurun_out/tcp -f python scripts/one_launch.py --M 3072 --K 768 --N 16384 --dtype f16 --opts executor=3 > gpurun_out/ncu_tcp.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_bert_f16.csv python bench.py --workload bert --dtype f16 --steps 3 --warmup 3 --quick > gpurun_out/launches_bert.log 2>&1
