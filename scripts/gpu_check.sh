#!/bin/bash
# One GPU pass (replaces the round-1 gpu_final*.sh variants).  Everything lands in gpurun_out/.
#   TESTS=1      pytest -m gpu + smoke()               (default 1)
#   BENCH=1      default bench line (conv b256 fp32 + BERT secondary), reference arm (default 1)
#   EXTRA="wl:dt ..."  extra bench lines (--no-cpu-baseline), e.g. "rn50_b8:f32 conv:f16"
#   RETUNE=--retune    re-run the autotuner for the EXTRA lines
#   LAUNCHES=1   ncu launch list of the default bench (gpu__time_duration per kernel)
#   NCU_FULL="regex"   one ncu --set full capture of the first timed kernel matching regex
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  timeout ${PYTEST_TIMEOUT:-1800} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if [ "${BENCH:-1}" = 1 ]; then
  timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "rc=$?" >> gpurun_out/bench_default.err
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
for item in ${EXTRA}; do
  wl=${item%%:*}; rest=${item#*:}; dt=${rest%%:*}; sp=90; [ "$rest" != "$dt" ] && sp=${rest#*:}
  timeout 900 python bench.py --workload $wl --dtype $dt --sparsity $sp --secondary '' --no-cpu-baseline ${RETUNE} > gpurun_out/bench_${wl}_${dt}_s${sp}.json 2> gpurun_out/bench_${wl}_${dt}_s${sp}.err
done
cp profiles/tuned_*.json gpurun_out/ 2>/dev/null
if [ "${LAUNCHES:-0}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_default.csv \
    python bench.py --steps 3 --warmup 3 --quick > gpurun_out/launches_default.log 2>&1
fi
if [ -n "${NCU_FULL}" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
    -k regex:"${NCU_FULL}" -c 1 -o gpurun_out/ncu_full -f \
    python bench.py --steps 2 --warmup 3 --quick ${NCU_ARGS} > gpurun_out/ncu_full.log 2>&1
fi
