#!/bin/bash
# Launch list + ncu --set full of two layers (first and dominant) of a workload.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
wl=${WL:-rn50_b8}; dt=${DT:-f32}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/launches_${wl}_${dt}.csv \
    python bench.py --workload $wl --dtype $dt --steps 3 --warmup 3 --quick > gpurun_out/launches_${wl}_${dt}.log 2>&1
for dom in ${DOMS:-0 6}; do
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
    -k regex:"spmm|srt_jit|conv3x3" -s $dom -c 1 -o gpurun_out/full_${wl}_${dt}_$dom -f \
    python bench.py --workload $wl --dtype $dt --steps 2 --warmup 3 --quick > gpurun_out/full_${wl}_${dt}_$dom.log 2>&1
done
