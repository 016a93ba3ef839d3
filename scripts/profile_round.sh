#!/bin/bash
# ncu evidence for a bench line: (1) launch list with per-launch duration and DRAM bytes of
# every executor launch inside the timed NVTX range; (2) --set full of the dominant kernel.
# usage: profile_round.sh WORKLOAD DTYPE DOMINANT_LAYER_INDEX
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
wl=$1; dt=$2; dom=$3
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/launches_${wl}_${dt}.csv \
    python bench.py --workload $wl --dtype $dt --steps 3 --warmup 3 --quick > gpurun_out/launches_${wl}_${dt}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
    -k regex:"spmm|srt_jit|conv3x3" -s $dom -c 1 -o gpurun_out/full_${wl}_${dt} -f \
    python bench.py --workload $wl --dtype $dt --steps 2 --warmup 3 --quick > gpurun_out/full_${wl}_${dt}.log 2>&1
