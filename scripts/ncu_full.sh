#!/bin/bash
# ncu --set full of one launch of the dominant executor kernel for a few workloads.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for spec in ${NCU_SPECS:-"bert f32 spmm" "bert f16 spmm" "conv f32 conv3x3"}; do
  set -- $spec
  wl=$1; dt=$2; k=$3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 2 -c 1 \
      -o gpurun_out/prof_${wl}_${dt} -f python bench.py --workload $wl --dtype $dt --quick --eager --steps 1 --warmup 1 \
      > gpurun_out/ncu_${wl}_${dt}.log 2>&1
done
