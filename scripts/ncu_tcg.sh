#!/bin/bash
# ncu --set full of the tcgen05 block executor (conv C5 batch 256), exported to csv on the box
# (raw metrics + source page), the .ncu-rep itself is not brought back (size)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for spec in ${NCU_SPECS:-"f32 conv_kernel=5,x_multicast=2"}; do
  set -- ${spec//:/ }
  tag=$1_${2//[=,]/_}
  timeout 300 python scripts/conv_one.py $1 $2 > gpurun_out/plain_$tag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tcg -s 1 -c 1 -o /tmp/tcg_$tag -f python scripts/conv_one.py $1 $2 > gpurun_out/ncu_$tag.log 2>&1 && {
    ncu -i /tmp/tcg_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$tag.csv 2>&1
    ncu -i /tmp/tcg_$tag.ncu-rep --page details --csv > gpurun_out/ncu_details_$tag.csv 2>&1
    ncu -i /tmp/tcg_$tag.ncu-rep --page source --csv > gpurun_out/ncu_source_$tag.csv 2>&1
  }
done
