#!/bin/bash
# ncu --set full of the tcgen05 block executor: conv fp32 (3xTF32) and fp16, C5 batch 256
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for spec in "f32 conv_kernel=5,x_multicast=2" "f16 conv_kernel=5,x_multicast=2"; do
  set -- $spec
  timeout 300 python scripts/conv_one.py $1 $2 > gpurun_out/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tcg -s 1 -c 1 -o gpurun_out/tcg_conv_$1 -f python scripts/conv_one.py $1 $2 > gpurun_out/ncu_tcg_conv_$1.log 2>&1
done
