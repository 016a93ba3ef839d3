#!/bin/bash
# split tail as column slices + conv k-block order (channel block, dx, dy): tests, A/B timings
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tcgen05 or conv_epilogue" > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_split.log
{
for st in 0 8; do
  echo "=== SRT_TCG_SPLIT_TAIL=$st"
  SRT_TCG_SPLIT_TAIL=$st timeout 300 python scripts/conv_time.py f32 "conv_kernel=5,x_multicast=2;conv_kernel=5"
  SRT_TCG_SPLIT_TAIL=$st timeout 300 python scripts/conv_time.py f16 "conv_kernel=5,x_multicast=2;conv_kernel=5"
  for s in "3072 768" "768 3072"; do for dt in f32 f16; do
    echo "== $s $dt"
    SRT_TCG_SPLIT_TAIL=$st timeout 300 python scripts/cfg_time.py $s 16384 $dt "executor=4,x_multicast=2;executor=4"
  done; done
done
} > gpurun_out/split_time.log 2>&1
echo done
