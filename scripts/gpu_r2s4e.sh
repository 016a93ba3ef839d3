#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tcgen05 or conv_epilogue" > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_split.log
OLD=paper_2008_11849_b200/build_variant/libsparsert_old.so bash scripts/gpu_ab_lib.sh
{
for st in 0 8; do
  echo "=== SRT_TCG_SPLIT_TAIL=$st"
  SRT_TCG_SPLIT_TAIL=$st timeout 300 python scripts/conv_time.py f32 "conv_kernel=5,x_multicast=2"
  SRT_TCG_SPLIT_TAIL=$st timeout 300 python scripts/conv_time.py f16 "conv_kernel=5,x_multicast=2"
  SRT_TCG_SPLIT_TAIL=$st timeout 300 python scripts/cfg_time.py 3072 768 16384 f16 "executor=4,x_multicast=2;executor=4"
done
} > gpurun_out/split_time.log 2>&1
