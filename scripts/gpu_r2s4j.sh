#!/bin/bash
# conv through im2col TMA: tests + A/B timings against the interleaved copies
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv_tcgen05 or conv_epilogue" > gpurun_out/pytest_i2c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_i2c.log
{
for ic in 0 1; do
  echo "=== SRT_CONV_IM2COL=$ic"
  SRT_CONV_IM2COL=$ic timeout 300 python scripts/conv_time.py f32 "conv_kernel=5;conv_kernel=5,x_multicast=2;conv_kernel=5,cta_pair=1"
  SRT_CONV_IM2COL=$ic timeout 300 python scripts/conv_time.py f16 "conv_kernel=5;conv_kernel=5,x_multicast=2;conv_kernel=5,cta_pair=1"
done
} > gpurun_out/i2c_time.log 2>&1
