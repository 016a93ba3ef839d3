#!/bin/bash
# im2col conv: vectorised NHWC pack + tile width filling the cluster rounds: tests + timings
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv_tcgen05 or conv_epilogue or pair" > gpurun_out/pytest_bn.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bn.log
{
for bn in 256 0 224 192 176; do
  echo "=== SRT_CONV_BN=$bn"
  SRT_CONV_BN=$bn timeout 300 python scripts/conv_time.py f32 "conv_kernel=5,cta_pair=1;conv_kernel=5,x_multicast=2"
  SRT_CONV_BN=$bn timeout 300 python scripts/conv_time.py f16 "conv_kernel=5,cta_pair=1;conv_kernel=5,x_multicast=2"
done
} > gpurun_out/bn_time.log 2>&1
python scripts/conv_one.py f32 conv_kernel=5,cta_pair=1 > gpurun_out/plain_one.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_conv_one.csv python scripts/conv_one.py f32 conv_kernel=5,cta_pair=1 > /dev/null 2>&1
