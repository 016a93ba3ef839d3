#!/bin/bash
# conv fp32 on the tcgen05 block executor (3xTF32): tests + warm timings
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv_tcgen05 or conv_epilogue" > gpurun_out/pytest_convtf.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_convtf.log
{
echo "== conv f32"
timeout 300 python scripts/conv_time.py f32 "conv_kernel=4,rows_per_warp=4,warps=16,k_chunk=32;conv_kernel=5;conv_kernel=5,x_multicast=2"
echo "== conv f16"
timeout 300 python scripts/conv_time.py f16 "conv_kernel=5;conv_kernel=5,x_multicast=2"
} > gpurun_out/convtf_time.log 2>&1
echo done
