#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tcgen05 or conv_epilogue or pair" > gpurun_out/pytest_tcg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tcg.log
{
  timeout 300 python scripts/conv_time.py f32 "conv_kernel=5,x_multicast=2;conv_kernel=5,cta_pair=1"
  timeout 300 python scripts/conv_time.py f16 "conv_kernel=5,x_multicast=2;conv_kernel=5,cta_pair=1"
  for s in "3072 768" "768 3072"; do for dt in f16 f32; do
    echo "== $s $dt"
    timeout 300 python scripts/cfg_time.py $s 16384 $dt "executor=4,x_multicast=2;executor=4,cta_pair=1"
  done; done
} > gpurun_out/pair_time.log 2>&1
