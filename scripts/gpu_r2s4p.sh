#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tcgen05 or conv_epilogue or pair or nhwc or kslices" > gpurun_out/pytest_tks.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tks.log
{
for tk in 0 1; do
  echo "=== SRT_TCG_TAIL_KS=$tk"
  SRT_TCG_TAIL_KS=$tk timeout 300 python scripts/conv_batch_time.py f32 256,128,64,32 "conv_kernel=5,cta_pair=1"
  SRT_TCG_TAIL_KS=$tk timeout 300 python scripts/cfg_time.py 3072 768 16384 f32 "executor=4,cta_pair=1"
done
for bn in 256 176 128; do
  echo "=== SRT_CONV_BN=$bn"
  SRT_CONV_BN=$bn timeout 300 python scripts/conv_batch_time.py f32 128,64,32 "conv_kernel=5,cta_pair=1"
done
timeout 300 python scripts/conv_batch_time.py f16 256,128,64,32 "conv_kernel=5,cta_pair=1"
} > gpurun_out/tks_time.log 2>&1
