#!/bin/bash
# tail K slices: tests + A/B (batch = the per-rank shares of 256 images on 1/2/4/8 GPUs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tcgen05 or conv_epilogue or pair or nhwc or kslices" > gpurun_out/pytest_tks.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tks.log
{
for tk in 0 1; do
  echo "=== SRT_TCG_TAIL_KS=$tk"
  SRT_TCG_TAIL_KS=$tk timeout 300 python scripts/conv_batch_time.py f32 256,128,64,32 "conv_kernel=5,cta_pair=1"
  SRT_TCG_TAIL_KS=$tk timeout 300 python scripts/conv_batch_time.py f16 256,128,64,32 "conv_kernel=5,cta_pair=1"
  for s in "3072 768" "768 3072"; do for dt in f16 f32; do
    SRT_TCG_TAIL_KS=$tk timeout 300 python scripts/cfg_time.py $s 16384 $dt "executor=4,cta_pair=1"
  done; done
done
} > gpurun_out/tks_time.log 2>&1
