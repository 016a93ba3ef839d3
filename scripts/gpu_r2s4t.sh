#!/bin/bash
# stream-K: tests + A/B timings (conv per-rank batches, BERT fp32)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streamk or tcgen05 or conv_epilogue or pair or nhwc or kslices or small_batch" > gpurun_out/pytest_sk.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sk.log
{
for sk in 0 1; do
  echo "=== SRT_TCG_STREAMK=$sk"
  SRT_TCG_STREAMK=$sk timeout 300 python scripts/conv_batch_time.py f32 256,128,64,32 "conv_kernel=5,cta_pair=1"
  for s in "3072 768" "768 3072"; do SRT_TCG_STREAMK=$sk timeout 300 python scripts/cfg_time.py $s 16384 f32 "executor=4,cta_pair=1"; done
done
} > gpurun_out/sk_time.log 2>&1
