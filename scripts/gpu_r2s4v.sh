#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tcgen05 or conv_epilogue or pair or nhwc or kslices or small_batch" > gpurun_out/pytest_v.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_v.log
{
for d in f16 f32; do timeout 300 python scripts/nhwc_time.py $d "conv_kernel=5,cta_pair=1"; done
for s in "3072 768" "768 3072"; do timeout 300 python scripts/cfg_time.py $s 16384 f16 "executor=4,cta_pair=1"; done
timeout 300 python scripts/conv_batch_time.py f16 256,32 "conv_kernel=5,cta_pair=1"
} > gpurun_out/v_time.log 2>&1
