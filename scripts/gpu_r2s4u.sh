#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
echo "=== default"; timeout 300 python scripts/conv_batch_time.py f32 256,128,64,32 "conv_kernel=5,cta_pair=1"
echo "=== TAIL_KS=0"; SRT_TCG_TAIL_KS=0 timeout 300 python scripts/conv_batch_time.py f32 128,32 "conv_kernel=5,cta_pair=1"
echo "=== BN=256"; SRT_CONV_BN=256 timeout 300 python scripts/conv_batch_time.py f32 128 "conv_kernel=5,cta_pair=1"
} > gpurun_out/chk_time.log 2>&1
