#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
for rep in 1 2; do
for bn in 0 224 208 256; do
  echo "=== SRT_CONV_BN=$bn"
  SRT_CONV_BN=$bn timeout 300 python scripts/conv_batch_time.py f32 256 "conv_kernel=5,cta_pair=1"
done; done
} > gpurun_out/bn2_time.log 2>&1
