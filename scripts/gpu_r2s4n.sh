#!/bin/bash
# tcgen05 K slices (small N): tests + timings of the RN50 batch-8 / MobileNet-like shapes
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "kslices or tcgen05_blocks or pair_exact" > gpurun_out/pytest_ks.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ks.log
{
for dt in f32 f16; do
  for s in "512 2048 392" "2048 512 392" "256 1024 1568" "1024 256 1568" "128 512 6272" "512 128 6272"; do
    echo "== $s $dt"
    timeout 300 python scripts/cfg_time.py $s $dt "executor=0;executor=4;executor=4,cta_pair=1;executor=4,cta_pair=1,k_split=2;executor=4,cta_pair=1,k_split=4;executor=4,cta_pair=1,k_split=8;executor=4,cta_pair=1,k_split=16;executor=4,k_split=4;executor=4,k_split=8;executor=4,k_split=16"
  done
done
} > gpurun_out/ks_time.log 2>&1
