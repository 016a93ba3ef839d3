#!/bin/bash
# A/B: before the K-slice commits (3d40f42) vs now, BERT fp16 / conv fp16 / conv fp32
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
OLD=paper_2008_11849_b200/build_variant/libsparsert_old.so
{
for rep in 1 2; do for lib in old new; do
  if [ $lib = old ]; then export SPARSERT_LIB=$OLD; else unset SPARSERT_LIB; fi
  echo "=== $lib"
  for s in "3072 768" "768 3072"; do timeout 300 python scripts/cfg_time.py $s 16384 f16 "executor=4,cta_pair=1"; done
  timeout 300 python scripts/cfg_time.py 3072 768 16384 f32 "executor=4,cta_pair=1"
  timeout 300 python scripts/conv_time.py f16 "conv_kernel=5,cta_pair=1"
done; done
} > gpurun_out/ab_ks.log 2>&1
