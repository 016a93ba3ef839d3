#!/bin/bash
# A/B of two builds in one box session: SPARSERT_LIB=<variant> vs the in-tree library
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
OLD=${OLD:-paper_2008_11849_b200/build_variant/libsparsert_old.so}
CONVCFG=${CONVCFG:-"conv_kernel=5,x_multicast=2;conv_kernel=5"}
SPMMCFG=${SPMMCFG:-"executor=4,x_multicast=2;executor=4"}
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/ab_clocks.csv &
SMI=$!
{
for rep in 1 2; do
for lib in old new; do
  if [ $lib = old ]; then export SPARSERT_LIB=$OLD; else unset SPARSERT_LIB; fi
  echo "=== $lib rep $rep"
  for s in "3072 768" "768 3072"; do for dt in f16 f32; do
    echo "== $s $dt"
    timeout 300 python scripts/cfg_time.py $s 16384 $dt "$SPMMCFG"
  done; done
  timeout 300 python scripts/conv_time.py f16 "$CONVCFG"
  timeout 300 python scripts/conv_time.py f32 "$CONVCFG"
done; done
} > gpurun_out/ab_lib.log 2>&1
kill $SMI
echo done
