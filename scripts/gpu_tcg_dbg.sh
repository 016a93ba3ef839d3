#!/bin/bash
# tcgen05 block executor diagnostics: full kernel / no Y stores / no MMAs (SRT_TCG_DBG)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
for dbg in 0 1 2 3; do
  echo "== SRT_TCG_DBG=$dbg"
  for s in "3072 768" "768 3072"; do
    SRT_TCG_DBG=$dbg timeout 120 python scripts/cfg_time.py $s 16384 f16 "executor=4;executor=4,x_multicast=2"
    SRT_TCG_DBG=$dbg timeout 120 python scripts/cfg_time.py $s 16384 f32 "executor=4"
  done
done
} > gpurun_out/tcg_dbg.log 2>&1
