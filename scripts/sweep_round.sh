#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/sweep.jsonl; : > $out
run() { echo "## $*" >> $out; timeout 300 python scripts/sweep.py "$@" >> $out 2>&1; }
for fl in none write writeread; do
run --M 256 --K 64 --N 25088 --dtype f32 --flush $fl --grid "rows_per_warp=4;stages=1,2;warps=8"
run --M 2048 --K 512 --N 392 --dtype f32 --flush $fl --grid "rows_per_warp=4;k_split=1,2;warps=8"
run --M 3072 --K 768 --N 16384 --dtype f32 --flush $fl --reps 5
done
