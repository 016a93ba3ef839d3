#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/sweep.jsonl; : > $out
run() { echo "## $*" >> $out; timeout 300 python scripts/sweep.py "$@" >> $out 2>&1; }
run --M 256 --K 64 --N 25088 --dtype f32 --flush write --grid "rows_per_warp=2,4,8;warps=8;stages=2,3"
run --M 64 --K 256 --N 25088 --dtype f32 --flush write --grid "rows_per_warp=2,4;warps=8;stages=2,3;k_split=1"
run --M 2048 --K 512 --N 392 --dtype f32 --flush write --grid "rows_per_warp=2,4;warps=8;k_split=1,2,4"
run --M 512 --K 2048 --N 392 --dtype f32 --flush write --grid "rows_per_warp=2,4;warps=8;k_split=1,4,8"
run --M 3072 --K 768 --N 16384 --dtype f32 --flush write --reps 5 --grid "rows_per_warp=4,8;warps=8;stages=2,3"
run --M 3072 --K 768 --N 16384 --dtype f16 --flush write --reps 5 --grid "rows_per_warp=4,8;warps=8;stages=2,3"
