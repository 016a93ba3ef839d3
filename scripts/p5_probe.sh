#!/bin/bash
# small-layer probe: tile / K-split / multicast / stage variants of RN50 p5 and p7 at batch 8
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
V=""
for R in 2 4 8; do for ks in 1 2 4 8; do for kc in 64 128; do V="$V;warps=16,rows_per_warp=$R,k_split=$ks,k_chunk=$kc"; done; done; done
for cm in 2 4; do for st in 2 4; do V="$V;warps=16,rows_per_warp=8,x_multicast=$cm,k_chunk=64,stages=$st"; done; done
timeout 600 python scripts/cfg_time.py 256 1024 1568 f32 "${V#;}" > gpurun_out/p5_f32.txt 2>&1
timeout 600 python scripts/cfg_time.py 512 2048 392 f32 "${V#;}" > gpurun_out/p7_f32.txt 2>&1
timeout 600 python scripts/cfg_time.py 64 256 25088 f32 "${V#;}" > gpurun_out/p1_f32.txt 2>&1
