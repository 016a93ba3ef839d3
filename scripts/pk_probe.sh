#!/bin/bash
# packed conv kernel: parity tests + timing sweep of its tile options against the TMA-fed kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "conv" > gpurun_out/pytest_conv.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_conv.log
V="conv_kernel=2,rows_per_warp=8,warps=16,k_chunk=32"
for cc in 4 8 12 16 24; do for R in 8 4; do V="$V;conv_kernel=4,rows_per_warp=$R,warps=16,k_chunk=$cc"; done; done
V="$V;conv_kernel=4,rows_per_warp=16,warps=16,k_chunk=8;conv_kernel=4,rows_per_warp=8,warps=8,k_chunk=8;conv_kernel=4,rows_per_warp=16,warps=8,k_chunk=8"
timeout 600 python scripts/conv_time.py f32 "$V" > gpurun_out/pk_f32.txt 2>&1
timeout 600 python scripts/conv_time.py f16 "${V//k_chunk=32/k_chunk=64}" > gpurun_out/pk_f16.txt 2>&1
