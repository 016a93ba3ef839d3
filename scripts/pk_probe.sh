#!/bin/bash
# packed conv kernel: parity tests + timing sweep of its tile options against the TMA-fed kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "conv" > gpurun_out/pytest_conv.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_conv.log
V="conv_kernel=2,rows_per_warp=8,warps=16,k_chunk=32"
for cc in ${CCS:-4 8 12 16}; do for RW in ${RWS:-8:16 4:16 8:12 8:8}; do V="$V;conv_kernel=4,rows_per_warp=${RW%%:*},warps=${RW##*:},k_chunk=$cc"; done; done
timeout 600 python scripts/conv_time.py f32 "$V" > gpurun_out/pk_f32.txt 2>&1
timeout 600 python scripts/conv_time.py f16 "${V//k_chunk=32/k_chunk=16}" > gpurun_out/pk_f16.txt 2>&1
if [ -n "$NCU_OPTS" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv3x3_il -s 1 -c 1 -o gpurun_out/ncu_pk -f \
    python scripts/conv_time.py ${NCU_DT:-f32} "$NCU_OPTS" > gpurun_out/ncu_pk.log 2>&1
fi
