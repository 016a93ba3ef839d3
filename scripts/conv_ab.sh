cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "conv or tail or ragged or rel_l2 or exact" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/conv_time.py f32 "conv_kernel=2,warps=16,rows_per_warp=8,k_chunk=32" > gpurun_out/conv_f32.txt 2>&1
timeout 600 python scripts/conv_time.py f16 "conv_kernel=2,warps=16,rows_per_warp=4,k_chunk=32;conv_kernel=2,warps=16,rows_per_warp=8,k_chunk=32" > gpurun_out/conv_f16.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:"pad_conv|conv3x3_tma" -c 4 --csv python scripts/conv_one.py f16 conv_kernel=2,warps=16,rows_per_warp=4,k_chunk=32 > gpurun_out/ncu_pad_f16.csv 2>&1
timeout 600 python scripts/ab_probe.py scripts/cases_pf.json paper_2008_11849_b200/libsparsert.so > gpurun_out/ab.txt 2>&1
