cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "conv" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/conv_time.py f32 "conv_kernel=3,warps=16,rows_per_warp=8,k_chunk=29;conv_kernel=2,warps=16,rows_per_warp=8,k_chunk=32" > gpurun_out/conv_f32.txt 2>&1
timeout 600 python scripts/conv_time.py f16 "conv_kernel=3,warps=16,rows_per_warp=8,k_chunk=18;conv_kernel=2,warps=16,rows_per_warp=4,k_chunk=32" > gpurun_out/conv_f16.txt 2>&1
