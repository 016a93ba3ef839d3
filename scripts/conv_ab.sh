cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "conv" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for dt in f32 f16; do
timeout 600 python scripts/conv_time.py $dt "warps=16,rows_per_warp=8,k_chunk=29;conv_kernel=2,warps=16,rows_per_warp=8;conv_kernel=2,warps=16,rows_per_warp=4;conv_kernel=2,warps=16,rows_per_warp=8,k_chunk=16;conv_kernel=2,warps=16,rows_per_warp=8,k_chunk=32;conv_kernel=2,warps=8,rows_per_warp=8;conv_kernel=2,warps=16,rows_per_warp=2;conv_kernel=2,warps=16,rows_per_warp=8,k_chunk=64" > gpurun_out/conv_$dt.txt 2>&1
done
