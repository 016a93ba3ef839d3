cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "tcp" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/tcp_time.txt
for shp in "3072 768 16384" "768 3072 16384" "1024 1024 1568" "2048 512 392" "512 2048 392" "64 256 25088"; do
  timeout 300 python scripts/cfg_time.py $shp f16 "executor=3;warps=16,rows_per_warp=4,k_chunk=128" >> gpurun_out/tcp_time.txt 2>&1
done
