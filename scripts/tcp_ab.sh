cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "tcp" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/ab_probe.py scripts/cases_tcp.json paper_2008_11849_b200/libsparsert.so > gpurun_out/ab.txt 2>&1
WLS="mbv1_b32 rn50_b8" bash scripts/gpu_full_f16.sh
