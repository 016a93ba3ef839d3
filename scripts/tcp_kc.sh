cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
SPARSERT_LIB=build_variants/libsparsert_kc32.so timeout 900 python -m pytest tests -m gpu -x -q -k "tcp" > gpurun_out/pytest_kc32.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_kc32.log
timeout 600 python scripts/ab_probe.py scripts/cases_tcp.json build_variants/libsparsert_kc64.so build_variants/libsparsert_kc32.so > gpurun_out/ab.txt 2>&1
