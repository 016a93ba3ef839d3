cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for v in cy2 cy4; do
  SPARSERT_LIB=build_variants/libsparsert_$v.so timeout 900 python -m pytest tests -m gpu -x -q -k "tcp" > gpurun_out/pytest_$v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$v.log
done
timeout 600 python scripts/ab_probe.py scripts/cases_tcp.json build_variants/libsparsert_cy1.so build_variants/libsparsert_cy2.so build_variants/libsparsert_cy4.so > gpurun_out/ab.txt 2>&1
