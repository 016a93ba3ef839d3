cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
[ -n "$TESTS" ] && { timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; }
for dt in f32 f16; do
  SPARSERT_TUNE_DEBUG=1 timeout 900 python bench.py --workload conv --dtype $dt --no-cpu-baseline --retune > gpurun_out/bench_conv_$dt.json 2> gpurun_out/bench_conv_$dt.err
done
cp profiles/tuned_conv_*.json gpurun_out/ 2>/dev/null
