#!/bin/bash
# A/B run on the GPU box: variant libraries (build_variants/) on a cases file, optional gpu tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
[ -n "$TESTS" ] && { timeout 1500 python -m pytest tests -m gpu -x -q $TESTS > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; }
timeout 900 python scripts/ab_probe.py $CASES $LIBS > gpurun_out/ab.txt 2>&1
