#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "nhwc or conv_tcgen05 or conv_epilogue" > gpurun_out/pytest_nhwc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_nhwc.log
