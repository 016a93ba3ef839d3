#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tcgen05 or conv_epilogue or pair" > gpurun_out/pytest_tcg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tcg.log
CONVCFG="conv_kernel=5,x_multicast=2;conv_kernel=5,cta_pair=1" SPMMCFG="executor=4,x_multicast=2;executor=4,cta_pair=1" bash scripts/gpu_ab_lib.sh
