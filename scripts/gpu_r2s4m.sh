#!/bin/bash
# 16-bit epilogue with 8 warps: tests + A/B against the 4-warp build
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tcgen05 or conv_epilogue or pair or nhwc" > gpurun_out/pytest_epi8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_epi8.log
CONVCFG="conv_kernel=5,cta_pair=1;conv_kernel=5,x_multicast=2" SPMMCFG="executor=4,cta_pair=1;executor=4,x_multicast=2" bash scripts/gpu_ab_lib.sh
