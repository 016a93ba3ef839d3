#!/bin/bash
# one compute-sanitizer tool per gpurun call (TOOL=memcheck|synccheck|racecheck)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool ${TOOL:-memcheck} --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_${TOOL:-memcheck}.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_${TOOL:-memcheck}.log
