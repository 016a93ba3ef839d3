cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; : > gpurun_out/tma4d.txt
for v in "10 34 1 0 0 1 20" "10 34 2 0 0 1 20" "10 34 4 0 0 1 16" "10 34 4 0 0 1 20" "10 34 1 0 0 1 32" "10 34 0 0 0 1 20"; do
  timeout 60 scripts/micro/tma4d $v >> gpurun_out/tma4d.txt 2>&1
done
