cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
i=0
for spec in "64 256 25088 warps=16,rows_per_warp=2,k_chunk=128" "64 256 25088 warps=16,rows_per_warp=4,k_chunk=128" "512 2048 392 warps=16,rows_per_warp=4,k_chunk=128,k_split=4" "256 1024 1568 warps=16,rows_per_warp=2,k_chunk=128"; do
  set -- $spec
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 2 -c 1 -o gpurun_out/q$i -f python scripts/one_launch.py --M $1 --K $2 --N $3 --opts $4 > gpurun_out/q$i.log 2>&1
  ncu -i gpurun_out/q$i.ncu-rep --page raw --csv > gpurun_out/q$i.csv 2>&1; ncu -i gpurun_out/q$i.ncu-rep --page details --csv > gpurun_out/q${i}_details.csv 2>&1; rm -f gpurun_out/q$i.ncu-rep
  i=$((i+1))
done
