cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_tcp -s 2 -c 1 -o gpurun_out/tcp -f python scripts/one_launch.py --M 3072 --K 768 --N 16384 --dtype f16 --opts executor=3 > gpurun_out/ncu_tcp.log 2>&1
ncu -i gpurun_out/tcp.ncu-rep --page raw --csv > gpurun_out/tcp.csv 2>&1
ncu -i gpurun_out/tcp.ncu-rep --page details --csv > gpurun_out/tcp_details.csv 2>&1
ncu -i gpurun_out/tcp.ncu-rep --page source --csv --print-source sass > gpurun_out/tcp_sass.csv 2>&1
