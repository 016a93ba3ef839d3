cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3x3_tma -s 2 -c 1 -o gpurun_out/conv16f -f python scripts/conv_one.py f16 conv_kernel=2,warps=16,rows_per_warp=4,k_chunk=32 > gpurun_out/ncu_conv16f.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_conv_f16.csv python bench.py --workload conv --dtype f16 --steps 3 --warmup 3 --quick > gpurun_out/launches_conv.log 2>&1
