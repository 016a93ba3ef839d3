cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for spec in "f32 conv_kernel=2,warps=16,rows_per_warp=8,k_chunk=32" "f16 conv_kernel=2,warps=16,rows_per_warp=4,k_chunk=32"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3x3_tma -s 2 -c 1 -o gpurun_out/conv_$1 -f python scripts/conv_one.py $1 $2 > gpurun_out/ncu_conv_$1.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pad_conv -c 3 --csv python scripts/conv_one.py $1 $2 > gpurun_out/ncu_pad_$1.csv 2>&1
done
