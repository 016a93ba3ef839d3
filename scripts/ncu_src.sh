#!/bin/bash
# ncu --set full with source of one launch per case; exports raw / details / source CSVs only.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
i=0
for spec in $NCU_CASES; do
  IFS=: read M K N opts dt <<< "$spec"
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 2 -c 1 -o gpurun_out/s$i -f python scripts/one_launch.py --M $M --K $K --N $N --opts $opts --dtype ${dt:-f32} > gpurun_out/s$i.log 2>&1
  ncu -i gpurun_out/s$i.ncu-rep --page raw --csv > gpurun_out/s$i.csv 2>&1
  ncu -i gpurun_out/s$i.ncu-rep --page details --csv > gpurun_out/s${i}_details.csv 2>&1
  ncu -i gpurun_out/s$i.ncu-rep --page source --csv --print-source sass > gpurun_out/s${i}_sass.csv 2>&1
  rm -f gpurun_out/s$i.ncu-rep
  i=$((i+1))
done
