#!/bin/bash
# retune the tuned files of the given workloads (WL="conv:f32 bert:f16 ..."), then the default
# bench line, its ncu launch list and one ncu --set full capture of the dominant kernel (csv)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/tuned
for wd in ${WL:-conv:f32 conv:f16 conv:bf16 bert:f32 bert:f16 bert:bf16}; do
  w=${wd%%:*}; d=${wd##*:}
  rm -f profiles/tuned_${w}_${d}_s90_x2.json
  timeout 900 python bench.py --workload $w --dtype $d --secondary "" --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/tuned/${w}_${d}.json 2> gpurun_out/tuned/${w}_${d}.err
  cp profiles/tuned_${w}_${d}_s90_x2.json gpurun_out/tuned/ 2>/dev/null
done
timeout 1200 python bench.py > gpurun_out/default.json 2> gpurun_out/default.err
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi_after.txt
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity --secondary "" > gpurun_out/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tcg -s 3 -c 1 -o /tmp/dom -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity --secondary "" > gpurun_out/ncu_dom.log 2>&1 && {
    ncu -i /tmp/dom.ncu-rep --page raw --csv > gpurun_out/ncu_dom_raw.csv 2>&1
    ncu -i /tmp/dom.ncu-rep --page details --csv > gpurun_out/ncu_dom_details.csv 2>&1
  }
fi
echo done
