#!/bin/bash
# retune the conv files (the tuner now has conv fp32 on tcgen05) and the bf16 BERT file, then the default bench line + ncu launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
mkdir -p gpurun_out/old_tuned; cp profiles/tuned_conv_f32_s90_x2.json profiles/tuned_conv_f16_s90_x2.json gpurun_out/old_tuned/
rm -f profiles/tuned_conv_f32_s90_x2.json profiles/tuned_conv_f16_s90_x2.json
timeout 900 python bench.py --workload conv --dtype f32 --secondary "" --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/conv_f32.json 2> gpurun_out/conv_f32.err
timeout 900 python bench.py --workload conv --dtype f16 --secondary "" --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/conv_f16.json 2> gpurun_out/conv_f16.err
cp profiles/tuned_conv_f32_s90_x2.json profiles/tuned_conv_f16_s90_x2.json gpurun_out/
timeout 1200 python bench.py > gpurun_out/default.json 2> gpurun_out/default.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity --secondary "" > gpurun_out/ncu_launch.log 2>&1
echo done
